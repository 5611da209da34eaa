# second round-2 capture set (after the packed-image / cross-stacking kernels): the new
# dominant kernel group (the fused 64->256 1x1 forward with the residual add) and the
# reworked 7x7 3x3 passes, plus a refreshed l1 3x3 update; summarised on the box
set -x
ncu --set full --clock-control none --import-source on -k regex:conv_fwd -s 2 -c 1 -o gpurun_out/r02_ncu_l1_1x1_res_F python tools/one_fused_fwd.py 64 256 56 > /dev/null 2>&1
LAYER=512,512,7,3 ncu --set full --clock-control none --import-source on -k regex:conv_upd_kernel -s 2 -c 1 -o gpurun_out/r02_ncu_l4_3x3_U python tools/one_upd.py > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:conv_fwd -s 2 -c 1 -o gpurun_out/r02_ncu_l4_3x3_F python tools/one_layer.py 512 512 7 3 f > /dev/null 2>&1
LAYER=64,64,56,3 ncu --set full --clock-control none --import-source on -k regex:conv_upd_kernel -s 2 -c 1 -o gpurun_out/r02_ncu_l1_3x3_U python tools/one_upd.py > /dev/null 2>&1
