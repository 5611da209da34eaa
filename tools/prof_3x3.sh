set -e
export N=256
LAYER=256,256,14,3 python tools/one_fwd.py > gpurun_out/p1.log 2>&1
LAYER=256,256,14,3 python tools/one_upd.py > gpurun_out/p2.log 2>&1
LAYER=64,64,56,3 python tools/one_fwd.py > gpurun_out/p3.log 2>&1
LAYER=64,64,56,3 python tools/one_upd.py > gpurun_out/p4.log 2>&1
LAYER=256,256,14,3 ncu --set full --clock-control none --import-source on -k regex:conv_fwd -s 2 -c 1 -o gpurun_out/r02_3x3_l3_fwd python tools/one_fwd.py > /dev/null 2>&1
LAYER=256,256,14,3 ncu --set full --clock-control none --import-source on -k regex:conv_upd_kernel -s 2 -c 1 -o gpurun_out/r02_3x3_l3_upd python tools/one_upd.py > /dev/null 2>&1
LAYER=64,64,56,3 ncu --set full --clock-control none --import-source on -k regex:conv_fwd -s 2 -c 1 -o gpurun_out/r02_3x3_l1_fwd python tools/one_fwd.py > /dev/null 2>&1
LAYER=64,64,56,3 ncu --set full --clock-control none --import-source on -k regex:conv_upd_kernel -s 2 -c 1 -o gpurun_out/r02_3x3_l1_upd python tools/one_upd.py > /dev/null 2>&1
