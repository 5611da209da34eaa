# Round-2 evidence on one B200 (outputs under gpurun_out/, summarised into profiles/ by
# tools/r02_summarise.py): the default bench line, the cfg2 line, a one-step launch list of
# the ResNet-50 stack, and ncu --set full captures of the dominant kernels.
set -x
export N=256
python bench.py > gpurun_out/r02_bench_default.json 2> gpurun_out/r02_bench_default.err
python bench.py --workload layer --no-cpu > gpurun_out/r02_bench_cfg2.json 2> gpurun_out/r02_bench_cfg2.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_stack.csv \
    python bench.py --steps 1 --warmup 0 --no-cpu --no-layers --no-graph > gpurun_out/r02_launches_stack.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_cfg2.csv \
    python bench.py --workload layer --steps 1 --warmup 0 --no-cpu > gpurun_out/r02_launches_cfg2.log 2>&1
LAYER=64,64,56,3 ncu --set full --clock-control none --import-source on -k regex:conv_upd_kernel -s 2 -c 1 -o gpurun_out/r02_ncu_l1_3x3_U python tools/one_upd.py > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:conv_fwd -s 2 -c 1 -o gpurun_out/r02_ncu_l1_3x3_F python tools/one_layer.py 64 64 56 3 f > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:conv_fwd -s 2 -c 1 -o gpurun_out/r02_ncu_l3_3x3_F python tools/one_layer.py 256 256 14 3 f > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:conv_fwd -s 2 -c 1 -o gpurun_out/r02_ncu_l3_1x1_F python tools/one_layer.py 1024 256 14 1 f > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:conv_upd_kernel -s 2 -c 1 -o gpurun_out/r02_ncu_l3_1x1_U python tools/one_layer.py 256 1024 14 1 u > /dev/null 2>&1
ITERS=3 ncu --set full --clock-control none --import-source on -k regex:conv_upd_ts_kernel -s 2 -c 1 -o gpurun_out/r02_ncu_cfg2_U python tools/prof_cfg2.py > /dev/null 2>&1
ITERS=3 ncu --set full --clock-control none --import-source on -k regex:conv_fwd -s 4 -c 2 -o gpurun_out/r02_ncu_cfg2_FB python tools/prof_cfg2.py > /dev/null 2>&1
ls -la gpurun_out
