# Round-2 final evidence on one B200, at the benchmarked commit: ncu launch lists and
# --set full captures first, summarised ON THE BOX into profiles/ (the .ncu-rep files are
# too large to bring back), then the bench lines (which read the fresh DRAM-traffic table),
# the per-layer reports and the stack profile. Outputs under gpurun_out/final/.
set -x
O=gpurun_out/final
mkdir -p $O
export N=256
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_stack.csv \
    python bench.py --steps 1 --warmup 0 --no-cpu --no-layers --no-graph > $O/launches_stack.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_cfg2.csv \
    python bench.py --workload layer --steps 1 --warmup 0 --no-cpu > $O/launches_cfg2.log 2>&1
NCU="ncu --set full --clock-control none --import-source on"
$NCU -k regex:conv_fwd -s 2 -c 1 -o gpurun_out/r02_ncu_l1_1x1_res_F python tools/one_fused_fwd.py 64 256 56 > /dev/null 2>&1
LAYER=64,64,56,3 $NCU -k regex:conv_upd_kernel -s 2 -c 1 -o gpurun_out/r02_ncu_l1_3x3_U python tools/one_upd.py > /dev/null 2>&1
$NCU -k regex:conv_fwd -s 2 -c 1 -o gpurun_out/r02_ncu_l1_3x3_F python tools/one_layer.py 64 64 56 3 f > /dev/null 2>&1
$NCU -k regex:conv_fwd -s 2 -c 1 -o gpurun_out/r02_ncu_l3_3x3_F python tools/one_layer.py 256 256 14 3 f > /dev/null 2>&1
$NCU -k regex:conv_fwd -s 2 -c 1 -o gpurun_out/r02_ncu_l3_1x1_F python tools/one_layer.py 1024 256 14 1 f > /dev/null 2>&1
$NCU -k regex:conv_upd_kernel -s 2 -c 1 -o gpurun_out/r02_ncu_l3_1x1_U python tools/one_layer.py 256 1024 14 1 u > /dev/null 2>&1
LAYER=512,512,7,3 $NCU -k regex:conv_upd_kernel -s 2 -c 1 -o gpurun_out/r02_ncu_l4_3x3_U python tools/one_upd.py > /dev/null 2>&1
$NCU -k regex:conv_fwd -s 2 -c 1 -o gpurun_out/r02_ncu_l4_3x3_F python tools/one_layer.py 512 512 7 3 f > /dev/null 2>&1
$NCU -k regex:conv_fwd -s 2 -c 1 -o gpurun_out/r02_ncu_l4_1x1_F python tools/one_layer.py 2048 512 7 1 f > /dev/null 2>&1
ITERS=3 $NCU -k regex:conv_upd_ts_kernel -s 2 -c 1 -o gpurun_out/r02_ncu_cfg2_U python tools/prof_cfg2.py > /dev/null 2>&1
ITERS=3 $NCU -k regex:conv_fwd -s 4 -c 2 -o gpurun_out/r02_ncu_cfg2_FB python tools/prof_cfg2.py > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep
python tools/r02_summarise.py gpurun_out > $O/summarise.log 2>&1
cp profiles/r02_ncu_full.json profiles/r02_ncu_traffic.json profiles/r02_launches_stack.csv profiles/r02_launches_cfg2.csv $O/
rm -f gpurun_out/*.ncu-rep
python bench.py > $O/bench_default.json 2> $O/bench_default.err
python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err
python bench.py --workload layer --no-cpu > $O/bench_cfg2.json 2> $O/bench_cfg2.err
python bench.py --workload cfg5 > $O/bench_cfg5.json 2> $O/bench_cfg5.err
python bench.py --workload cfg5 --impl reference > $O/bench_cfg5_reference.json 2> $O/bench_cfg5_reference.err
python bench.py --no-cpu --no-layers --steps 10 --sm-budget 132 > $O/bench_sm132.json 2>&1
N=256 python tools/stack_profile.py > $O/stack_layers_n256.txt 2>&1
N=32 python tools/stack_profile.py > $O/stack_layers_n32.txt 2>&1
for p in F B U; do for dt in f32 bf16; do
  python -m paper_1808_05567_b200.layer_bench --layers resnet50 --minibatch 32 --iters 5 --pass $p --dtype $dt --check --out $O/r02_layers_${p}_${dt}.json > $O/r02_layers_${p}_${dt}.txt 2>&1
done; done
ls -la $O
