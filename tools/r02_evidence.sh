set -x
python bench.py --workload cfg5 > gpurun_out/bench_cfg5.log 2>&1
python bench.py --workload cfg5 --impl reference > gpurun_out/bench_cfg5_ref.log 2>&1
python bench.py --no-cpu --no-layers --steps 10 --sm-budget 132 > gpurun_out/bench_sm132.log 2>&1
python bench.py --no-cpu --no-layers --steps 10 > gpurun_out/bench_sm148.log 2>&1
for p in F B U; do for dt in f32 bf16; do
  python -m paper_1808_05567_b200.layer_bench --layers resnet50 --minibatch 32 --iters 5 --pass $p --dtype $dt --check --out gpurun_out/r02_layers_${p}_${dt}.json > gpurun_out/r02_layers_${p}_${dt}.txt 2>&1
done; done
