# Bench lines for every BASELINE IEP / MoE config on one GPU (profiles/r01_bench_<cfg>.json).
set -x
timeout 600 python bench.py --workload cfg1 --no-moe > gpurun_out/r01_bench_cfg1.json 2> gpurun_out/cfg1.err
for d in 4 5 6 7 8; do
  timeout 600 python bench.py --workload cfg2 --depth $d --no-moe > gpurun_out/r01_bench_cfg2_d$d.json 2> gpurun_out/cfg2_$d.err
done
timeout 600 python bench.py --workload cfg4 --steps 20 > gpurun_out/r01_bench_cfg4.json 2> gpurun_out/cfg4.err
timeout 600 python bench.py --workload cfg5 --steps 5 > gpurun_out/r01_bench_cfg5_ep1.json 2> gpurun_out/cfg5.err
