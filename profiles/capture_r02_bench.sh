# Round-2 bench lines only (profiles/README.md): every BASELINE config and the reference arm, one box.
set -x
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/r02_bench_reference.json 2> gpurun_out/r02_ref.err
timeout 600 python bench.py --workload cfg1 --no-moe > gpurun_out/r02_bench_cfg1.json 2> gpurun_out/cfg1.err
for d in 4 5 6 7 8; do
  timeout 600 python bench.py --workload cfg2 --depth $d --no-moe --cpu-seconds 6 > gpurun_out/r02_bench_cfg2_d$d.json 2> gpurun_out/cfg2_$d.err
done
timeout 600 python bench.py --workload cfg4 --steps 20 > gpurun_out/r02_bench_cfg4.json 2> gpurun_out/cfg4.err
timeout 900 python bench.py --workload cfg5 --steps 5 > gpurun_out/r02_bench_cfg5.json 2> gpurun_out/cfg5.err
