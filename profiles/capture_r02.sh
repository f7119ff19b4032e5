# Round-2 evidence on one box: tests, every BASELINE config's bench line, the
# reference arm, the ncu launch list and full captures (profiles/README.md).
set -x
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/r02_gputest.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/r02_bench_reference.json 2> gpurun_out/r02_ref.err
timeout 600 python bench.py --workload cfg1 --no-moe > gpurun_out/r02_bench_cfg1.json 2> gpurun_out/cfg1.err
for d in 4 5 6 7 8; do
  timeout 600 python bench.py --workload cfg2 --depth $d --no-moe --cpu-seconds 6 > gpurun_out/r02_bench_cfg2_d$d.json 2> gpurun_out/cfg2_$d.err
done
timeout 600 python bench.py --workload cfg4 --steps 20 > gpurun_out/r02_bench_cfg4.json 2> gpurun_out/cfg4.err
timeout 900 python bench.py --workload cfg5 --steps 5 > gpurun_out/r02_bench_cfg5.json 2> gpurun_out/cfg5.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_launches.csv python bench.py --steps 2 --warmup 3 --no-moe --no-cpu-baseline > gpurun_out/ncu_l.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_rb_step -c 1 -o gpurun_out/conv python profiles/ncu_conv_capture.py > gpurun_out/ncu_c.log 2>&1
python profiles/summarize_ncu.py gpurun_out/conv.ncu-rep --json gpurun_out/r02_ncu_step.json --traffic gpurun_out/ncu_traffic.json > gpurun_out/sum.log 2>&1
ncu -i gpurun_out/conv.ncu-rep --page source --csv --print-source sass -k regex:k_rb_step > gpurun_out/src.csv 2>/dev/null; python profiles/ncu_top_stalls.py gpurun_out/src.csv 30 > gpurun_out/r02_step_stalls.txt 2>&1
timeout 600 ncu --set full --clock-control none -k regex:k_moe -c 12 -o gpurun_out/moe python bench.py --workload cfg4 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_m.log 2>&1
python profiles/summarize_ncu.py gpurun_out/moe.ncu-rep --json gpurun_out/r02_ncu_moe.json > gpurun_out/sum_m.log 2>&1
rm -f gpurun_out/conv.ncu-rep gpurun_out/moe.ncu-rep gpurun_out/src.csv
ls -la gpurun_out
