set -x
timeout 600 python bench.py > gpurun_out/r01b_bench.json 2> gpurun_out/r01b_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/r01b_bench_reference.json 2> gpurun_out/r01b_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r01b_launches.csv python bench.py --steps 2 --warmup 3 --no-moe --no-cpu-baseline > gpurun_out/ncu_l.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_rb_step -c 16 -o /tmp/conv python profiles/ncu_conv_capture.py > gpurun_out/ncu_c.log 2>&1
python profiles/summarize_ncu.py /tmp/conv.ncu-rep --json gpurun_out/r01b_ncu_step.json --traffic gpurun_out/ncu_traffic.json > gpurun_out/sum.log 2>&1
ncu -i /tmp/conv.ncu-rep --page source --csv --print-source sass -k regex:k_rb_step --launch-skip 12 --launch-count 1 > /tmp/src.csv 2>/dev/null; python profiles/ncu_top_stalls.py /tmp/src.csv 25 > gpurun_out/r01b_step_stalls.txt 2>&1
timeout 600 ncu --set full --clock-control none -k regex:k_moe -c 12 -o /tmp/moe python bench.py --workload cfg4 --steps 1 --warmup 1 > gpurun_out/ncu_m.log 2>&1
python profiles/summarize_ncu.py /tmp/moe.ncu-rep --json gpurun_out/r01b_ncu_moe.json > gpurun_out/sum_m.log 2>&1
ls -la gpurun_out
