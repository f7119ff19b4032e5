set -x
timeout 300 python profiles/step_waits.py > gpurun_out/r02_step_waits.json 2> gpurun_out/sw.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_rb_step -c 1 -o gpurun_out/conv python profiles/ncu_conv_capture.py > gpurun_out/ncu_c.log 2>&1
python profiles/summarize_ncu.py gpurun_out/conv.ncu-rep --json gpurun_out/r02_ncu_step.json --traffic gpurun_out/ncu_traffic.json > gpurun_out/sum.log 2>&1
ncu -i gpurun_out/conv.ncu-rep --page source --csv --print-source sass -k regex:k_rb_step > gpurun_out/src.csv 2>/dev/null; python profiles/ncu_top_stalls.py gpurun_out/src.csv 30 > gpurun_out/r02_step_stalls.txt 2>&1
ncu -i gpurun_out/conv.ncu-rep --page details --csv > gpurun_out/details.csv 2>/dev/null
ls -la gpurun_out
