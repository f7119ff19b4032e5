DYNBATCH_CACHE=12 timeout 600 python -m pytest tests/test_device_resblock.py tests/test_device_resblock_full.py -x -q -m gpu > gpurun_out/rbtests12.log 2>&1
timeout 500 python profiles/ab_time.py build_ab/lib_new.so:DYNBATCH_CACHE=4 build_ab/lib_new.so:DYNBATCH_CACHE=12 --rounds 5 > gpurun_out/ab2.txt 2>&1
for c in 4 12; do DYNBATCH_CACHE=$c timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k_rb_step -c 1 python profiles/ncu_conv_capture.py > gpurun_out/ncu_dram_$c.txt 2>&1; done
