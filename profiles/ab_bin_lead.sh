# conv1x1 lead (DYNBATCH_BIN_LEAD, SM-rows of tiles; 0 = all conv1x1 tiles first) × consumed-line discard
timeout 600 python -m pytest tests/test_device_resblock.py tests/test_device_resblock_full.py tests/test_device_resblock_errors.py -x -q -m gpu > gpurun_out/order_tests.log 2>&1
DYNBATCH_CACHE=12 timeout 300 python -m pytest tests/test_device_resblock.py -x -q -m gpu >> gpurun_out/order_tests.log 2>&1
L=build_ab/lib_order.so
timeout 900 python profiles/ab_time.py $L:DYNBATCH_BIN_LEAD=0 $L:DYNBATCH_BIN_LEAD=1 $L:DYNBATCH_BIN_LEAD=1,DYNBATCH_CACHE=12 $L:DYNBATCH_BIN_LEAD=2,DYNBATCH_CACHE=12 $L:DYNBATCH_BIN_LEAD=0,DYNBATCH_CACHE=12 --rounds 4 > gpurun_out/ab_order.txt 2>&1
for v in "0 4" "1 12"; do set -- $v; DYNBATCH_BIN_LEAD=$1 DYNBATCH_CACHE=$2 timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k_rb_step -c 1 python profiles/ncu_conv_capture.py > gpurun_out/ncu_order_$1_$2.txt 2>&1; done
