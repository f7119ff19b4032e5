DYNBATCH_TILE_M=64 timeout 300 python -m pytest tests/test_device_resblock.py -q -m gpu -x > gpurun_out/t64_tests.log 2>&1
timeout 600 python profiles/ab_time.py build_ab/lib_t64.so:DYNBATCH_TILE_M=128 build_ab/lib_t64.so:DYNBATCH_TILE_M=64 --rounds 3 --batch 64 --bp 0.1 > gpurun_out/ab_t64.txt 2>&1
timeout 600 python profiles/ab_time.py build_ab/lib_t64.so:DYNBATCH_TILE_M=128 build_ab/lib_t64.so:DYNBATCH_TILE_M=64 --rounds 2 --batch 512 --bp 0.3 >> gpurun_out/ab_t64.txt 2>&1
