CLIPSEG_LIB=build/libclipseg_ns16.so timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_canary.py tests/test_gpu_defer.py -m gpu -q -x > gpurun_out/r02ah_tests.txt 2>&1; tail -1 gpurun_out/r02ah_tests.txt
timeout 900 bash scripts/ab_long.sh 2 cur ns16 ns15
