CLIPSEG_LIB=build/libclipseg_da2.so timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_canary.py -m gpu -q -x > gpurun_out/r02ai_tests.txt 2>&1; tail -1 gpurun_out/r02ai_tests.txt
timeout 900 bash scripts/ab_long.sh 3 cur da2
