CLIPSEG_LIB=build/libclipseg_cw12i4.so timeout 400 python -m pytest tests/test_gpu_parity.py tests/test_gpu_canary.py tests/test_gpu_wide.py tests/test_gpu_int.py tests/test_gpu_homog.py -m gpu -q -x > gpurun_out/r02ee_tests.txt 2>&1; tail -2 gpurun_out/r02ee_tests.txt
timeout 400 bash scripts/ab_long.sh 2 base cw12 cw12i3 cw12i4
