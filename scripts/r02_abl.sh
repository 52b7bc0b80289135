CLIPSEG_LIB=build/libclipseg_d3i2.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_defer.py tests/test_gpu_wide.py -m gpu -q -x > gpurun_out/r02ac_tests.txt 2>&1; tail -2 gpurun_out/r02ac_tests.txt
bash scripts/ab_args.sh 3 "--kernel compact --n 100000000 --dim 3 --reps 10" cur d3 d3i2 i2
