CLIPSEG_LIB=build/libclipseg_fl.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_defer.py tests/test_gpu_canary.py tests/test_gpu_int.py tests/test_gpu_homog.py -m gpu -q -x > gpurun_out/r02ww_tests.txt 2>&1; tail -2 gpurun_out/r02ww_tests.txt
timeout 900 bash scripts/ab_long.sh 3 cur fl
bash scripts/ab_args.sh 2 "--kernel compact --n 100000000 --family homog --reps 10" cur fl
bash scripts/ab_args.sh 2 "--kernel compact --n 100000000 --dim 3 --reps 10" cur fl
