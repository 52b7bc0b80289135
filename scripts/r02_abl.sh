CLIPSEG_LIB=build/libclipseg_nv.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_defer.py tests/test_gpu_homog.py tests/test_gpu_int.py -m gpu -q -x > gpurun_out/r02rr_tests.txt 2>&1; tail -2 gpurun_out/r02rr_tests.txt
timeout 900 bash scripts/ab_long.sh 3 cur nv pp
bash scripts/ab_args.sh 2 "--kernel compact --n 10000000 --family adv --reps 10" cur nv pp
