CLIPSEG_LIB=build/libclipseg_cry.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_defer.py tests/test_gpu_wide.py tests/test_gpu_canary.py -m gpu -q -x > gpurun_out/r02ag_tests.txt 2>&1; tail -1 gpurun_out/r02ag_tests.txt
timeout 1200 bash scripts/ab_long.sh 2 cur cry cr0
bash scripts/ab_args.sh 2 "--kernel compact --n 10000000 --family adv --reps 10" cur cry cr0
bash scripts/ab_args.sh 2 "--kernel compact --n 100000000 --dim 3 --reps 10" cur cry cr0
