CLIPSEG_LIB=build/libclipseg_vw.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_defer.py tests/test_gpu_wide.py tests/test_gpu_canary.py -m gpu -q -x > gpurun_out/r02uu_tests.txt 2>&1; tail -2 gpurun_out/r02uu_tests.txt
timeout 900 bash scripts/ab_long.sh 3 ref vl vw
bash scripts/ab_args.sh 2 "--kernel compact --n 10000000 --family adv --reps 10" ref vl vw
bash scripts/ab_args.sh 2 "--kernel compact --n 100000000 --family mix33 --reps 10" ref vl vw
