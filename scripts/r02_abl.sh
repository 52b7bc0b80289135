CLIPSEG_LIB=build/libclipseg_vf.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_defer.py tests/test_gpu_wide.py -m gpu -q -x > gpurun_out/r02ab_tests.txt 2>&1; tail -2 gpurun_out/r02ab_tests.txt
bash scripts/ab_args.sh 2 "--kernel compact --n 10000000 --family adv --dtype f64 --reps 10" cur vf
bash scripts/ab_args.sh 2 "--kernel compact --n 50000000 --dtype f64 --reps 10" cur vf
