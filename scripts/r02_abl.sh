CLIPSEG_LIB=build/libclipseg_hk.so timeout 900 python -m pytest tests/test_gpu_homog.py -m gpu -q -x > gpurun_out/r02qq_tests.txt 2>&1; tail -2 gpurun_out/r02qq_tests.txt
bash scripts/ab_args.sh 3 "--kernel compact --n 100000000 --family homog --reps 10" cur hk
bash scripts/ab_args.sh 2 "--kernel compact --n 100000000 --family homog --ndc 1 --reps 10" cur hk
