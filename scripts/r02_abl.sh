CLIPSEG_LIB=build/libclipseg_r24.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "3 or packed" > gpurun_out/r02ad_tests.txt 2>&1; tail -2 gpurun_out/r02ad_tests.txt
bash scripts/ab_args.sh 3 "--kernel compact --n 100000000 --dim 3 --reps 10" cur r24
