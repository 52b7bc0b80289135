CLIPSEG_LIB=build/libclipseg_b0t.so timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r02pp_tests.txt 2>&1; tail -2 gpurun_out/r02pp_tests.txt
bash scripts/ab_args.sh 2 "--kernel compact --n 10000000 --family adv --reps 10" b0o b0t
bash scripts/ab_args.sh 2 "--kernel compact --n 100000000 --dim 3 --reps 10" b0o b0t
timeout 600 bash scripts/ab_long.sh 3 b0o b0t
