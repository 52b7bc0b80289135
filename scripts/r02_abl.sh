CLIPSEG_LIB=build/libclipseg_pd.so timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r02yy_tests.txt 2>&1; tail -2 gpurun_out/r02yy_tests.txt
timeout 900 bash scripts/ab_long.sh 3 cur pd
bash scripts/ab_args.sh 2 "--kernel compact --n 100000000 --family homog --reps 10" cur pd
bash scripts/ab_args.sh 2 "--kernel compact --n 100000000 --dim 3 --reps 10" cur pd
bash scripts/ab_args.sh 2 "--kernel compact --n 10000000 --family adv --reps 10" cur pd
