bash scripts/ab_args.sh 3 "--kernel compact --n 100000000 --dim 3 --reps 10" cur t11 t12 t9 tb0
