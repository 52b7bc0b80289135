timeout 600 python -m pytest tests/test_gpu_homog.py -m gpu -q > gpurun_out/r02ll_new.txt 2>&1; tail -3 gpurun_out/r02ll_new.txt
bash scripts/ab_args.sh 2 "--kernel compact --n 100000000 --family homog --reps 10" hold hnew
bash scripts/ab_args.sh 2 "--kernel compact --n 100000000 --family homog --ndc 1 --reps 10" hold hnew
bash scripts/ab_args.sh 2 "--kernel dense --n 100000000 --family homog --reps 10" hold hnew
bash scripts/ab_args.sh 2 "--kernel dense --n 100000000 --family homog --ndc 1 --reps 10" hold hnew
CLIPSEG_LIB=build/libclipseg_hold.so ncu --set full --clock-control none --import-source on -k regex:compact -s 3 -c 1 -f -o gpurun_out/homog python scripts/kernel_probe.py --n 100000000 --family homog --reps 1 --kernel compact > gpurun_out/homog_ncu.log 2>&1; echo "ncu rc $?"
ncu -i gpurun_out/homog.ncu-rep --page source --csv --print-source sass > gpurun_out/homog_src.csv 2>/dev/null
ncu -i gpurun_out/homog.ncu-rep --page raw --csv > gpurun_out/homog_raw.csv 2>/dev/null
rm -f gpurun_out/homog.ncu-rep
