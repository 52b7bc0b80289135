# prof_variant.sh <variant> <tag> [n] : ncu --set full of the compacting kernel of build/libclipseg_<variant>.so
v=$1; tag=$2; n=${3:-1000000000}
CLIPSEG_LIB=build/libclipseg_$v.so ncu --set full --clock-control none --import-source on -k regex:compact -s 3 -c 1 -f -o gpurun_out/${tag} python scripts/kernel_probe.py --n $n --reps 1 --kernel compact > gpurun_out/${tag}_ncu.log 2>&1; echo "ncu rc $?"
ncu -i gpurun_out/${tag}.ncu-rep --page source --csv --print-source sass > gpurun_out/${tag}_src.csv 2>/dev/null
ncu -i gpurun_out/${tag}.ncu-rep --page raw --csv > gpurun_out/${tag}_raw.csv 2>/dev/null
rm -f gpurun_out/${tag}.ncu-rep
