set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
python -m pytest tests -m gpu -q -x > gpurun_out/r02a_tests.txt 2>&1; tail -3 gpurun_out/r02a_tests.txt
python bench.py --no-configs --no-next1 --no-next2 --no-next3 --no-next4 > gpurun_out/r02a_bench.json 2> gpurun_out/r02a_bench.err; tail -c 1500 gpurun_out/r02a_bench.json
NO="--no-e2e --no-cpu-baseline --no-next1 --no-next2 --no-next3 --no-next4 --no-configs"
ncu --set full --clock-control none --import-source on -k regex:clip_compact_kernel -s 3 -c 1 -f -o gpurun_out/r02a_prof python bench.py --steps 1 --warmup 3 $NO > gpurun_out/r02a_ncu.log 2>&1; echo full rc $?
ncu -i gpurun_out/r02a_prof.ncu-rep --page source --csv --print-source sass > gpurun_out/r02a_src.csv 2>/dev/null; echo src rc $?
ncu -i gpurun_out/r02a_prof.ncu-rep --page raw --csv > gpurun_out/r02a_raw.csv 2>/dev/null; echo raw rc $?
rm -f gpurun_out/r02a_prof.ncu-rep
