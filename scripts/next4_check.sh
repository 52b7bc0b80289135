set -x
python -m pytest tests/test_gpu_int.py tests/test_abi.py -q -x > gpurun_out/n4_tests.txt 2>&1; tail -15 gpurun_out/n4_tests.txt
NO="--no-e2e --no-cpu-baseline --no-next1 --no-next2 --no-next3 --no-configs"
python bench.py --steps 3 --warmup 3 $NO > gpurun_out/n4_bench.json 2> gpurun_out/n4_bench.err; python -c "import json;d=json.load(open('gpurun_out/n4_bench.json'));print(json.dumps(d['next4']))"
ncu --set full --clock-control none --import-source on -k regex:clip_int_kernel -s 3 -c 1 -f -o gpurun_out/prof_next4 python bench.py --steps 1 --warmup 3 $NO > gpurun_out/n4_ncu.log 2>&1; echo full rc $?
ncu -i gpurun_out/prof_next4.ncu-rep --page raw --csv > gpurun_out/prof_next4_raw.csv 2>&1; echo raw rc $?
