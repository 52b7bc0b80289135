set -x
python -m pytest tests -m gpu -q -x > gpurun_out/tl.txt 2>&1; tail -3 gpurun_out/tl.txt
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
python bench.py > gpurun_out/bench_r01l.json 2> gpurun_out/bench_r01l.err; tail -c 3000 gpurun_out/bench_r01l.json
NO="--no-e2e --no-cpu-baseline --no-next1 --no-next2 --no-next3 --no-configs"
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r01l.csv python bench.py --steps 3 --warmup 3 > gpurun_out/ncu_launch_l.log 2>&1; echo launch rc $?
ncu --set full --clock-control none --import-source on -k regex:clip_compact_kernel -s 3 -c 1 -f -o gpurun_out/prof_bench_r01l python bench.py --steps 1 --warmup 3 $NO > gpurun_out/ncu_full_l.log 2>&1; echo full rc $?
