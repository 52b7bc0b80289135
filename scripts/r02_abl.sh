timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r02bb_tests.txt 2>&1; tail -2 gpurun_out/r02bb_tests.txt
timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-configs --no-next1 --no-next2 --no-next3 > gpurun_out/r02bb_bench.json 2> gpurun_out/r02bb_bench.err; tail -3 gpurun_out/r02bb_bench.err
python -c "import json; d=json.loads(open('gpurun_out/r02bb_bench.json').read().strip().splitlines()[-1]); print(json.dumps(d['next4']))"
