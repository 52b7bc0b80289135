NO="--no-e2e --no-cpu-baseline --no-next1 --no-next2 --no-next3 --no-configs"
python -m pytest tests/test_gpu_int.py -q -x 2>&1 | tail -1
for i in 1 2; do python bench.py --steps 3 --warmup 3 $NO 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print(d['next4']['ms'], d['next4']['roofline']['frac'], d['next4']['parity'])"; done
