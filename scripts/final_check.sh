set -x
python -m pytest tests -m gpu -q -x > gpurun_out/final3_tests.txt 2>&1; tail -3 gpurun_out/final3_tests.txt
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
python bench.py > gpurun_out/final3_bench.json 2> gpurun_out/final3_bench.err; tail -c 1500 gpurun_out/final3_bench.json
timeout 400 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/final3_ref.json 2>&1; tail -c 800 gpurun_out/final3_ref.json
