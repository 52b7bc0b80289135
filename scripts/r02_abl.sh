timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r02oo_tests.txt 2>&1; tail -2 gpurun_out/r02oo_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02oo_smoke.txt 2>&1; echo smoke rc $?
timeout 900 python bench.py > gpurun_out/r02oo_bench.json 2> gpurun_out/r02oo_bench.err; echo bench rc $?; tail -c 400 gpurun_out/r02oo_bench.json
