# round-2 final evidence run: GPU tests, smoke, bench, profiles
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/r02f_tests.txt 2>&1; tail -2 gpurun_out/r02f_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02f_smoke.txt 2>&1; echo smoke rc $?
timeout 900 python bench.py > gpurun_out/r02f_bench.json 2> gpurun_out/r02f_bench.err; echo bench rc $?
bash scripts/r02_profiles.sh > gpurun_out/r02f_profiles.log 2>&1; echo profiles rc $?
