timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r02jj_tests.txt 2>&1; tail -3 gpurun_out/r02jj_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02jj_smoke.txt 2>&1; echo smoke rc $?; tail -3 gpurun_out/r02jj_smoke.txt
