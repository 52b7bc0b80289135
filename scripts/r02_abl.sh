timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r02cc_tests.txt 2>&1; tail -2 gpurun_out/r02cc_tests.txt
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
