# final sanity of the committed tree: GPU tests + smoke
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/r02_final_tests.txt 2>&1; tail -1 gpurun_out/r02_final_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
