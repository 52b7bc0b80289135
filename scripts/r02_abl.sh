timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/r02r_tests.txt 2>&1; tail -3 gpurun_out/r02r_tests.txt
bash scripts/ab_compact.sh 1000000000 2 pkI gs gs15 gs17 gsnd gs15r2 > gpurun_out/r02r_ab.txt 2>&1; grep -v "^ \|Traceback\|File\|raise\|^pap\|Index\|Import\|_lib" gpurun_out/r02r_ab.txt
