timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r02w_tests.txt 2>&1; tail -2 gpurun_out/r02w_tests.txt
bash scripts/ab.sh "--kernel compact --n 100000000 --dim 3" 2 p3off p3a p3b p3c
