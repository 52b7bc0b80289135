set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/r02b_tests.txt 2>&1; tail -15 gpurun_out/r02b_tests.txt
bash scripts/ab_compact.sh 1000000000 3 old pk > gpurun_out/r02b_ab.txt 2>&1; cat gpurun_out/r02b_ab.txt
