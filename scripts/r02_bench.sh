set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r02z_tests.txt 2>&1; tail -3 gpurun_out/r02z_tests.txt
timeout 900 python bench.py > gpurun_out/r02z_bench.json 2> gpurun_out/r02z_bench.err; tail -5 gpurun_out/r02z_bench.err
