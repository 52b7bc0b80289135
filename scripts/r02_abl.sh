timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r02x_tests.txt 2>&1; tail -2 gpurun_out/r02x_tests.txt
bash scripts/ab.sh "--kernel compact --n 100000000 --family homog" 2 phoff ph ph11
bash scripts/ab.sh "--kernel compact --n 100000000 --family homog --ndc 1" 2 phoff ph ph11
