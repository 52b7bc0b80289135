timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r02aa_tests.txt 2>&1; tail -2 gpurun_out/r02aa_tests.txt
bash scripts/ab.sh "--kernel compact --n 10000000 --family adv" 2 df0 df
bash scripts/ab.sh "--kernel compact --n 10000000 --dtype f64 --family adv" 2 df0 df
bash scripts/ab.sh "--kernel compact --n 1000000000" 1 df0 df
bash scripts/ab.sh "--kernel compact --n 100000000 --family homog" 1 df0 df
bash scripts/ab.sh "--kernel compact --n 100000000 --dim 3" 1 df0 df
