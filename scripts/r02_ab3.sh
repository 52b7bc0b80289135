timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_canary.py tests/test_gpu_fullsize.py -m gpu -q -x > gpurun_out/r02e_tests.txt 2>&1; tail -3 gpurun_out/r02e_tests.txt
bash scripts/ab_compact.sh 1000000000 2 old pk2 pk1 pk2w15 > gpurun_out/r02e_ab.txt 2>&1; cat gpurun_out/r02e_ab.txt
bash scripts/prof_variant.sh pk2w15 r02e
