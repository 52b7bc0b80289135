CLIPSEG_LIB=build/libclipseg_it2.so timeout 600 python -m pytest tests/test_gpu_int.py -m gpu -q -x > gpurun_out/r02af_tests.txt 2>&1; tail -1 gpurun_out/r02af_tests.txt
PROBE=scripts/int_probe.py bash scripts/ab_args.sh 3 "--reps 20" it0 it2
