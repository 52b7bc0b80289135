timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/r02m_tests.txt 2>&1; tail -3 gpurun_out/r02m_tests.txt
bash scripts/ab_compact.sh 1000000000 2 pkH pkI > gpurun_out/r02m_ab.txt 2>&1; cat gpurun_out/r02m_ab.txt

