for mode in 0 1; do for B in 4 32; do for x0 in 0 4 12 1 2 3 37; do timeout 30 ./build/tma_probe2 $B $x0 $mode; done; done; done > gpurun_out/tma_probe2_cases.txt 2>&1
cat gpurun_out/tma_probe2_cases.txt
