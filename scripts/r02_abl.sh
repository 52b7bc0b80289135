# scratch A/B command list run through gpurun during round 2 (the last one is kept); see
# profiles/r02_summary.md for the measurements
timeout 1200 bash scripts/ab_long.sh 2 cur sp1 sp4 bo64
