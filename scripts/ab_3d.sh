#!/bin/bash
# Interleaved A/B timing of library variants in build/ on the 3D fp32 compacting kernel (C4, 1e8):
# ab_3d.sh reps variant...   -> "variant compact_ms"
reps=$1; shift 1
for r in $(seq $reps); do
  for v in "$@"; do
    CLIPSEG_LIB=build/libclipseg_$v.so timeout 120 python scripts/kernel_probe.py --dim 3 --reps 10 --kernel compact | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', '%.3f' % d['compact']['ms'])"
  done
done
