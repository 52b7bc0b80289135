#!/bin/bash
# Interleaved A/B timing of library variants in build/ on the NEXT-1 (homogeneous) kernels:
# ab_homog.sh reps ndc variant...   -> "variant dense_ms compact_ms" lines
reps=$1; ndc=$2; shift 2
for r in $(seq $reps); do
  for v in "$@"; do
    CLIPSEG_LIB=build/libclipseg_$v.so timeout 120 python scripts/kernel_probe.py --family homog --dtype ${DT:-f32} --ndc $ndc --reps 10 --kernel both | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', '%.3f %.3f' % (d['dense']['ms'], d['compact']['ms']))"
  done
done
