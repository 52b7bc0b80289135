#!/bin/bash
# Interleaved A/B timing of library variants in build/: ab_compact.sh n reps variant...
n=$1; reps=$2; shift 2
for r in $(seq $reps); do
  for v in "$@"; do
    ms=$(CLIPSEG_LIB=build/libclipseg_$v.so timeout 120 python scripts/kernel_probe.py --n $n --reps 5 --kernel compact | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('%.3f' % d['compact']['ms'])")
    echo "$v $ms"
  done
done
