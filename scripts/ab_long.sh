#!/bin/bash
# Sustained A/B (power cap relevant): ab_long.sh reps variant... ; 1e9 headline, 60 launches each
reps=$1; shift
for r in $(seq $reps); do
  for v in "$@"; do
    ms=$(CLIPSEG_LIB=build/libclipseg_$v.so timeout 300 python scripts/kernel_probe.py --kernel compact --n 1000000000 --reps 60 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('%.3f best %.3f' % (d['compact']['ms'], d['compact']['best_ms']))")
    echo "$v $ms"
  done
done
