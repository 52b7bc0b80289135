#!/bin/bash
# Interleaved A/B of library variants in build/:  ab.sh "<kernel_probe args>" reps variant...
args=$1; reps=$2; shift 2
for r in $(seq $reps); do
  for v in "$@"; do
    ms=$(CLIPSEG_LIB=build/libclipseg_$v.so timeout 300 python scripts/kernel_probe.py $args --reps 5 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k='compact' if 'compact' in d else 'dense'; print('%.3f %.3f' % (d[k]['ms'], d[k].get('GBps',0)))" 2>/dev/null)
    echo "$v $ms"
  done
done
