#!/bin/bash
# Interleaved A/B of library variants on one kernel_probe configuration:
#   ab_args.sh reps "<kernel_probe args>" variant...
reps=$1; args=$2; shift 2
for r in $(seq $reps); do
  for v in "$@"; do
    ms=$(CLIPSEG_LIB=build/libclipseg_$v.so timeout 120 python ${PROBE:-scripts/kernel_probe.py} $args | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=[x for x in d if isinstance(d[x], dict)][0]; print('%.4f' % d[k]['ms'])")
    echo "[$args] $v $ms"
  done
done
