#!/bin/bash
# A/B two library builds in one GPU session: alternate bench runs.
# usage: scripts/ab_bench.sh libA.so libB.so [rounds] [extra bench args]
A=$1; B=$2; R=${3:-3}; shift 3; EXTRA="$@"
for i in $(seq 1 $R); do
  for v in A B; do
    lib=$([ $v = A ] && echo $A || echo $B)
    LYNX_LIB=$lib timeout 300 python bench.py --no-cpu-baseline --steps 400 $EXTRA 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('$v', round(d['us_per_step'],1), {k: round(v*1000,1) for k,v in d['kernel_ms'].items()})"
  done
done
