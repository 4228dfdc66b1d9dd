#!/bin/bash
# A/B library builds over several bench configs, alternating:
#   scripts/ab_configs.sh "cfg args;cfg args" libA.so libB.so [libC.so ...]
IFS=';' read -ra CFGS <<< "$1"; shift
for i in 1 2; do
  for c in "${CFGS[@]}"; do
    for lib in "$@"; do
      LYNX_LIB=$lib timeout 300 python bench.py --no-cpu-baseline --steps 200 $c 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$(basename $lib)', '$c', round(d['us_per_step'],1), round(d['kernel_ms']['ffn']*1000,1))"
    done
  done
done
