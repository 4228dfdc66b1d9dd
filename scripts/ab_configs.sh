#!/bin/bash
# A/B two library builds over several bench configs: scripts/ab_configs.sh libA libB "cfg args;cfg args"
A=$1; B=$2; IFS=';' read -ra CFGS <<< "$3"
for i in 1 2; do
  for c in "${CFGS[@]}"; do
    for v in A B; do
      lib=$([ $v = A ] && echo $A || echo $B)
      LYNX_LIB=$lib timeout 300 python bench.py --no-cpu-baseline --steps 200 $c 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v', '$c', round(d['us_per_step'],1), round(d['kernel_ms']['ffn']*1000,1))"
    done
  done
done
