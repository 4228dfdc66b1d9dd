#!/bin/bash
# A/B an environment switch over bench configs: scripts/ab_env.sh VAR "v1 v2" "cfg args;cfg args"
VAR=$1; VALS=$2; IFS=';' read -ra CFGS <<< "$3"
for i in 1 2; do
  for c in "${CFGS[@]}"; do
    for v in $VALS; do
      env $VAR=$v timeout 300 python bench.py --no-cpu-baseline --steps 200 $c 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$VAR=$v', '$c', round(d['us_per_step'],1), round(d['kernel_ms']['ffn']*1000,1), round(d['roofline']['achieved']))"
    done
  done
done
