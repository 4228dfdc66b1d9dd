#!/bin/bash
# Phase-1 split sweep (LYNX_KB2_PER) at one config, same box: ab_kb2.sh cfg "values"
cd "$(dirname "$0")/.."
cfg=$1; vals=$2
for round in 1 2; do for v in $vals; do
  b=$(LYNX_KB2_PER=$v python bench.py --config $cfg --steps 200 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['us_per_step'],1), {k: round(v*1e3,1) for k,v in d['kernel_ms'].items()})")
  echo "$cfg $round kb2_per=$v: $b"
done; done
