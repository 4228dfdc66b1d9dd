#!/bin/bash
# A/B of an env switch on one box: ab_env.sh VAR "cfgs" -> bench + timeline for VAR=1 / VAR=0, twice
cd "$(dirname "$0")/.."
var=$1; cfgs=$2
for c in $cfgs; do
  for round in 1 2; do
    for v in 1 0; do
      tl=$(env $var=$v python scripts/timeline.py --$c 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); k=d['kernels']; print(' '.join(f\"{x['kernel'][:14]}:{x['end_us']:.1f}\" for x in k), 'period', round(d['step_period_us'],1))")
      b=$(env $var=$v python bench.py --config $c --steps 200 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['us_per_step'],1), {k: round(v*1e3,1) for k,v in d['kernel_ms'].items()})")
      echo "$c $round $var=$v: $tl | bench $b"
    done
  done
done
