#!/bin/bash
# A/B of env settings on one config: ab_env.sh <config> "<ENV=..>" "<ENV=..>" ...  (bench K3 + step time, twice)
cd "$(dirname "$0")/.."
cfg=$1; shift
for round in 1 2; do
  for e in "$@"; do
    b=$(env $e python bench.py --config $cfg --steps 100 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['us_per_step'],1), 'frac', round(d['roofline']['frac'],3), {k: round(v*1e3,1) for k,v in d['kernel_ms'].items()})")
    echo "$round [$e]: $b"
  done
done
