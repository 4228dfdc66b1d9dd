#!/bin/bash
cd "$(dirname "$0")/.."
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for c in c4; do
  for f in 1 0; do
    echo "fused=$f $c: $(LYNX_FUSED_FRONT=$f python scripts/timeline.py --$c 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print([(k['kernel'][:14], round(k['end_us'],1)) for k in d['kernels']], d['step_period_us'])")"
  done
done
bash scripts/ab_env.sh c4 "LYNX_FUSED_FRONT=1" "LYNX_FUSED_FRONT=0"
