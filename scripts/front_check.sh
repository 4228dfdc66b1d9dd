#!/bin/bash
cd "$(dirname "$0")/.."
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
LYNX_LIB=paper_2411_08982_b200/_lib/liblynx_b200_trace.so python scripts/trace_front.py
for c in c2 c5; do
  echo "$c: $(python scripts/timeline.py --$c 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print([(k['kernel'][:14], round(k['end_us'],1)) for k in d['kernels']], d['step_period_us'])")"
done
bash scripts/ab_env.sh c2 "LYNX_FUSED_FRONT=1" "LYNX_FUSED_FRONT=0"
