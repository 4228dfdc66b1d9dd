#!/bin/bash
# Decode-stack tests with the clustered decode attention, then C3 A/B (LYNX_ATTN_CLUSTER=1/0) and the stack timeline.
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests/test_gpu_decode.py tests/test_gpu_shapes.py -x -q 2>&1 | tail -3
LYNX_ATTN_CLUSTER=0 timeout 900 python -m pytest tests/test_gpu_decode.py -x -q 2>&1 | tail -1
for e in 1 0; do
  LYNX_ATTN_CLUSTER=$e timeout 900 python bench.py --config c3 --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c3 cluster=$e', round(d['ms_per_step'],3), 'ms', d['clocks'], d.get('run',{}).get('sweep_ms_per_step'))"
done
LYNX_ATTN_CLUSTER=1 timeout 300 python scripts/timeline_stack.py 2>/dev/null | head -c 600
