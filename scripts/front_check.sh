#!/bin/bash
cd "$(dirname "$0")/.."
timeout 1200 python -m pytest tests/test_gpu_ffn.py tests/test_gpu_decode.py tests/test_gpu_shapes.py -x -q 2>&1 | tail -3
LYNX_LIB=paper_2411_08982_b200/_lib/liblynx_b200_trace.so python scripts/trace_front.py
for c in c2 c5; do
  for f in 1 0; do
    echo "fused=$f $c: $(LYNX_FUSED_FRONT=$f python scripts/timeline.py --$c 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print([(k['kernel'][:14], round(k['end_us'],1)) for k in d['kernels']], d['step_period_us'])")"
  done
done
bash scripts/ab_env.sh c2 "LYNX_FUSED_FRONT=1" "LYNX_FUSED_FRONT=0"
for f in 1 0; do LYNX_FUSED_FRONT=$f python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c3 fused=$f', round(d['ms_per_step'],3), {k: round(v['ms_per_step'],3) for k,v in d['run']['budget_sweep'].items()})"; done
