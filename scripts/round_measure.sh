#!/bin/bash
# One GPU session of round-end evidence -> gpurun_out/: GPU tests + smoke,
# every bench line, the ncu launch lists + full captures, CUPTI timelines,
# compute-sanitizer.  Summarise afterwards (here, no GPU):
#   python scripts/summarize_round.py rNN
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/gpu_tests.log; cat gpurun_out/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; cat gpurun_out/smoke.log
bash scripts/bench_all.sh
bash scripts/ncu_round.sh
for c in c2 c4 c5; do python scripts/timeline.py --$c > gpurun_out/timeline_$c.json 2>/dev/null; done
python scripts/timeline_stack.py > gpurun_out/timeline_stack.json 2>/dev/null
SAN_TIMEOUT=900 bash scripts/sanitize.sh > gpurun_out/sanitize_summary.txt 2>&1; cat gpurun_out/sanitize_summary.txt
echo done
