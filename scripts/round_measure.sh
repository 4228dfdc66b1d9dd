#!/bin/bash
# One GPU session of round-end evidence -> gpurun_out/: GPU tests + smoke,
# every bench line, the ncu launch list + full captures, CUPTI timelines.
# Summarise afterwards (here, no GPU): python scripts/summarize_round.py rNN
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/gpu_tests.log; cat gpurun_out/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; cat gpurun_out/smoke.log
bash scripts/bench_all.sh
bash scripts/ncu_round.sh
python scripts/timeline.py > gpurun_out/timeline_c2.json 2>/dev/null
python scripts/timeline.py --c4 > gpurun_out/timeline_c4.json 2>/dev/null
python scripts/timeline_stack.py > gpurun_out/timeline_stack.json 2>/dev/null
echo done
