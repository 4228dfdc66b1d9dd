#!/bin/bash
# K1 phase timestamps (trace build) + CUPTI timelines + short benches (C2, C4).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
LYNX_LIB=paper_2411_08982_b200/_lib/liblynx_b200_trace.so python scripts/trace_select.py > gpurun_out/k1_trace_c2.json 2> gpurun_out/k1_trace_c2.err; echo "trace c2 rc=$?"
LYNX_LIB=paper_2411_08982_b200/_lib/liblynx_b200_trace.so python scripts/trace_select.py --c4 > gpurun_out/k1_trace_c4.json 2> gpurun_out/k1_trace_c4.err; echo "trace c4 rc=$?"
python scripts/timeline.py > gpurun_out/timeline_c2.json 2>/dev/null; echo "tl c2 rc=$?"
python scripts/timeline.py --c4 > gpurun_out/timeline_c4.json 2>/dev/null; echo "tl c4 rc=$?"
for cfg in c2 c4; do
  python bench.py --config $cfg --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/bench_$cfg.json 2> gpurun_out/bench_$cfg.err; echo "bench $cfg rc=$?"
done
