#!/bin/bash
# One GPU session: GPU tests, then the bench configs given as arguments.
# usage: scripts/gpu_check.sh [bench-config ...]
set -o pipefail
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
for c in "$@"; do
  timeout 600 python bench.py --config $c --steps 200 --warmup 10 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  echo "== $c rc=$?"; tail -2 gpurun_out/bench_$c.err; cat gpurun_out/bench_$c.json
done
