#!/bin/bash
# One GPU session: full GPU suite, smoke, racecheck, short benches of the default and C5 configs.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -rs -s > gpurun_out/gpu_all.log 2>&1; echo "gpu tests rc=$?"; tail -3 gpurun_out/gpu_all.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
SAN_CASES="fast group pair apply forward ep stack" SAN_TIMEOUT=600 bash scripts/sanitize.sh 2>&1
for cfg in c2 c5; do
  python bench.py --config $cfg --steps 60 --warmup 5 > gpurun_out/bench_$cfg.json 2> gpurun_out/bench_$cfg.err; echo "bench $cfg rc=$?"
done
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err; echo "ref rc=$?"
