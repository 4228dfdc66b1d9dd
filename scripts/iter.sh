#!/bin/bash
# Iteration session: selected GPU tests (-k expr in $TESTS), then bench configs ($@), then the C4 timeline.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q ${TESTS:+-k "$TESTS"} 2>&1 | tail -25
for c in "$@"; do
  timeout 600 python bench.py --config $c --steps 200 --warmup 10 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  echo "== $c rc=$?"; tail -3 gpurun_out/bench_$c.err
  python -c "
import json,sys; d=json.loads(open('gpurun_out/bench_$c.json').read().strip().splitlines()[-1])
print('$c', round(d['us_per_step'],2), 'us', d['kernel_ms'], 'frac', round(d['roofline']['frac'],3), d['clocks'])"
done
[ -n "$TIMELINE" ] && for t in $TIMELINE; do timeout 300 python scripts/timeline.py --$t 2>/dev/null | python -c "
import json,sys; d=json.load(sys.stdin); print([(k['kernel'][:24], round(k['start_us'],1), round(k['end_us'],1)) for k in d['kernels']], d['step_period_us'])"; done
exit 0
