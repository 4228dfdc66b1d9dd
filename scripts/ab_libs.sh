#!/bin/bash
# A/B of library variants: ab_libs.sh "<cfg flags>" lib1.so lib2.so ...
# prints the C2-style timeline (K1 end, step period) and the bench step time per variant, interleaved twice.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
flags=$1; shift
for round in 1 2; do
  for lib in "$@"; do
    tl=$(LYNX_LIB=$lib python scripts/timeline.py $flags 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); k=d['kernels']; print(' '.join(f\"{x['kernel'][:14]}:{x['end_us']:.1f}\" for x in k), 'period', round(d['step_period_us'],1))")
    b=$(LYNX_LIB=$lib python bench.py --config ${CFG:-c2} --steps 200 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['us_per_step'],1), {k: round(v*1e3,1) for k,v in d['kernel_ms'].items()})")
    echo "$round $(basename $lib): $tl | bench $b"
  done
done
