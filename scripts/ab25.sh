run() { label=$1; shift; env "$@" timeout 300 python bench.py --no-cpu-baseline --steps 400 $BENCH_ARGS 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('$label', round(d['us_per_step'],1), {k: round(v*1000,1) for k,v in d['kernel_ms'].items()}, round(d['roofline']['achieved']))"; }
for i in 1 2 3; do
 run rowmajor LYNX_TILED_EXPERIMENT=0
 run tiled LYNX_TILED_EXPERIMENT=1
done
BENCH_ARGS="--config c2-nolynx"
run rowmajor_nolynx LYNX_TILED_EXPERIMENT=0
run tiled_nolynx LYNX_TILED_EXPERIMENT=1
