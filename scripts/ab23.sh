run() { label=$1; shift; env "$@" timeout 300 python bench.py --no-cpu-baseline --steps 400 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('$label', round(d['us_per_step'],1), {k: round(v*1000,1) for k,v in d['kernel_ms'].items()})"; }
for i in 1 2 3; do
 run C0 LYNX_FUSED_GATHER=0 LYNX_DEBUG_FLAGS=0
 run C1 LYNX_FUSED_GATHER=0 LYNX_DEBUG_FLAGS=1
 run A LYNX_LIB=paper_2411_08982_b200/_lib/liblynx_A.so
done
