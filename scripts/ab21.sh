for i in 1 2 3; do
 for f in 0 1; do
  LYNX_FUSED_GATHER=$f timeout 300 python bench.py --no-cpu-baseline --steps 400 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('fused=$f', round(d['us_per_step'],1), {k: round(v*1000,1) for k,v in d['kernel_ms'].items()})"
 done
 LYNX_LIB=paper_2411_08982_b200/_lib/liblynx_A.so timeout 300 python bench.py --no-cpu-baseline --steps 400 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('A', round(d['us_per_step'],1), {k: round(v*1000,1) for k,v in d['kernel_ms'].items()})"
done
