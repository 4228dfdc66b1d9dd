cd /root/repo
for c in c4 c5; do for round in 1 2; do for v in 0 1 2 3; do
  b=$(LYNX_L2_DISCARD=$v python bench.py --config $c --steps 200 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['us_per_step'],1), {k: round(v*1e3,1) for k,v in d['kernel_ms'].items()})")
  echo "$c $round mode=$v: $b"
done; done; done
