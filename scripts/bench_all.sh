#!/bin/bash
# All bench configs in one GPU session -> gpurun_out/bench_<cfg>.json
mkdir -p gpurun_out
run() { out=$1; shift; timeout 1500 python bench.py "$@" > gpurun_out/bench_$out.json 2> gpurun_out/bench_$out.err; echo "== $out rc=$?"; }
run c2 --config c2

LYNX_FUSED_FRONT=0 timeout 1200 python bench.py --config c2 --no-cpu-baseline > gpurun_out/bench_c2-unfused.json 2> gpurun_out/bench_c2-unfused.err
run c2-nolynx --config c2-nolynx --no-cpu-baseline
run c2-acc --config c2-acc --no-cpu-baseline
run c4 --config c4
run c5 --config c5
run c5-bs32 --config c5-bs32 --no-cpu-baseline
run c3 --config c3 --steps 30 --warmup 5
run reference --impl reference --steps 5 --warmup 3
run ep4-share-c5 --gpus 4 --share-gpu --config c5 --steps 6 --warmup 3
for f in gpurun_out/bench_*.json; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); c=d.get('config',{}); r=d.get('run',{})
print('$f', round(d.get('us_per_step', d.get('ms_per_step',0)*1e3),1), 'us', round(d['value']), d['unit'], 'e2e', round(d['e2e']['value']), 'K3', round(d.get('roofline',{}).get('achieved',0)), 'frac', round(d.get('roofline',{}).get('frac',0),3), r.get('mean_used_experts'))" 2>/dev/null; done
