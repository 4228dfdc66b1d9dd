#!/bin/bash
# ncu --set full captures for round 2: K1 (C2 fast path, C4 group path), K0 routing (C4),
# K3 at C4 (ffn_kernel) and C5 T=256 (ffn_pair_kernel); launch lists of C2 / C4 / C5.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:route_select_fast -s 4 -c 1 \
  -o gpurun_out/r02_k1_c2 $B --config c2 > /dev/null 2>&1; echo "k1 c2 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"route_select_group|router_route" -s 8 -c 2 \
  -o gpurun_out/r02_k01_c4 $B --config c4 > /dev/null 2>&1; echo "k01 c4 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ffn_kernel -s 4 -c 1 \
  -o gpurun_out/r02_ffn_c4 $B --config c4 > /dev/null 2>&1; echo "ffn c4 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ffn_pair_kernel -s 3 -c 1 \
  -o gpurun_out/r02_ffn_pair_c5 $B --config c5 > /dev/null 2>&1; echo "ffn pair c5 rc=$?"
for cfg in c2 c4 c5; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/r02_launches_$cfg.csv python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
  echo "launches $cfg rc=$?"
done
ls -la gpurun_out/*.ncu-rep
