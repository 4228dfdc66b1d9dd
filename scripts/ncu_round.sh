#!/bin/bash
# ncu evidence for one round: launch list of the default bench (C2) and one
# full capture of the expert GEMM (K3) -> gpurun_out/
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
echo "launches rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:ffn_kernel -s 6 -c 1 \
  -o gpurun_out/ffn_full python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
echo "full rc=$?"
timeout 900 ncu --set full --clock-control none -k regex:"route_select|router_logits|gather_kernel|combine_kernel" -s 8 -c 4 \
  -o gpurun_out/small_full python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
echo "small rc=$?"
ls -la gpurun_out/
