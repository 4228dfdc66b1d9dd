#!/bin/bash
# ncu evidence for one round -> gpurun_out/: launch lists of C2 / C4 / C5 and
# --set full captures of K3 at C2 (ffn_kernel) and C5 T=256 (ffn_pair_kernel)
# plus the C2 front / combine kernels, K3 / K0 / K1 at C4
mkdir -p gpurun_out
B="python bench.py --warmup 3 --no-cpu-baseline"
for cfg in c2 c4 c5; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv \
    --log-file gpurun_out/launches_$cfg.csv $B --steps 20 --config $cfg > /dev/null 2>&1
  echo "launches $cfg rc=$?"
done
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:ffn_kernel -s 6 -c 1 \
  -o gpurun_out/ffn_full $B --steps 3 --config c2 > /dev/null 2>&1; echo "ffn c2 rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:ffn_pair_kernel -s 3 -c 1 \
  -o gpurun_out/ffn_pair_full $B --steps 3 --config c5 > /dev/null 2>&1; echo "ffn pair c5 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"front_kernel|combine_kernel" -s 8 -c 2 \
  -o gpurun_out/small_full $B --steps 3 --config c2 > /dev/null 2>&1; echo "small rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:ffn_kernel -s 6 -c 1 \
  -o gpurun_out/ffn_c4_full $B --steps 3 --config c4 > /dev/null 2>&1; echo "ffn c4 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"route_select_group|router_route" -s 12 -c 2 \
  -o gpurun_out/k01_c4_full $B --steps 3 --config c4 > /dev/null 2>&1; echo "k01 c4 rc=$?"
ls -la gpurun_out/*.ncu-rep
