#!/bin/bash
# build_ab.sh <name> <extra nvcc flags...> : variant liblynx into paper_2411_08982_b200/_lib/ab_<name>.so
set -e
name=$1; shift
cd /root/repo
B=/tmp/ab/$name; mkdir -p $B
for f in select dispatch ffn attention ep_p2p capi; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 --expt-relaxed-constexpr -diag-suppress 550 "$@" -I include -c paper_2411_08982_b200/csrc/$f.cu -o $B/$f.o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC -o paper_2411_08982_b200/_lib/ab_$name.so $B/*.o -cudart static
echo built ab_$name.so
