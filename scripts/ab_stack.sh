cd /root/repo
timeout 900 python -m pytest tests/test_gpu_decode.py -x -q 2>&1 | tail -1
cp paper_2411_08982_b200/_lib/liblynx_b200.so paper_2411_08982_b200/_lib/ab_new.so
for r in 1 2; do for lib in ab_base ab_new; do
  LYNX_LIB=paper_2411_08982_b200/_lib/$lib.so timeout 300 python scripts/timeline_stack.py 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('$lib', d['between_ffn_us'], d['step_us'])"
done; done
