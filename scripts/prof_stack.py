"""Per-kernel device time of one graphed C3 decode step (4 layers of the
Mixtral shape, B=64) under ncu's launch list.  Diagnostic only:
ncu --metrics gpu__time_duration.sum --clock-control none --csv python scripts/prof_stack.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_08982_b200 as L  # noqa: E402

nl, B, d, ff = 4, 64, 4096, 14336
spec = L.MoEModelSpec(nl, 8, 2, d, ff)
model = L.build_swiglu_model(spec, seed=0)
attn = L.build_attention(nl, d, 16, seed=1)
stack = L.DecodeStack(model, attn, B, max_len=64, policy=L.PolicyConfig(mode="latency", drop_count=4))
stack.prefill(torch.randn((B, 16, d)).to(torch.bfloat16))
for _ in range(int(os.environ.get("STEPS", "3"))):
    stack.step()
torch.cuda.synchronize()
print("used", [layer.used_experts() for layer in stack._decode_layers])
