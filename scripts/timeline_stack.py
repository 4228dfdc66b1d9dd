"""Device timeline (CUPTI via torch.profiler) of one graphed C3 decode step:
per-layer kernel start/end, so the non-expert overhead per layer is visible.
    python scripts/timeline_stack.py [layers]"""
import json
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_08982_b200 as L  # noqa: E402


def main():
    nl = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    B, d, ff = 64, 4096, 14336
    spec = L.MoEModelSpec(nl, 8, 2, d, ff)
    model = L.build_swiglu_model(spec, seed=0)
    attn = L.build_attention(nl, d, 16, seed=1)
    stack = L.DecodeStack(model, attn, B, max_len=64, policy=L.PolicyConfig(mode="latency", drop_count=4))
    stack.prefill(torch.randn((B, 16, d)).to(torch.bfloat16))
    for _ in range(3):
        stack.step()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(2):
            stack.step()
        torch.cuda.synchronize()
    ev = sorted([e for e in prof.events() if e.device_type.name == "CUDA" and "lynx" in e.name],
                key=lambda e: e.time_range.start)
    # last step: from the last attn_qkv of layer 0 (after an advance_position)
    starts = [i for i, e in enumerate(ev) if "advance_position" in e.name]
    seg = ev[starts[0] + 1:starts[1] + 1]
    t0 = seg[0].time_range.start
    rows = [(e.name.split("(")[0].replace("void ", "").replace("lynx::", ""), round(e.time_range.start - t0, 1),
             round(e.time_range.end - t0, 1)) for e in seg]
    ffn = [(s, e) for n, s, e in rows if n.startswith("ffn_kernel")]
    # critical path: each kernel's end minus the previous kernel's end (second layer)
    ends = [(n, e) for n, s_, e in rows]
    per = [(ends[i][0], round(ends[i][1] - ends[i - 1][1], 1)) for i in range(1, len(ends))]
    out = {"layers": nl, "step_us": rows[-1][2], "end_to_end_increments_us": per[7:15],
           "ffn_spans": [round(e - s, 1) for s, e in ffn],
           "between_ffn_us": [round(ffn[i + 1][0] - ffn[i][1], 1) for i in range(len(ffn) - 1)]}
    print(json.dumps(out, indent=0))


if __name__ == "__main__":
    main()
