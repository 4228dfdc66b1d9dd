"""Device timeline of graphed layer steps (CUPTI via torch.profiler): per
kernel start/end relative to the step's first kernel, and the gaps.
    python scripts/timeline.py [--c4 | --c5] [--tokens T]"""
import json
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_08982_b200 as L  # noqa: E402


def main():
    if "--c4" in sys.argv:
        T, N, k, d, ff, S = 128, 64, 6, 2048, 1408, 2
        pol = L.PolicyConfig(mode="accuracy", freq_keep_budget=16)
    elif "--c5" in sys.argv:
        T, N, k, d, ff, S = 256, 8, 2, 6144, 16384, 0
        pol = L.PolicyConfig(mode="latency", drop_count=4)
    else:
        T, N, k, d, ff, S = 32, 8, 2, 4096, 14336, 0
        pol = L.PolicyConfig(mode="latency", drop_count=4)
    if "--tokens" in sys.argv:
        T = int(sys.argv[sys.argv.index("--tokens") + 1])
    n = 3 if "--c5" in sys.argv else 4
    spec = L.MoEModelSpec(n, N, k, d, ff, num_shared_experts=S)
    model = L.build_swiglu_model(spec, seed=0)
    layers = [L.LynxMoELayer(model, l, T, policy=pol) for l in range(n)]
    hid = [torch.randn((T, d), device="cuda").to(torch.bfloat16) for _ in range(n)]
    outs = [torch.empty_like(h) for h in hid]
    for l in range(n):
        layers[l](hid[l], outs[l])
    torch.cuda.synchronize()
    graphs = []
    for l in range(n):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            layers[l](hid[l], outs[l])
        graphs.append(g)
    for _ in range(3):
        for g in graphs:
            g.replay()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(3):
            for g in graphs:
                g.replay()
        torch.cuda.synchronize()
    ev = [e for e in prof.events() if e.device_type.name == "CUDA" and "lynx" in e.name]
    ev.sort(key=lambda e: e.time_range.start)
    steps, cur = [], []
    for e in ev:
        if ("router_" in e.name or "front_" in e.name) and cur:  # K0 (router_logits_kernel, router_route_kernel) or the fused front
            steps.append(cur)
            cur = []
        cur.append(e)
    steps.append(cur)
    rows = []
    for st in steps[1:-1]:
        t0 = st[0].time_range.start
        rows.append([(e.name.split("(")[0].replace("void ", "").replace("lynx::", ""),
                      e.time_range.start - t0, e.time_range.end - t0) for e in st])
    # median over steps per kernel position
    out = []
    for i in range(len(rows[0])):
        s = sorted(r[i][1] for r in rows)
        e = sorted(r[i][2] for r in rows)
        out.append({"kernel": rows[0][i][0], "start_us": s[len(s) // 2], "end_us": e[len(e) // 2]})
    nxt = [r[0] for r in steps[2:]]
    period = sorted(steps[i + 1][0].time_range.start - steps[i][0].time_range.start for i in range(len(steps) - 1))
    print(json.dumps({"T": T, "kernels": out, "step_period_us": period[len(period) // 2]}, indent=1))


if __name__ == "__main__":
    main()
