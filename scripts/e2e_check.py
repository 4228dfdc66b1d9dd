"""stream_host end-to-end timing at C2 (diagnostic): device-resident graph replay vs the copy-overlapped host API.
    [LYNX_LIB=...] python scripts/e2e_check.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_08982_b200 as L  # noqa: E402


def main():
    T, d, ff, N, k = 32, 4096, 14336, 8, 2
    spec = L.MoEModelSpec(num_layers=1, num_experts=N, top_k=k, d_model=d, d_ff=ff)
    model = L.build_swiglu_model(spec, seed=0)
    layer = L.LynxMoELayer(model, 0, T, policy=L.PolicyConfig(mode="latency", drop_count=4))
    h = torch.randn((T, d), device="cuda").to(torch.bfloat16)
    out = torch.empty_like(h)
    for _ in range(5):
        layer(h, out)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        layer(h, out)
    steps = 200
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    g.replay()
    torch.cuda.synchronize()
    a.record()
    for _ in range(steps):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    dev = a.elapsed_time(b) / steps
    hh = [h.cpu().pin_memory() for _ in range(steps)]
    oh = [torch.empty_like(hh[0]).pin_memory() for _ in range(steps)]
    layer.stream_host(hh[:4], oh[:4])
    torch.cuda.synchronize()
    a.record()
    layer.stream_host(hh, oh)
    b.record()
    torch.cuda.synchronize()
    e2e = a.elapsed_time(b) / steps
    print(f"device graph {dev * 1e3:.1f} us/step (one weight copy: L2-warm-ish), stream_host e2e {e2e * 1e3:.1f} us/step")


if __name__ == "__main__":
    main()
