"""K3 rate (used-expert bytes / event-timed K3) for a DeepSeek-MoE-shaped layer with and without shared
experts (diagnostic: does the shared experts' width cap the routed stream?).  python scripts/k3_rate.py"""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_08982_b200 as L  # noqa: E402


def rate(S, T=128, N=64, k=6, d=2048, ff=1408, n=6):
    spec = L.MoEModelSpec(n, N, k, d, ff, num_shared_experts=S)
    model = L.build_swiglu_model(spec, seed=0)
    pol = L.PolicyConfig(mode="accuracy", freq_keep_budget=16)
    layers = [L.LynxMoELayer(model, l, T, policy=pol) for l in range(n)]
    hid = [torch.randn((T, d), device="cuda").to(torch.bfloat16) for _ in range(n)]
    for i in range(2 * n):
        layers[i % n](hid[i % n])
    torch.cuda.synchronize()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(6)] for _ in range(60)]
    for i in range(60):
        layers[i % n].profiled(hid[i % n], evs[i])
    torch.cuda.synchronize()
    k3 = statistics.mean(evs[i][3].elapsed_time(evs[i][4]) for i in range(60))
    used = statistics.mean(layers[l].used_experts() for l in range(n))
    gb = used * 3 * d * ff * 2 / 1e9
    return used, k3 * 1e3, gb / (k3 * 1e-3)


for S in (2, 0):
    u, us, r = rate(S)
    print(f"S={S}: used {u:.1f}, K3 {us:.1f} us, {r:.0f} GB/s")
