"""Device time per kernel: R calls captured in one CUDA graph, replayed.
Diagnostic only (no host-submission gaps in the measurement)."""
import ctypes
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_08982_b200 as L  # noqa: E402
from paper_2411_08982_b200 import _native as nat  # noqa: E402

R = 50


def graph_time(fn, reps=R):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            fn()
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(3):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) * 1000 / (3 * reps)


def main():
    T, N, k, d, ff = 32, 8, 2, 4096, 14336
    lib = nat.lib()
    ref = lambda s: ctypes.cast(ctypes.pointer(s), ctypes.c_void_p)  # noqa: E731
    st = lambda: torch.cuda.current_stream().cuda_stream  # noqa: E731
    z = torch.randn((T, N), dtype=torch.float64, device="cuda") * 2
    o = {n: torch.zeros(s, dtype=dt, device="cuda") for n, s, dt in [
        ("ids", (T, k), torch.int32), ("probs", (T, k), torch.float64), ("full", (T, N), torch.float64),
        ("conf", (T,), torch.float64), ("asg", (T, k), torch.int32), ("w", (T, k), torch.float64),
        ("flags", (1,), torch.int32)]}
    sel = nat.LynxSelection(expert_ids=o["ids"].data_ptr(), probs=o["probs"].data_ptr(),
                            full_probs=o["full"].data_ptr(), conf=o["conf"].data_ptr(),
                            assigned=o["asg"].data_ptr(), weights=o["w"].data_ptr(), flags=o["flags"].data_ptr())
    pol = L.PolicyConfig(mode="latency", drop_count=4).to_native()
    h = torch.randn((T, d), device="cuda").to(torch.bfloat16)
    wr = torch.randn((N, d), device="cuda").to(torch.bfloat16)
    lg = torch.empty((T, N), dtype=torch.float64, device="cuda")
    res = {}
    res["route_select_us"] = graph_time(
        lambda: lib.lynx_route_select(z.data_ptr(), T, N, k, 1, ref(pol), ref(sel), st()))
    res["route_select_nopolicy_us"] = graph_time(
        lambda: lib.lynx_route_select(z.data_ptr(), T, N, k, 1, None, ref(sel), st()))
    res["router_us"] = graph_time(
        lambda: lib.lynx_router_logits(h.data_ptr(), wr.data_ptr(), T, d, N, lg.data_ptr(), st()))
    spec = L.MoEModelSpec(1, N, k, d, ff)
    model = L.build_swiglu_model(spec, seed=0)
    cfg = L.PolicyConfig(mode="latency", drop_count=4)
    layer = L.LynxMoELayer(model, 0, T, policy=cfg)
    out = torch.empty_like(h)
    layer(h, out)
    mask = layer.mask()
    res["used"] = layer.used_experts()
    res["layer_us"] = graph_time(lambda: layer(h, out), reps=10)
    res["forward_us"] = graph_time(lambda: L.forward_layer(h, model, 0, mask), reps=10)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
