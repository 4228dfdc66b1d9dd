"""Micro-benchmark of the small kernels: warm (back-to-back) vs cold (after
an L2-evicting sweep), device-timed with CUDA events.  Diagnostic only."""
import ctypes
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2411_08982_b200 as L  # noqa: E402
from paper_2411_08982_b200 import _native as nat  # noqa: E402


def timeit(fn, reps, cold):
    big = torch.empty(2 << 30, dtype=torch.uint8, device="cuda") if cold else None
    ts = []
    for _ in range(reps):
        if cold:
            big.zero_()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1000)
    return float(np.median(ts))


def main():
    T, N, k, d = 32, 8, 2, 4096
    lib = nat.lib()
    z = torch.randn((T, N), dtype=torch.float64, device="cuda") * 2
    out = {n: torch.zeros(s, dtype=dt, device="cuda") for n, s, dt in [
        ("ids", (T, k), torch.int32), ("probs", (T, k), torch.float64), ("full", (T, N), torch.float64),
        ("conf", (T,), torch.float64), ("asg", (T, k), torch.int32), ("w", (T, k), torch.float64),
        ("flags", (1,), torch.int32)]}
    sel = nat.LynxSelection(expert_ids=out["ids"].data_ptr(), probs=out["probs"].data_ptr(),
                            full_probs=out["full"].data_ptr(), conf=out["conf"].data_ptr(),
                            assigned=out["asg"].data_ptr(), weights=out["w"].data_ptr(), flags=out["flags"].data_ptr())
    pol = L.PolicyConfig(mode="latency", drop_count=4).to_native()
    ref = lambda s: ctypes.cast(ctypes.pointer(s), ctypes.c_void_p)  # noqa: E731
    stream = lambda: torch.cuda.current_stream().cuda_stream  # noqa: E731
    sel_fn = lambda: lib.lynx_route_select(z.data_ptr(), T, N, k, 1, ref(pol), ref(sel), stream())  # noqa: E731
    h = torch.randn((T, d), device="cuda").to(torch.bfloat16)
    wr = torch.randn((N, d), device="cuda").to(torch.bfloat16)
    lg = torch.empty((T, N), dtype=torch.float64, device="cuda")
    rt_fn = lambda: lib.lynx_router_logits(h.data_ptr(), wr.data_ptr(), T, d, N, lg.data_ptr(), stream())  # noqa
    res = {}
    for name, fn in [("route_select", sel_fn), ("router", rt_fn)]:
        fn()
        res[name + "_warm_us"] = timeit(fn, 50, False)
        res[name + "_cold_us"] = timeit(fn, 20, True)
    empty = lambda: None  # noqa: E731
    res["empty_us"] = timeit(empty, 50, False)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
