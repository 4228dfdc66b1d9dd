"""Timeline of one FFN launch from the diagnostic library (LYNX_TRACE).
Run:  LYNX_LIB=paper_2411_08982_b200/_lib/liblynx_b200_trace.so python scripts/trace_ffn.py"""
import ctypes
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_08982_b200 as L  # noqa: E402
from paper_2411_08982_b200 import _native as nat  # noqa: E402

ROLES = {1: "dep_wait", 2: "epilogue_unit", 4: "mma_unit", 5: "cta"}


def stats(x):
    x = np.asarray(x, dtype=np.float64)
    if x.size == 0:
        return None
    return {"n": int(x.size), "mean": round(float(x.mean()), 2), "p50": round(float(np.median(x)), 2),
            "max": round(float(x.max()), 2), "min": round(float(x.min()), 2)}


def main():
    lib = nat.lib()
    lib.lynx_debug_trace.restype = ctypes.c_int
    lib.lynx_debug_trace.argtypes = [ctypes.c_void_p, ctypes.c_int]
    if "--c4" in sys.argv:
        T, N, k, d, ff, S = 128, 64, 6, 2048, 1408, 2
        pol = L.PolicyConfig(mode="accuracy", freq_keep_budget=16)
    elif "--c5" in sys.argv:  # CTA-pair kernel: role-4 records are unit drains (epilogue end), per CTA
        T, N, k, d, ff, S = 256, 8, 2, 6144, 16384, 0
        pol = L.PolicyConfig(mode="latency", drop_count=4)
    else:
        T, N, k, d, ff, S = 32, 8, 2, 4096, 14336, 0
        pol = L.PolicyConfig(mode="latency", drop_count=4)
    spec = L.MoEModelSpec(1, N, k, d, ff, num_shared_experts=S)
    model = L.build_swiglu_model(spec, seed=0)
    layer = L.LynxMoELayer(model, 0, T, policy=pol)
    h = torch.randn((T, d), device="cuda").to(torch.bfloat16)
    for _ in range(3):
        layer(h)
    torch.cuda.synchronize()
    buf = np.zeros((65536, 4), dtype=np.uint64)
    lib.lynx_debug_trace(buf.ctypes.data, 65536)
    layer(h)
    torch.cuda.synchronize()
    n = lib.lynx_debug_trace(buf.ctypes.data, 65536)
    rec = buf[:n]
    cta = (rec[:, 0] >> 32).astype(np.int64)
    role = (rec[:, 0] & 0xFFFFFFFF).astype(np.int64)
    uid = rec[:, 1].astype(np.int64)
    t0 = rec[:, 2].astype(np.int64)
    t1 = rec[:, 3].astype(np.int64)
    base = t0.min()
    used = layer.used_experts()
    nrows = int(((torch.bincount(layer.assigned.flatten().long(), minlength=N) + 15) // 16 * 16).sum().item())
    # unit classes (queue order: phase-0 units, then phase-1 units)
    tiles1 = 2 * ((ff + 63) // 64) * 64 // 128
    ngather = 0
    nA = used * (tiles1 // 4 if "--c5" in sys.argv else tiles1)  # pair kernel, MT=2: 4 tiles per unit
    out = {"records": int(n), "kernel_span_us": float((t1.max() - base) / 1e3), "nA": nA}
    m = role == 4
    dur = (t1[m] - t0[m]) / 1e3
    u = uid[m]
    out["mma_phase0"] = stats(dur[(u >= ngather) & (u < ngather + nA)])
    out["mma_phase1"] = stats(dur[u >= ngather + nA])
    out["mma_first_start"] = float((t0[m].min() - base) / 1e3)
    out["mma_last_end"] = float((t1[m].max() - base) / 1e3)
    # per-CTA MMA busy time and gaps
    busy, gaps, first, last = [], [], [], []
    for c in np.unique(cta[m]):
        mm = m & (cta == c)
        s, e = np.sort(t0[mm]), np.sort(t1[mm])
        busy.append((e - s).sum() / 1e3)
        first.append((s[0] - base) / 1e3)
        last.append((e[-1] - base) / 1e3)
        gaps.append(((s[1:] - e[:-1]).clip(min=0)).sum() / 1e3)
    out["cta_mma_busy"] = stats(busy)
    out["cta_mma_gaps"] = stats(gaps)
    out["cta_mma_first"] = stats(first)
    out["cta_mma_last"] = stats(last)
    mw = role == 1
    out["dep_wait"] = stats((t1[mw] - t0[mw]) / 1e3)
    me = role == 2
    out["epilogue"] = stats((t1[me] - t0[me]) / 1e3)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
