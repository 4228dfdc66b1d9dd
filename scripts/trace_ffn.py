"""Timeline of one FFN launch from the diagnostic library (LYNX_TRACE).
Run:  LYNX_LIB=paper_2411_08982_b200/_lib/liblynx_b200_trace.so python scripts/trace_ffn.py"""
import collections
import ctypes
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_08982_b200 as L  # noqa: E402
from paper_2411_08982_b200 import _native as nat  # noqa: E402

ROLES = {1: "h_wait", 2: "epilogue_unit", 3: "reduce_task", 4: "mma_unit", 5: "cta", 6: "reduce+combine_task"}


def main():
    lib = nat.lib()
    lib.lynx_debug_trace.restype = ctypes.c_int
    lib.lynx_debug_trace.argtypes = [ctypes.c_void_p, ctypes.c_int]
    T, N, k, d, ff = 32, 8, 2, 4096, 14336
    spec = L.MoEModelSpec(1, N, k, d, ff)
    model = L.build_swiglu_model(spec, seed=0)
    layer = L.LynxMoELayer(model, 0, T, policy=L.PolicyConfig(mode="latency", drop_count=4))
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
    t0 = rec[:, 2].astype(np.int64)
    t1 = rec[:, 3].astype(np.int64)
    base = t0.min()
    out = {"records": int(n), "kernel_span_us": float((t1.max() - base) / 1e3)}
    for r, name in ROLES.items():
        m = role == r
        if not m.any():
            continue
        dur = (t1[m] - t0[m]) / 1e3
        out[name] = {"n": int(m.sum()), "mean_us": float(dur.mean()), "max_us": float(dur.max()),
                     "p50_us": float(np.median(dur)), "last_end_us": float((t1[m].max() - base) / 1e3),
                     "first_start_us": float((t0[m].min() - base) / 1e3)}
    ends = collections.defaultdict(int)
    m = role == 5
    out["cta_end_us_sorted_tail"] = sorted(((t1[m] - base) / 1e3).tolist())[-10:]
    out["cta_start_us_sorted_tail"] = sorted(((t0[m] - base) / 1e3).tolist())[-5:]
    # slowest reduce/combine tasks
    m = (role == 3) | (role == 6)
    idx = np.argsort(-(t1[m] - t0[m]))[:8]
    out["slowest_tasks"] = [{"cta": int(cta[m][i]), "role": int(role[m][i]), "task": int(rec[m][i, 1]),
                             "start_us": float((t0[m][i] - base) / 1e3), "dur_us": float((t1[m][i] - t0[m][i]) / 1e3)}
                            for i in idx]
    m = role == 2
    e_end = (t1[m] - base) / 1e3
    out["epilogue_end_p99_us"] = float(np.percentile(e_end, 99))
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
