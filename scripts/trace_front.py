"""Phase timestamps of the fused front kernel (block 0) in a layer step (diagnostic library).
LYNX_LIB=paper_2411_08982_b200/_lib/liblynx_b200_trace.so python scripts/trace_front.py [--c5]"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_08982_b200 as L  # noqa: E402
from paper_2411_08982_b200 import _native as nat  # noqa: E402

NAMES = ["griddep_wait", "A logits", "B softmax/topk", "barrier", "C policy + D remap (all tokens)", "E plan",
         "E gather + tables"]


def main():
    lib = nat.lib()
    lib.lynx_debug_select_ts.argtypes = [ctypes.c_void_p]
    T, d, ff = (256, 6144, 16384) if "--c5" in sys.argv else (32, 4096, 14336)
    N, k, S = 8, 2, 0
    cfg = L.PolicyConfig(mode="latency", drop_count=4)
    spec = L.MoEModelSpec(2, N, k, d, ff, num_shared_experts=S)
    model = L.build_swiglu_model(spec, seed=0)
    layers = [L.LynxMoELayer(model, l, T, policy=cfg) for l in range(2)]
    h = torch.randn((T, d), device="cuda").to(torch.bfloat16)
    rows = []
    for rep in range(8):
        layers[rep % 2](h)
        torch.cuda.synchronize()
        buf = np.zeros(32, dtype=np.uint64)
        lib.lynx_debug_select_ts(buf.ctypes.data)
        ts = buf[24:31].astype(np.int64)
        rows.append(np.diff(ts) / 1e3)
    m = np.median(np.array(rows[2:]), axis=0)
    if "--c4" not in sys.argv:  # per-CTA skew of the last step (entry, after the wait, at / after the barrier)
        lib.lynx_debug_front_cta_ts.argtypes = [ctypes.c_void_p]
        cb = np.zeros(1024, dtype=np.uint64)
        lib.lynx_debug_front_cta_ts(cb.ctypes.data)
        c = cb[:4 * T].reshape(T, 4).astype(np.int64)
        w0 = c[:, 1].min()
        rel = (c - w0) / 1e3
        print("per-CTA (us, vs the first wait return): entry min/max", round(rel[:, 0].min(), 2), round(rel[:, 0].max(), 2),
              "| wait return min/max", round(rel[:, 1].min(), 2), round(rel[:, 1].max(), 2),
              "| barrier arrival min/median/max", round(rel[:, 2].min(), 2), round(float(np.median(rel[:, 2])), 2),
              round(rel[:, 2].max(), 2), "| barrier exit min/max", round(rel[:, 3].min(), 2), round(rel[:, 3].max(), 2))
    for n, v in zip(NAMES[1:], m):
        print(f"{n:22s} {v:7.2f} us")
    print(f"{'total after wait':22s} {m.sum():7.2f} us")


if __name__ == "__main__":
    main()
