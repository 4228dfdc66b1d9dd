"""Phase timestamps of the clustered decode attention kernel (diagnostic library).
LYNX_LIB=paper_2411_08982_b200/_lib/liblynx_b200_trace.so python scripts/trace_attn.py"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_08982_b200 as L  # noqa: E402
from paper_2411_08982_b200 import _native as nat  # noqa: E402

NAMES = ["entry -> griddep_wait", "qkv (DSMEM q, cache k/v)", "cluster.sync", "row norm", "attention",
         "ctx reduce", "Wo + residual", "router (DSMEM finish)"]


def main():
    lib = nat.lib()
    lib.lynx_debug_attn_ts.argtypes = [ctypes.c_void_p]
    nl, B, d, ff = 2, 64, 4096, (64 if "--tiny-experts" in sys.argv else 14336)
    model = L.build_swiglu_model(L.MoEModelSpec(nl, 8, 2, d, ff), seed=0)
    attn = L.build_attention(nl, d, 16, seed=1)
    stack = L.DecodeStack(model, attn, B, max_len=64, policy=L.PolicyConfig(mode="latency", drop_count=4))
    stack.prefill(torch.randn((B, 16, d)).to(torch.bfloat16))
    rows, qk = [], []
    for _ in range(8):
        stack.step()
        torch.cuda.synchronize()
        buf = np.zeros(16, dtype=np.uint64)
        lib.lynx_debug_attn_ts(buf.ctypes.data)
        rows.append(np.diff(buf[:9].astype(np.int64)) / 1e3)
        qk.append(np.diff(buf[[1, 10, 11, 9, 2]].astype(np.int64)) / 1e3)
    m = np.median(np.array(rows[2:]), axis=0)
    print("qkv split (us): stage row, cluster wait, first projection, rest:",
          np.round(np.median(np.array(qk[2:]), axis=0), 2).tolist())
    for n, v in zip(NAMES, m):
        print(f"{n:28s} {v:7.2f} us")
    print(f"{'total after wait':28s} {m[1:].sum():7.2f} us")


if __name__ == "__main__":
    main()
