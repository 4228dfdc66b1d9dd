"""Phase timestamps of K1 inside a real layer step (diagnostic library).
LYNX_LIB=paper_2411_08982_b200/_lib/liblynx_b200_trace.so python scripts/trace_select.py"""
import ctypes
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_08982_b200 as L  # noqa: E402
from paper_2411_08982_b200 import _native as nat  # noqa: E402

PHASES = ["start->griddep_wait", "wait", "route(softmax/topk/conf)", "policy", "remap", "outputs", "plan"]


def main():
    lib = nat.lib()
    lib.lynx_debug_select_ts.argtypes = [ctypes.c_void_p]
    if "--c4" in sys.argv:  # DeepSeek-MoE-16B shape, accuracy policy
        T, N, k, d, ff, S = 128, 64, 6, 2048, (64 if "--tiny-experts" in sys.argv else 1408), 2
        cfg = L.PolicyConfig(mode="accuracy", freq_keep_budget=16)
    else:
        T, N, k, d, ff, S = 32, 8, 2, 4096, 14336, 0
        cfg = L.PolicyConfig(mode="latency", drop_count=4)
    spec = L.MoEModelSpec(2, N, k, d, ff, num_shared_experts=S)
    model = L.build_swiglu_model(spec, seed=0)
    layers = [L.LynxMoELayer(model, l, T, policy=cfg) for l in range(2)]
    h = torch.randn((T, d), device="cuda").to(torch.bfloat16)
    res = {}
    for label, warm in (("cold_after_stream", False), ("warm_repeat", True)):
        rows = []
        for rep in range(5):
            if "--touch" in sys.argv and not warm:
                # read the layer's workspace and selection buffers first (L2 and TLB warm for
                # K1's data; its code stays cold): separates data from instruction-fetch cost
                lay = layers[rep % 2]
                for b in (lay.workspace, lay.expert_ids, lay.probs, lay.full_probs, lay.conf, lay.counts,
                          lay.retained_mask, lay.assigned, lay.weights, lay.important):
                    b.view(torch.uint8).sum()
            layers[rep % 2](h)  # streams weights -> evicts L2
            torch.cuda.synchronize()
            if warm:
                # run the select path alone twice: second run warm
                lg = L.router_logits(model, 0, h)
                for _ in range(2):
                    sel = L.route_batch(L.RoutingLogits(0, L.Phase.DECODE, lg), k, check=False)
                    torch.cuda.synchronize()
            buf = np.zeros(32, dtype=np.uint64)
            lib.lynx_debug_select_ts(buf.ctypes.data)
            ts = buf[:7].astype(np.int64)
            rows.append(np.diff(ts) / 1e3)
            if buf[16]:  # policy sub-phases (thread 0): important, ranking, votes, retention order, keep
                sub = buf[[2, 16, 17, 18, 19, 3]].astype(np.int64)
                print(label, "policy sub-phases (us): important, sample-rank, votes, order, keep:",
                      np.round(np.diff(sub) / 1e3, 2).tolist(), file=sys.stderr)
            if buf[20]:  # group remap sub-phases (thread 0)
                sub = buf[[3, 20, 21, 24, 25, 22, 23, 4]].astype(np.int64)
                print(label, "remap sub-phases (us): start, slot loads, occupancy, round count, arg-max rounds, "
                      "pre-sum, sum+write:",
                      np.round(np.diff(sub) / 1e3, 2).tolist(), file=sys.stderr)
            if "--c4" in sys.argv and not warm and buf[12]:  # K0 (router_route_kernel) phases, block (0,0)
                k0 = buf[8:13].astype(np.int64)
                print(label, "K0 (us): entry->wait, logits, cluster wait+DSMEM+sync, routing:",
                      np.round(np.diff(k0) / 1e3, 2).tolist(), file=sys.stderr)
            if buf[8] and "--c4" not in sys.argv:  # group path sub-phases (warp 0's own timeline)
                sub = buf[[1, 8, 9, 10, 11, 12, 13]].astype(np.int64)
                print(label, "route sub-phases (us): load+max, exp, sum, div, write, topk:",
                      np.round(np.diff(sub) / 1e3, 2).tolist(), file=sys.stderr)
        m = np.median(np.array(rows), axis=0)
        res[label] = {p: round(float(v), 2) for p, v in zip(PHASES[1:], m)}
        res[label]["total_us"] = round(float(m.sum()), 2)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
