"""Small K1 repro: route_batch + apply_policy at one shape, with the CUDA error string."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_08982_b200 as L  # noqa: E402

T, N, k = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (128, 64, 6)))
z = np.random.default_rng(0).normal(0, 2, size=(T, N))
try:
    sel = L.route_batch(L.RoutingLogits(0, L.Phase.DECODE, z), k)
    torch.cuda.synchronize()
    print("route ok", sel.expert_ids[:2].tolist())
    m = L.apply_policy(sel, L.Phase.DECODE, L.PolicyConfig(mode="accuracy", freq_keep_budget=16))
    torch.cuda.synchronize()
    print("policy ok", m.retained.tolist())
except Exception as e:
    print("ERR", type(e).__name__, e)
