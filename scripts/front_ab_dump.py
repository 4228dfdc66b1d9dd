"""Dump one layer call's outputs (selection, plan-visible results, layer output)
for the fused-front A/B test: LYNX_FUSED_FRONT=0/1 python scripts/front_ab_dump.py <out.npz> <case>"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_08982_b200 as L  # noqa: E402

CASES = {  # T, N, k, d, ff, policy
    "c2": (32, 8, 2, 512, 1024, L.PolicyConfig(mode="latency", drop_count=4)),
    "acc": (77, 8, 3, 256, 512, L.PolicyConfig(mode="accuracy", freq_keep_budget=3, confidence_metric="margin")),
    "t256": (256, 8, 2, 256, 384, L.PolicyConfig(mode="latency", drop_count=2)),
    "n5": (19, 5, 2, 128, 256, L.PolicyConfig(mode="accuracy", freq_keep_budget=1, min_experts=3)),
}


def main():
    out, case = sys.argv[1], sys.argv[2]
    T, N, k, d, ff, pol = CASES[case]
    model = L.build_swiglu_model(L.MoEModelSpec(1, N, k, d, ff), seed=T + N)
    g = torch.Generator(device="cuda").manual_seed(T)
    res = {}
    for phase in (L.Phase.DECODE, L.Phase.PREFILL):
        h = torch.randn((T, d), generator=g, device="cuda").to(torch.bfloat16)
        layer = L.LynxMoELayer(model, 0, T, policy=pol, phase=phase)
        y = layer(h)
        torch.cuda.synchronize()
        p = phase.value
        for name in ("expert_ids", "probs", "full_probs", "conf", "counts", "retained_mask", "assigned", "weights",
                     "important", "flags"):
            res[f"{p}_{name}"] = getattr(layer, name).cpu().numpy()
        res[f"{p}_y"] = y.view(torch.int16).cpu().numpy()
    np.savez(out, **res)


if __name__ == "__main__":
    main()
