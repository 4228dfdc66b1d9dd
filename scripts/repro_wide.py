"""Repro one wide-router edge case (tests/test_gpu_ffn.py::test_wide_router_edge_shapes_vs_oracle).
    python scripts/repro_wide.py T rep"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_08982_b200 as L  # noqa: E402


def main():
    T, want = int(sys.argv[1]), int(sys.argv[2])
    rng = np.random.default_rng(1000 + T)
    for rep in range(5):
        N = int(rng.choice([9, 16, 17, 40, 64]))
        k = int(rng.integers(1, min(8, N) + 1))
        S = int(rng.integers(0, 3))
        d, ff = int(rng.choice([64, 128])), int(rng.choice([64, 192]))
        decode = rep != 4
        kind = rep % 3
        if kind == 0:
            cfg = L.PolicyConfig(mode="latency", drop_count=int(rng.integers(0, N + 2)))
        elif kind == 1:
            mk = int(rng.integers(k, N + 1))
            rw = tuple(float(x) for x in rng.uniform(0.1, 1.0, size=k))
            cfg = L.PolicyConfig(mode="latency", drop_count=int(rng.integers(0, N + 1)), min_experts=mk,
                                 vote_rank_weights=rw)
        else:
            cfg = L.PolicyConfig(mode="accuracy", confidence_threshold=float(rng.choice([0.1, 0.3])),
                                 sample_threshold=int(rng.integers(1, 10)), freq_keep_budget=int(rng.integers(1, N + 1)),
                                 confidence_metric=str(rng.choice(["top1", "margin"])))
        if rep != want:
            continue
        print(dict(T=T, N=N, k=k, S=S, d=d, ff=ff, decode=decode, cfg=cfg), flush=True)
        model = L.build_swiglu_model(L.MoEModelSpec(1, N, k, d, ff, num_shared_experts=S), seed=T * 10 + rep)
        g = torch.Generator(device="cuda").manual_seed(rep)
        hidden = torch.randn((T, d), generator=g, device="cuda").to(torch.bfloat16)
        layer = L.LynxMoELayer(model, 0, T, policy=cfg, phase=L.Phase.DECODE if decode else L.Phase.PREFILL)
        layer(hidden)
        torch.cuda.synchronize()
        print("ok", layer.used_experts())


if __name__ == "__main__":
    main()
