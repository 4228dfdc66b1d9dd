"""Small-shape driver for compute-sanitizer (memcheck / racecheck / synccheck).

    compute-sanitizer --tool memcheck python scripts/sanitize.py [case ...]

Every case runs the product kernels once at a small shape:
  fast     -- lynx_moe_layer, N=8 k=2 (K0 -> K1 thread-per-token -> K2 -> K3 single-CTA -> K4)
  group    -- lynx_moe_layer, N=64 k=6 + 2 shared (K0 cluster routing -> K1 group path -> ...)
  pair     -- lynx_moe_layer with wide segments (K3 CTA-pair kernel, cta_group::2)
  apply    -- lynx_apply_policy / lynx_remap / lynx_topk / lynx_vote on a given selection
  forward  -- lynx_permute + lynx_moe_forward + lynx_moe_forward_partial
  ep       -- peer-memory EP (lynx_ep_p2p_*), 2 simulated ranks on one GPU
  stack    -- DecodeStack: attention + fused router + layer, prefill + 2 graphed decode steps
Exits non-zero if any CUDA call fails.
"""

from __future__ import annotations

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2411_08982_b200 as L  # noqa: E402


def layer_case(T, N, k, S, d, ff, cfg, pair=None):
    if pair is not None:
        os.environ["LYNX_FFN_PAIR"] = pair
    spec = L.MoEModelSpec(1, N, k, d, ff, num_shared_experts=S)
    model = L.build_swiglu_model(spec, seed=T + N)
    g = torch.Generator(device="cuda").manual_seed(T)
    hidden = torch.randn((T, d), generator=g, device="cuda").to(torch.bfloat16)
    layer = L.LynxMoELayer(model, 0, T, policy=cfg)
    for _ in range(2):
        y = layer(hidden)
    torch.cuda.synchronize()
    assert bool(torch.isfinite(y.float()).all())
    os.environ.pop("LYNX_FFN_PAIR", None)


def case_fast():
    layer_case(32, 8, 2, 0, 256, 512, L.PolicyConfig(mode="latency", drop_count=4))
    layer_case(16, 8, 2, 0, 128, 256, L.PolicyConfig(mode="accuracy", freq_keep_budget=3))


def case_group():
    layer_case(128, 64, 6, 2, 256, 192, L.PolicyConfig(mode="accuracy", freq_keep_budget=16))
    layer_case(40, 24, 3, 0, 128, 128, L.PolicyConfig(mode="latency", drop_count=8))


def case_pair():
    layer_case(256, 8, 2, 0, 256, 512, L.PolicyConfig(mode="latency", drop_count=4), pair="1")
    layer_case(48, 8, 2, 1, 128, 192, L.PolicyConfig(mode="latency", drop_count=2), pair="1")


def case_apply():
    import numpy as np
    rng = np.random.default_rng(0)
    for (T, N, k) in [(32, 8, 2), (100, 64, 6)]:
        z = rng.normal(0, 2, size=(T, N))
        sel = L.route_batch(L.RoutingLogits(0, L.Phase.DECODE, z), k)
        for cfg in (L.PolicyConfig(mode="latency", drop_count=N // 2),
                    L.PolicyConfig(mode="accuracy", freq_keep_budget=3, confidence_metric="margin")):
            L.apply_policy(sel, L.Phase.DECODE, cfg)
        L.remap_tokens(sel, np.array([1, 2]))
        L.vote_expert_frequencies(sel)
    torch.cuda.synchronize()


def case_forward():
    spec = L.MoEModelSpec(1, 8, 2, 256, 384)
    model = L.build_swiglu_model(spec, seed=5)
    z = torch.randn((48, 8), dtype=torch.float64).numpy()
    sel = L.route_batch(L.RoutingLogits(0, L.Phase.DECODE, z), 2)
    mask = L.apply_policy(sel, L.Phase.DECODE, L.PolicyConfig(mode="latency", drop_count=3))
    hidden = torch.randn((48, 256), device="cuda").to(torch.bfloat16)
    L.forward_layer(hidden, model, 0, mask)
    L.forward_partial(hidden, model, 0, mask.remap_assigned.contiguous(), mask.remap_weights.contiguous())
    torch.cuda.synchronize()


def case_ep():
    from paper_2411_08982_b200 import ep as EP
    from paper_2411_08982_b200 import ep_p2p as P2P
    G, Tl, N, k, d, ff = 2, 16, 8, 2, 256, 256
    model = L.build_swiglu_model(L.MoEModelSpec(1, N, k, d, ff), seed=3)
    cfg = L.PolicyConfig(mode="latency", drop_count=4)
    peers = P2P.simulated_peers(G, Tl, N, d)
    layers = [P2P.P2PEPLayer(peers[r], model.router_wt[0], EP.shard_experts(model.w13[0], r, G),
                             EP.shard_experts(model.w2[0], r, G), N, k, ff, cfg) for r in range(G)]
    hs = [torch.randn((Tl, d), device="cuda").to(torch.bfloat16) for _ in range(G)]
    for _ in range(2):
        P2P.run_simulated(layers, hs)
    torch.cuda.synchronize()


def case_stack():
    nl, B, d, ff = 2, 8, 128, 256
    model = L.build_swiglu_model(L.MoEModelSpec(nl, 8, 2, d, ff), seed=0)
    attn = L.build_attention(nl, d, 16, seed=1)
    stack = L.DecodeStack(model, attn, B, max_len=16, policy=L.PolicyConfig(mode="latency", drop_count=3))
    stack.prefill(torch.randn((B, 4, d)).to(torch.bfloat16))
    for _ in range(2):
        stack.step()
    torch.cuda.synchronize()


CASES = {n[5:]: f for n, f in globals().items() if n.startswith("case_")}

if __name__ == "__main__":
    todo = sys.argv[1:] or list(CASES)
    for name in todo:
        CASES[name]()
        print(f"sanitize case {name}: ok", flush=True)
