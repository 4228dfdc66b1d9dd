"""GPU parity: dispatch permutation (K2), grouped expert FFN (K3, tcgen05) and
combine (K4) against the CPU oracle.

Tolerance for bf16 layer outputs (north star): norm-wise relative error
max|y - y_ref| / max|y_ref| <= 1e-2 against the fp32 CPU oracle on the same
bf16-valued inputs.
"""

from __future__ import annotations

import ctypes

import numpy as np
import pytest

from conftest import has_gpu
from oracle import lynx_oracle as O

pytestmark = pytest.mark.gpu

TOL = 1e-2  # norm-wise relative error vs fp32 oracle (bf16 output)

if has_gpu():
    import torch

    import paper_2411_08982_b200 as L
    from paper_2411_08982_b200 import _native as nat


def _np(t):
    return t.detach().float().cpu().numpy() if t.dtype == torch.bfloat16 else t.detach().cpu().numpy()


def make_mask(T, N, k, seed, drop=None):
    rng = np.random.default_rng(seed)
    z = rng.normal(0, 2.0, size=(T, N))
    sel = L.route_batch(L.RoutingLogits(0, L.Phase.DECODE, z), k)
    cfg = L.PolicyConfig(mode="latency", drop_count=drop if drop is not None else N // 2)
    return L.apply_policy(sel, L.Phase.DECODE, cfg)


def oracle_swiglu(model, layer, hidden_bf16, mask):
    w1, w3 = L.unpack_w13(model.w13[layer], model.spec.d_ff)
    f = lambda t: t.float().cpu().numpy()  # noqa: E731
    N, S = model.spec.num_experts, model.spec.num_shared_experts
    return O.forward_swiglu(f(hidden_bf16), f(w1), f(w3), f(model.w2[layer]), _np(mask.remap_assigned).astype(np.int64),
                            _np(mask.remap_weights), round_h_bf16=True, shared=range(N, N + S))


def test_permute_order_matches_reference_dispatch():
    T, N, k, d = 48, 8, 3, 64
    mask = make_mask(T, N, k, 3, drop=3)
    assigned = mask.remap_assigned.contiguous()
    weights = mask.remap_weights.contiguous()
    hidden = torch.randn((T, d), device="cuda").to(torch.bfloat16)
    max_seg, rows_cap = ctypes.c_int32(), ctypes.c_int32()
    nat.lib().lynx_dispatch_caps(T, N, k, ctypes.byref(max_seg), ctypes.byref(rows_cap))
    S, R = max_seg.value, rows_cap.value
    buf = {n: torch.full(s, -7, dtype=dt, device="cuda") for n, s, dt in [
        ("n_seg", (1,), torch.int32), ("n_used", (1,), torch.int32), ("n_rows", (1,), torch.int32),
        ("seg_expert", (S,), torch.int32),
        ("seg_row", (S,), torch.int32), ("seg_count", (S,), torch.int32), ("perm_token", (R,), torch.int32),
        ("perm_weight", (R,), torch.float32), ("tok_rows", (T, k), torch.int32),
        ("tok_weight", (T, k), torch.float32)]}
    x_perm = torch.zeros((R, d), dtype=torch.bfloat16, device="cuda")
    disp = nat.LynxDispatch(**{n: t.data_ptr() for n, t in buf.items()}, x_perm=x_perm.data_ptr())
    st = nat.lib().lynx_permute(assigned.data_ptr(), weights.data_ptr(), hidden.data_ptr(), T, N, k, d,
                                ctypes.cast(ctypes.pointer(disp), ctypes.c_void_p),
                                torch.cuda.current_stream().cuda_stream)
    assert st == 0
    torch.cuda.synchronize()
    ref = O.dispatch(_np(assigned).astype(np.int64), _np(weights))
    nseg = int(buf["n_seg"].item())
    assert nseg == len(ref.experts) and int(buf["n_used"].item()) == len(ref.experts)
    assert _np(buf["seg_expert"])[:nseg].tolist() == ref.experts
    for s, (e, rows, rw) in enumerate(zip(ref.experts, ref.rows, ref.row_weight)):
        r0, n = int(buf["seg_row"][s]), int(buf["seg_count"][s])
        assert r0 % 16 == 0 and n == len(rows)
        assert _np(buf["perm_token"])[r0:r0 + n].tolist() == rows.tolist()
        assert np.array_equal(_np(buf["perm_weight"])[r0:r0 + n], rw.astype(np.float32))
        assert torch.equal(x_perm[r0:r0 + n], hidden[torch.from_numpy(rows).cuda()])


@pytest.mark.parametrize("T,N,k,d,ff", [
    (16, 8, 2, 128, 256),     # tiny, one tile each way
    (32, 8, 2, 256, 384),     # ff not a multiple of 128 (3 phase-0 tiles of 64 features)
    (16, 8, 2, 32, 64),       # BASELINE C1 shape (d=32 < one 64-wide k block)
    (40, 4, 2, 512, 1408),    # > 32 rows per segment (BN=64), DeepSeek-like ff
    (300, 8, 2, 256, 512),    # segments split at 256 rows, BN=256
    (128, 64, 6, 256, 192),   # DeepSeek-like routing width (64 experts, top-6)
])
def test_forward_swiglu_vs_oracle(T, N, k, d, ff):
    spec = L.MoEModelSpec(1, N, k, d, ff)
    model = L.build_swiglu_model(spec, seed=T + ff)
    mask = make_mask(T, N, k, seed=T)
    hidden = torch.randn((T, d), device="cuda").to(torch.bfloat16)
    y = L.forward_layer(hidden, model, 0, mask)
    ref = oracle_swiglu(model, 0, hidden, mask)
    err = O.norm_rel_err(_np(y), ref)
    assert err <= TOL, err
    # the expert contribution alone (residual removed) must also match
    delta = _np(y) - _np(hidden)
    ref_delta = ref - _np(hidden)
    assert O.norm_rel_err(delta, ref_delta) <= 3 * TOL


def test_forward_is_deterministic():
    spec = L.MoEModelSpec(1, 8, 2, 256, 512)
    model = L.build_swiglu_model(spec, seed=1)
    mask = make_mask(64, 8, 2, seed=9)
    hidden = torch.randn((64, 256), device="cuda").to(torch.bfloat16)
    a = L.forward_layer(hidden, model, 0, mask)
    b = L.forward_layer(hidden, model, 0, mask)
    assert torch.equal(a, b)


def test_forward_tanh2_vs_reference_golden(forward_golden):
    """The reference's own expert (tanh(x w1) w2) through the tcgen05 kernel vs
    forward_layer outputs recorded from the reference (bf16 tolerance)."""
    for c in forward_golden:
        N, d, ff = c["w1"].shape
        k = int(c["k"])
        if d % 8 or ff % 8:
            continue
        spec = L.MoEModelSpec(1, N, k, d, ff)

        class Ref:  # duck-typed SyntheticMoE
            pass
        ref = Ref()
        ref.spec = spec
        ref.router_w, ref.w1, ref.w2 = c["router_w"][None], c["w1"][None], c["w2"][None]
        model = L.from_reference(ref)
        hidden = c["hidden"]
        mask = L.ExpertMask(layer_index=0, phase=L.Phase.DECODE, retained=torch.arange(N),
                            remap_original=torch.from_numpy(c["assigned"].astype(np.int32)).cuda(),
                            remap_assigned=torch.from_numpy(c["assigned"].astype(np.int32)).cuda(),
                            remap_weights=torch.from_numpy(c["weights"]).cuda())
        y = L.forward_layer(hidden, model, 0, mask)
        # oracle on the same bf16-rounded weights/input, and the f64 reference output
        f = lambda a: O.bf16_round(np.asarray(a, dtype=np.float32)).astype(np.float64)  # noqa: E731
        ref_bf = O.forward_tanh2(f(hidden), f(c["w1"]), f(c["w2"]), c["assigned"].astype(np.int64), c["weights"])
        assert O.norm_rel_err(_np(y), ref_bf) <= TOL
        assert O.norm_rel_err(_np(y), c["y"]) <= 2 * TOL


def test_layer_op_matches_stepwise_pipeline():
    """lynx_moe_layer (K0..K4 in one call) == router_logits -> route_batch ->
    apply_policy -> forward_layer, bit for bit."""
    spec = L.MoEModelSpec(1, 8, 2, 512, 1024)
    model = L.build_swiglu_model(spec, seed=4)
    T = 32
    hidden = torch.randn((T, 512), device="cuda").to(torch.bfloat16)
    cfg = L.PolicyConfig(mode="latency", drop_count=4)
    layer = L.LynxMoELayer(model, 0, T, policy=cfg)
    y = layer(hidden)
    logits = L.router_logits(model, 0, hidden)
    sel = L.route_batch(L.RoutingLogits(0, L.Phase.DECODE, logits), 2)
    mask = L.apply_policy(sel, L.Phase.DECODE, cfg)
    y2 = L.forward_layer(hidden, model, 0, mask)
    assert torch.equal(layer.assigned, mask.remap_assigned)
    assert torch.equal(y, y2)
    # logits vs fp64 oracle on the same bf16 values
    ref_logits = O.router_logits(_np(hidden).astype(np.float64), _np(model.router_wt[0]).astype(np.float64).T)
    assert np.max(np.abs(_np(logits) - ref_logits)) < 1e-3 * max(1.0, np.max(np.abs(ref_logits)))
    assert layer.used_experts() <= 4


def test_mixtral_shape_layer_vs_oracle():
    """C2: Mixtral-8x7B layer shape, T=32, Lynx latency drop 4, vs fp32 oracle."""
    spec = L.MoEModelSpec(1, 8, 2, 4096, 14336)
    model = L.build_swiglu_model(spec, seed=0)
    T = 32
    g = torch.Generator(device="cuda").manual_seed(0)
    hidden = torch.randn((T, 4096), generator=g, device="cuda").to(torch.bfloat16)
    layer = L.LynxMoELayer(model, 0, T, policy=L.PolicyConfig(mode="latency", drop_count=4))
    y = layer(hidden)
    mask = layer.mask()
    ref = oracle_swiglu(model, 0, hidden, mask)
    assert O.norm_rel_err(_np(y), ref) <= TOL
    assert O.norm_rel_err(_np(y) - _np(hidden), ref - _np(hidden)) <= 3 * TOL


@pytest.mark.parametrize("T,N,k,S,d,ff", [
    (16, 8, 2, 1, 128, 256),     # one shared expert
    (37, 16, 4, 2, 256, 192),    # T not a multiple of 16 (padded shared segment)
    (300, 8, 2, 2, 128, 128),    # shared segments split at 256 rows
])
def test_forward_shared_experts_vs_oracle(T, N, k, S, d, ff):
    """Always-on shared experts (DeepSeek-MoE, builder extension): every token,
    weight 1, after the routed experts."""
    spec = L.MoEModelSpec(1, N, k, d, ff, num_shared_experts=S)
    model = L.build_swiglu_model(spec, seed=T + S)
    mask = make_mask(T, N, k, seed=T)
    hidden = torch.randn((T, d), device="cuda").to(torch.bfloat16)
    y = L.forward_layer(hidden, model, 0, mask)
    ref = oracle_swiglu(model, 0, hidden, mask)
    assert O.norm_rel_err(_np(y), ref) <= TOL
    assert O.norm_rel_err(_np(y) - _np(hidden), ref - _np(hidden)) <= 3 * TOL


def test_deepseek_shape_layer_vs_oracle():
    """C4: DeepSeek-MoE-16B layer shape (64 routed + 2 shared, top-6, d=2048,
    ff=1408), T=128, Lynx accuracy policy (dynamic selection), vs fp32 oracle;
    the selection is checked bit-exactly against the oracle on the kernel's logits."""
    spec = L.MoEModelSpec(1, 64, 6, 2048, 1408, num_shared_experts=2)
    model = L.build_swiglu_model(spec, seed=0)
    T = 128
    g = torch.Generator(device="cuda").manual_seed(0)
    hidden = torch.randn((T, 2048), generator=g, device="cuda").to(torch.bfloat16)
    cfg = L.PolicyConfig(mode="accuracy", freq_keep_budget=16)
    layer = L.LynxMoELayer(model, 0, T, policy=cfg)
    y = layer(hidden)
    mask = layer.mask()
    logits = _np(L.router_logits(model, 0, hidden))
    ids, probs, full = O.route(logits, 6)
    ref_mask = O.apply(ids, probs, full, O.Policy(mode="accuracy", freq_keep_budget=16))
    assert np.array_equal(_np(layer.expert_ids), ids)
    assert np.array_equal(_np(mask.retained), ref_mask.retained)
    assert np.array_equal(_np(layer.assigned), ref_mask.assigned)
    ref = oracle_swiglu(model, 0, hidden, mask)
    assert O.norm_rel_err(_np(y), ref) <= TOL
    assert O.norm_rel_err(_np(y) - _np(hidden), ref - _np(hidden)) <= 3 * TOL
    assert layer.used_experts() == len(np.unique(ref_mask.assigned)) + 2


def test_host_step_graph_matches_device_call():
    """LynxMoELayer.host_step (H2D + layer + D2H replayed as one CUDA graph)
    returns exactly what the device-resident call returns, step after step."""
    spec = L.MoEModelSpec(1, 8, 2, 256, 512)
    model = L.build_swiglu_model(spec, seed=2)
    layer = L.LynxMoELayer(model, 0, 24, policy=L.PolicyConfig(mode="latency", drop_count=3))
    h_host = torch.randn((24, 256)).to(torch.bfloat16).pin_memory()
    o_host = torch.empty_like(h_host).pin_memory()
    for step in range(3):
        h_host.copy_(torch.randn((24, 256)).to(torch.bfloat16))  # new input, same pinned buffer
        layer.host_step(h_host, o_host)
        torch.cuda.synchronize()
        ref = layer(h_host.cuda()).cpu()
        assert torch.equal(o_host, ref), step


def test_stream_host_matches_device_calls():
    """LynxMoELayer.stream_host (copy-overlapped host batches) returns exactly
    the device-resident outputs, batch by batch, including the slot reuse."""
    spec = L.MoEModelSpec(1, 8, 2, 256, 512)
    model = L.build_swiglu_model(spec, seed=3)
    layer = L.LynxMoELayer(model, 0, 16, policy=L.PolicyConfig(mode="latency", drop_count=2))
    hs = [torch.randn((16, 256)).to(torch.bfloat16).pin_memory() for _ in range(5)]
    outs = [torch.empty_like(hs[0]).pin_memory() for _ in range(5)]
    layer.stream_host(hs, outs)
    torch.cuda.synchronize()
    for h, o in zip(hs, outs):
        assert torch.equal(o, layer(h.cuda()).cpu())


# ---- the reference's forward_layer known answers (test_simulator.py:71-125),
# embedded at d = ff = 8 (the kernels need 16-byte rows): the reference's
# 2x2 blocks sit top-left, the padding is zero, so columns 0-1 carry the
# reference's numbers and the rest stay equal to the input.
def _embed_model(w1_blocks, w2_blocks, N, k, d=8):
    class Ref:  # duck-typed SyntheticMoE
        pass
    ref = Ref()
    ref.spec = L.MoEModelSpec(1, N, k, d, d)
    ref.w1 = np.zeros((1, N, d, d))
    ref.w2 = np.zeros((1, N, d, d))
    ref.w1[0, :, :2, :2] = w1_blocks
    ref.w2[0, :, :2, :2] = w2_blocks
    ref.router_w = np.zeros((1, d, N))
    return L.from_reference(ref)


def _mask(assigned, weights, N):
    a = torch.as_tensor(np.asarray(assigned), dtype=torch.int32).cuda()
    return L.ExpertMask(layer_index=0, phase=L.Phase.DECODE, retained=torch.arange(N).cuda(), remap_original=a,
                        remap_assigned=a, remap_weights=torch.as_tensor(np.asarray(weights, dtype=np.float64)).cuda())


def _hid(rows, d=8):
    h = np.zeros((len(rows), d))
    h[:, :2] = rows
    return torch.from_numpy(h).float().cuda().to(torch.bfloat16)


def test_reference_hand_computed_forward():
    """test_simulator.py:71-83: token 0 -> expert 0 gives h + 0.5 tanh(h),
    token 1 -> expert 1 gives h + swap(tanh(2h))."""
    model = _embed_model(np.stack([np.eye(2), 2 * np.eye(2)]), np.stack([0.5 * np.eye(2), [[0, 1], [1, 0]]]), 2, 1)
    hidden = _hid([[1.0, 0.0], [0.0, 1.0]])
    y = _np(L.forward_layer(hidden, model, 0, _mask([[0], [1]], [[1.0], [1.0]], 2)))
    h = np.array([[1.0, 0.0], [0.0, 1.0]])
    exp0 = h[0] + 0.5 * np.tanh(h[0])
    exp1 = h[1] + np.tanh(2.0 * h[1]) @ np.array([[0.0, 1.0], [1.0, 0.0]])
    assert np.allclose(y[0, :2], exp0, atol=1e-2) and np.allclose(y[1, :2], exp1, atol=1e-2)
    assert np.all(y[:, 2:] == 0)


def test_reference_collapsed_slots_apply_expert_once():
    """test_simulator.py:94-118: remap onto retained {1} with k=2 collapses
    both slots onto expert 1; the expert runs once with the merged weight 1."""
    rng = np.random.default_rng(3)
    w1 = rng.normal(size=(4, 2, 2))
    w2 = rng.normal(size=(4, 2, 2))
    model = _embed_model(w1, w2, 4, 2)
    logits = rng.normal(size=(3, 4))
    sel = L.route_batch(L.RoutingLogits(0, L.Phase.DECODE, logits), 2)
    _, assigned, weights = L.remap_tokens(sel, np.array([1]))
    assert torch.all(assigned == 1)
    hx = rng.normal(size=(3, 2))
    hidden = _hid(hx)
    y = _np(L.forward_layer(hidden, model, 0, _mask(assigned.cpu().numpy(), weights.cpu().numpy(), 4)))
    hb = _np(hidden)[:, :2].astype(np.float64)
    f = lambda a: O.bf16_round(np.asarray(a, dtype=np.float32)).astype(np.float64)  # noqa: E731
    ref = hb + np.tanh(hb @ f(w1[1])) @ f(w2[1])
    assert O.norm_rel_err(y[:, :2], ref) <= 1e-2


def test_forward_rejects_token_mismatch():
    """test_simulator.py:120-125: mask rows != hidden rows -> ValidationError."""
    model = _embed_model(np.stack([np.eye(2), np.eye(2)]), np.stack([np.eye(2), np.eye(2)]), 2, 1)
    with pytest.raises(L.ValidationError):
        L.forward_layer(_hid([[1.0, 0.0], [0.0, 1.0]]), model, 0, _mask([[0]], [[1.0]], 2))


@pytest.mark.parametrize("seed", range(64))
def test_random_layer_configs_vs_oracle(seed):
    """Randomised whole-layer parity (lynx_moe_layer: K0..K4) over shapes and
    policies: T 1..300, N 2..64, k 1..min(8,N), shared 0..2, d / ff multiples
    of 8 (including ones that are not multiples of 64), latency / accuracy
    policies with random settings, decode and prefill.  Selection bit-exact
    vs the oracle on the kernel's logits; output within the bf16 tolerance."""
    rng = np.random.default_rng(1000 + seed)
    N = int(rng.choice([1, 2, 3, 5, 8, 12, 16, 24, 33, 48, 64]))
    k = int(rng.integers(1, min(8, N) + 1))
    S = int(rng.choice([0, 0, 1, 2]))
    T = int(rng.choice([1, 3, 16, 31, 64, 100, 257, 300]))
    d = int(rng.choice([64, 136, 256, 512]))
    ff = int(rng.choice([64, 120, 192, 512]))
    decode = bool(rng.integers(0, 4))  # mostly decode
    if rng.integers(0, 2):
        cfg = L.PolicyConfig(mode="latency", drop_count=int(rng.integers(0, N + 1)))
        opol = O.Policy(mode="latency", drop_count=cfg.drop_count)
    else:
        mk = int(rng.integers(k, N + 1)) if rng.integers(0, 2) else None
        cfg = L.PolicyConfig(mode="accuracy", confidence_threshold=float(rng.choice([0.2, 0.4, 0.6])),
                             sample_threshold=int(rng.integers(1, 12)), min_experts=mk,
                             freq_keep_budget=int(rng.integers(1, N + 1)),
                             confidence_metric=str(rng.choice(["top1", "margin"])))
        opol = O.Policy(mode="accuracy", confidence_threshold=cfg.confidence_threshold,
                        sample_threshold=cfg.sample_threshold, min_experts=mk,
                        freq_keep_budget=cfg.freq_keep_budget, confidence_metric=cfg.confidence_metric)
    spec = L.MoEModelSpec(1, N, k, d, ff, num_shared_experts=S)
    model = L.build_swiglu_model(spec, seed=seed)
    g = torch.Generator(device="cuda").manual_seed(seed)
    hidden = torch.randn((T, d), generator=g, device="cuda").to(torch.bfloat16)
    layer = L.LynxMoELayer(model, 0, T, policy=cfg, phase=L.Phase.DECODE if decode else L.Phase.PREFILL)
    y = layer(hidden)
    torch.cuda.synchronize()
    logits = _np(L.router_logits(model, 0, hidden))
    ids, probs, full = O.route(logits, k)
    ref_mask = O.apply(ids, probs, full, opol, decode=decode)
    tag = dict(N=N, k=k, S=S, T=T, d=d, ff=ff, decode=decode, cfg=cfg)
    assert np.array_equal(_np(layer.expert_ids), ids), tag
    assert np.array_equal(_np(layer.assigned), ref_mask.assigned), tag
    keep = np.zeros(N, dtype=np.uint8)
    keep[ref_mask.retained] = 1
    assert np.array_equal(_np(layer.retained_mask), keep), tag
    assert np.allclose(_np(layer.weights), ref_mask.weights, rtol=1e-12, atol=1e-15), tag
    w1, w3 = L.unpack_w13(model.w13[0], ff)
    f = lambda t: t.float().cpu().numpy()  # noqa: E731
    ref = O.forward_swiglu(f(hidden), f(w1), f(w3), f(model.w2[0]), ref_mask.assigned, ref_mask.weights,
                           round_h_bf16=True, shared=range(N, N + S))
    assert O.norm_rel_err(_np(y), ref) <= TOL, tag


@pytest.mark.parametrize("seed", range(32))
def test_random_layer_configs_large_batches_vs_oracle(seed):
    """A second randomised sweep for the large-batch paths: T 257..2048 (K1
    in global memory once its per-token arrays do not fit shared memory,
    expert segments split at 256 rows, the CTA-pair K3 on wide segments),
    rank-weighted latency votes and min_experts floors included."""
    rng = np.random.default_rng(5000 + seed)
    N = int(rng.choice([2, 8, 9, 16, 17, 40, 64]))
    k = int(rng.integers(1, min(8, N) + 1))
    S = int(rng.choice([0, 0, 1, 2]))
    T = int(rng.choice([257, 333, 512, 700, 1024, 2048]))
    d = int(rng.choice([64, 136, 256]))
    ff = int(rng.choice([64, 120, 192]))
    decode = bool(rng.integers(0, 4))
    kind = int(rng.integers(0, 3))
    if kind == 0:
        cfg = L.PolicyConfig(mode="latency", drop_count=int(rng.integers(0, N + 1)))
        opol = O.Policy(mode="latency", drop_count=cfg.drop_count)
    elif kind == 1:
        mk = int(rng.integers(k, N + 1))
        rw = tuple(float(x) for x in rng.uniform(0.1, 1.0, size=k))
        cfg = L.PolicyConfig(mode="latency", drop_count=int(rng.integers(0, N + 1)), min_experts=mk,
                             vote_rank_weights=rw)
        opol = O.Policy(mode="latency", drop_count=cfg.drop_count, min_experts=mk, vote_rank_weights=rw)
    else:
        mk = int(rng.integers(k, N + 1)) if rng.integers(0, 2) else None
        cfg = L.PolicyConfig(mode="accuracy", confidence_threshold=float(rng.choice([0.1, 0.3, 0.5])),
                             sample_threshold=int(rng.integers(1, 40)), min_experts=mk,
                             freq_keep_budget=int(rng.integers(1, N + 1)),
                             confidence_metric=str(rng.choice(["top1", "margin"])))
        opol = O.Policy(mode="accuracy", confidence_threshold=cfg.confidence_threshold,
                        sample_threshold=cfg.sample_threshold, min_experts=mk,
                        freq_keep_budget=cfg.freq_keep_budget, confidence_metric=cfg.confidence_metric)
    spec = L.MoEModelSpec(1, N, k, d, ff, num_shared_experts=S)
    model = L.build_swiglu_model(spec, seed=seed + 100)
    g = torch.Generator(device="cuda").manual_seed(seed)
    hidden = torch.randn((T, d), generator=g, device="cuda").to(torch.bfloat16)
    layer = L.LynxMoELayer(model, 0, T, policy=cfg, phase=L.Phase.DECODE if decode else L.Phase.PREFILL)
    y = layer(hidden)
    torch.cuda.synchronize()
    logits = _np(L.router_logits(model, 0, hidden))
    ids, probs, full = O.route(logits, k)
    ref_mask = O.apply(ids, probs, full, opol, decode=decode)
    tag = dict(N=N, k=k, S=S, T=T, d=d, ff=ff, decode=decode, cfg=cfg)
    assert np.array_equal(_np(layer.expert_ids), ids), tag
    assert np.array_equal(_np(layer.assigned), ref_mask.assigned), tag
    keep = np.zeros(N, dtype=np.uint8)
    keep[ref_mask.retained] = 1
    assert np.array_equal(_np(layer.retained_mask), keep), tag
    assert np.allclose(_np(layer.weights), ref_mask.weights, rtol=1e-12, atol=1e-15), tag
    assert bool(int(layer.flags.item()) & 1) == bool(ref_mask.clipped), tag
    w1, w3 = L.unpack_w13(model.w13[0], ff)
    f = lambda t: t.float().cpu().numpy()  # noqa: E731
    ref = O.forward_swiglu(f(hidden), f(w1), f(w3), f(model.w2[0]), ref_mask.assigned, ref_mask.weights,
                           round_h_bf16=True, shared=range(N, N + S))
    assert O.norm_rel_err(_np(y), ref) <= TOL, tag


@pytest.mark.parametrize("T,N,k,S,mode", [(4096, 64, 8, 2, "accuracy"), (4096, 64, 8, 0, "latency"),
                                          (4096, 8, 2, 0, "latency"), (1024, 33, 5, 1, "accuracy")])
def test_layer_at_maximum_sizes_vs_oracle(T, N, k, S, mode):
    """The whole layer at the ABI limits (T <= 4096, N <= 64, k <= 8): K1
    works in global memory when its per-token arrays do not fit in shared
    memory, segments split at LYNX_SEG_ROWS, and the K3 queue holds more
    segments than K1 ranks in shared memory."""
    d, ff = 128, 64
    cfg = (L.PolicyConfig(mode="latency", drop_count=N // 2) if mode == "latency"
           else L.PolicyConfig(mode="accuracy", freq_keep_budget=N // 3))
    opol = (O.Policy(mode="latency", drop_count=N // 2) if mode == "latency"
            else O.Policy(mode="accuracy", freq_keep_budget=N // 3))
    spec = L.MoEModelSpec(1, N, k, d, ff, num_shared_experts=S)
    model = L.build_swiglu_model(spec, seed=7)
    g = torch.Generator(device="cuda").manual_seed(7)
    hidden = torch.randn((T, d), generator=g, device="cuda").to(torch.bfloat16)
    layer = L.LynxMoELayer(model, 0, T, policy=cfg)
    y = layer(hidden)
    torch.cuda.synchronize()
    logits = _np(L.router_logits(model, 0, hidden))
    ids, probs, full = O.route(logits, k)
    ref_mask = O.apply(ids, probs, full, opol)
    assert np.array_equal(_np(layer.expert_ids), ids)
    assert np.array_equal(_np(layer.assigned), ref_mask.assigned)
    assert np.allclose(_np(layer.weights), ref_mask.weights, rtol=1e-12, atol=1e-15)
    w1, w3 = L.unpack_w13(model.w13[0], ff)
    f = lambda t: t.float().cpu().numpy()  # noqa: E731
    ref = O.forward_swiglu(f(hidden), f(w1), f(w3), f(model.w2[0]), ref_mask.assigned, ref_mask.weights,
                           round_h_bf16=True, shared=range(N, N + S))
    assert O.norm_rel_err(_np(y), ref) <= TOL


def test_cta_pair_kernel_forced_on_every_shape():
    """K3's CTA-pair kernel (tcgen05 cta_group::2) normally runs only for wide
    segments; force it (LYNX_FFN_PAIR=1) and rerun the layer parity tests so
    narrow, odd-tile and shared-expert shapes go through it too (and =0 for
    the single-CTA kernel on the wide shapes)."""
    import os
    import subprocess
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    for force in ("1", "0"):
        env = dict(os.environ, LYNX_FFN_PAIR=force)
        r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider",
                            os.path.join(here, "test_gpu_ffn.py"), "-k",
                            "random_layer or maximum_sizes or shared_experts or deepseek or swiglu_vs_oracle"],
                           env=env, capture_output=True, text=True, timeout=900)
        assert r.returncode == 0, (force, r.stdout[-3000:], r.stderr[-2000:])


@pytest.mark.parametrize("env", ["LYNX_ROUTE_IN_K1=1", "LYNX_FFN_MT=1", "LYNX_L2_DISCARD=0", "LYNX_L2_DISCARD=2"])
def test_runtime_switches_keep_parity(env):
    """The A/B switches (run-time switches) change how the layer
    runs, never its results: rerun the layer parity tests under each."""
    import os
    import subprocess
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    key, val = env.split("=")
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider",
                        os.path.join(here, "test_gpu_ffn.py"), "-k",
                        "random_layer_configs_vs or deepseek or swiglu_vs_oracle or tanh2"],
                       env=dict(os.environ, **{key: val}), capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, (env, r.stdout[-3000:], r.stderr[-2000:])


@pytest.mark.parametrize("kb2_per", ["3", "1000"])
def test_split_k_slot_counts(kb2_per):
    """K4 is specialised on the split-K slot count (1 or 2 at every BASELINE
    shape, a generic loop otherwise): force many slots (LYNX_KB2_PER=3, the
    generic path) and a single slot (1000) and rerun the layer parity tests."""
    import os
    import subprocess
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    env = dict(os.environ, LYNX_KB2_PER=kb2_per)
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider",
                        os.path.join(here, "test_gpu_ffn.py"), "-k",
                        "random_layer or shared_experts or deepseek or swiglu_vs_oracle or tanh2"],
                       env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, (kb2_per, r.stdout[-3000:], r.stderr[-2000:])


@pytest.mark.parametrize("case", ["c2", "acc", "t256", "n5"])
def test_fused_front_identical_to_kernel_chain(case, tmp_path):
    """The fused front (K0 + K1 + K2 in one launch, N <= 8) against the
    K0 -> K1 -> K2 chain (LYNX_FUSED_FRONT=0): every selection output, the
    flags and the layer output bit for bit, decode and prefill."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for f in ("1", "0"):
        path = str(tmp_path / f"front{f}.npz")
        r = subprocess.run([sys.executable, os.path.join(root, "scripts", "front_ab_dump.py"), path, case],
                           env=dict(os.environ, LYNX_FUSED_FRONT=f), capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(np.load(path))
    a, b = outs
    assert sorted(a.files) == sorted(b.files)
    for key in a.files:
        assert np.array_equal(a[key], b[key]), key


@pytest.mark.parametrize("T", [1, 2, 31, 32, 33, 255, 256])
def test_fused_front_edge_shapes_vs_oracle(T):
    """The fused front's edges (N <= 8, T <= 256): one token, a partial warp,
    exactly one / just over one warp of tokens (the warp-level plan switches
    at 32), the 256-token limit; N from 1 to 8, k up to N; latency policies
    with drops past the floor, min_experts and rank weights (the batch_policy
    path), accuracy policies, prefill.  Selection bit-exact vs the oracle on
    the kernel's logits, layer output within the bf16 tolerance."""
    rng = np.random.default_rng(T)
    for rep in range(6):
        N = int(rng.choice([1, 2, 5, 7, 8]))
        k = int(rng.integers(1, N + 1))
        d, ff = int(rng.choice([64, 128])), int(rng.choice([64, 192]))
        decode = rep != 5
        kind = rep % 4
        if kind == 0:
            cfg = L.PolicyConfig(mode="latency", drop_count=int(rng.integers(0, N + 2)))
            opol = O.Policy(mode="latency", drop_count=cfg.drop_count)
        elif kind == 1:
            mk = int(rng.integers(k, N + 1))
            rw = tuple(float(x) for x in rng.uniform(0.1, 1.0, size=k))
            cfg = L.PolicyConfig(mode="latency", drop_count=int(rng.integers(0, N + 1)), min_experts=mk,
                                 vote_rank_weights=rw)
            opol = O.Policy(mode="latency", drop_count=cfg.drop_count, min_experts=mk, vote_rank_weights=rw)
        else:
            cfg = L.PolicyConfig(mode="accuracy", confidence_threshold=float(rng.choice([0.2, 0.5])),
                                 sample_threshold=int(rng.integers(1, 10)), freq_keep_budget=int(rng.integers(1, N + 1)),
                                 confidence_metric=str(rng.choice(["top1", "margin"])))
            opol = O.Policy(mode="accuracy", confidence_threshold=cfg.confidence_threshold,
                            sample_threshold=cfg.sample_threshold, freq_keep_budget=cfg.freq_keep_budget,
                            confidence_metric=cfg.confidence_metric)
        model = L.build_swiglu_model(L.MoEModelSpec(1, N, k, d, ff), seed=T * 10 + rep)
        g = torch.Generator(device="cuda").manual_seed(rep)
        hidden = torch.randn((T, d), generator=g, device="cuda").to(torch.bfloat16)
        layer = L.LynxMoELayer(model, 0, T, policy=cfg, phase=L.Phase.DECODE if decode else L.Phase.PREFILL)
        y = layer(hidden)
        torch.cuda.synchronize()
        logits = _np(L.router_logits(model, 0, hidden))
        ids, probs, full = O.route(logits, k)
        ref_mask = O.apply(ids, probs, full, opol, decode=decode)
        tag = dict(T=T, N=N, k=k, rep=rep, decode=decode, cfg=cfg)
        assert np.array_equal(_np(layer.expert_ids), ids), tag
        assert np.array_equal(_np(layer.assigned), ref_mask.assigned), tag
        keep = np.zeros(N, dtype=np.uint8)
        keep[ref_mask.retained] = 1
        assert np.array_equal(_np(layer.retained_mask), keep), tag
        assert np.allclose(_np(layer.weights), ref_mask.weights, rtol=1e-12, atol=1e-15), tag
        assert bool(int(layer.flags.item()) & 1) == bool(ref_mask.clipped), tag
        w1, w3 = L.unpack_w13(model.w13[0], ff)
        f = lambda t: t.float().cpu().numpy()  # noqa: E731
        ref = O.forward_swiglu(f(hidden), f(w1), f(w3), f(model.w2[0]), ref_mask.assigned, ref_mask.weights)
        assert O.norm_rel_err(_np(y), ref) <= TOL, tag


@pytest.mark.parametrize("T", [1, 7, 8, 9, 33, 128, 255, 256])
def test_wide_router_edge_shapes_vs_oracle(T):
    """Wide routers (8 < N <= 64: K1's thread-per-token path up to 16, K0's
    cluster routing + K1's group path above) at the decode batch edges: one
    token, partial / whole / just over one 4-token routing cluster, 256
    tokens; N across the 8-expert CTA widths (9, 16, 17, 40, 64), k up to 8,
    shared experts 0..2; latency policies with drops past the
    floor, min_experts and rank weights, accuracy policies (top1 / margin),
    prefill.  Selection bit-exact vs the oracle on the kernel's logits,
    layer output within the bf16 tolerance."""
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
            opol = O.Policy(mode="latency", drop_count=cfg.drop_count)
        elif kind == 1:
            mk = int(rng.integers(k, N + 1))
            rw = tuple(float(x) for x in rng.uniform(0.1, 1.0, size=k))
            cfg = L.PolicyConfig(mode="latency", drop_count=int(rng.integers(0, N + 1)), min_experts=mk,
                                 vote_rank_weights=rw)
            opol = O.Policy(mode="latency", drop_count=cfg.drop_count, min_experts=mk, vote_rank_weights=rw)
        else:
            cfg = L.PolicyConfig(mode="accuracy", confidence_threshold=float(rng.choice([0.1, 0.3])),
                                 sample_threshold=int(rng.integers(1, 10)), freq_keep_budget=int(rng.integers(1, N + 1)),
                                 confidence_metric=str(rng.choice(["top1", "margin"])))
            opol = O.Policy(mode="accuracy", confidence_threshold=cfg.confidence_threshold,
                            sample_threshold=cfg.sample_threshold, freq_keep_budget=cfg.freq_keep_budget,
                            confidence_metric=cfg.confidence_metric)
        model = L.build_swiglu_model(L.MoEModelSpec(1, N, k, d, ff, num_shared_experts=S), seed=T * 10 + rep)
        g = torch.Generator(device="cuda").manual_seed(rep)
        hidden = torch.randn((T, d), generator=g, device="cuda").to(torch.bfloat16)
        layer = L.LynxMoELayer(model, 0, T, policy=cfg, phase=L.Phase.DECODE if decode else L.Phase.PREFILL)
        y = layer(hidden)
        torch.cuda.synchronize()
        logits = _np(L.router_logits(model, 0, hidden))
        ids, probs, full = O.route(logits, k)
        ref_mask = O.apply(ids, probs, full, opol, decode=decode)
        tag = dict(T=T, N=N, k=k, S=S, rep=rep, decode=decode, cfg=cfg)
        assert np.array_equal(_np(layer.expert_ids), ids), tag
        assert np.allclose(_np(layer.full_probs), full, rtol=1e-12, atol=1e-15), tag
        assert np.array_equal(_np(layer.assigned), ref_mask.assigned), tag
        keep = np.zeros(N, dtype=np.uint8)
        keep[ref_mask.retained] = 1
        assert np.array_equal(_np(layer.retained_mask), keep), tag
        assert np.allclose(_np(layer.weights), ref_mask.weights, rtol=1e-12, atol=1e-15), tag
        assert bool(int(layer.flags.item()) & 1) == bool(ref_mask.clipped), tag
        w1, w3 = L.unpack_w13(model.w13[0], ff)
        f = lambda t: t.float().cpu().numpy()  # noqa: E731
        ref = O.forward_swiglu(f(hidden), f(w1), f(w3), f(model.w2[0]), ref_mask.assigned, ref_mask.weights,
                               shared=range(N, N + S))
        assert O.norm_rel_err(_np(y), ref) <= TOL, tag
