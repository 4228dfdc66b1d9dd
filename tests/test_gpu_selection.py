"""GPU parity: routing + retention policies vs the reference's golden vectors.

Bit-exact for every decision (ids, retained set, remap, important tokens,
clipped flag) and -- since the device softmax restates numpy's own float64
exp (csrc/npexp.cuh), pairwise row sum and division -- for the float64
probabilities, confidences and weights too, on the fixtures made on the
generator machine (tests/golden/make_golden.py).  Comparisons against the
oracle run on the GPU box's own numpy keep 1e-12 for floats (its numpy may
take another exp path).
"""

from __future__ import annotations

import ctypes

import numpy as np
import pytest

from conftest import has_gpu
from oracle import lynx_oracle as O

pytestmark = pytest.mark.gpu

if has_gpu():
    import torch

    import paper_2411_08982_b200 as L
    from paper_2411_08982_b200 import _native as nat


def _policy(meta):
    cfg = meta["cfg"]
    if cfg is None:
        return None
    rw = cfg["vote_rank_weights"]
    return L.PolicyConfig(mode=cfg["mode"], drop_count=cfg["drop_count"],
                          confidence_threshold=cfg["confidence_threshold"],
                          sample_threshold=cfg["sample_threshold"], min_experts=cfg["min_experts"],
                          freq_keep_budget=cfg["freq_keep_budget"], confidence_metric=cfg["confidence_metric"],
                          vote_rank_weights=None if rw is None else tuple(rw))


def _np(t):
    return t.detach().cpu().numpy()


def close(a, b):
    return np.allclose(a, b, rtol=1e-12, atol=1e-15)


def test_golden_through_mirror_api(selection_golden):
    """route_batch + apply_policy exactly as the reference's callers use them."""
    for i, c in enumerate(selection_golden):
        meta = c["meta"]
        tag = (i, meta["tag"])
        phase = L.Phase.DECODE if meta["phase"] == "decode" else L.Phase.PREFILL
        sel = L.route_batch(L.RoutingLogits(0, phase, c["logits"]), meta["k"])
        assert np.array_equal(_np(sel.expert_ids), c["expert_ids"]), tag
        assert close(_np(sel.probs), c["probs"]), tag
        if "full_probs" in c:
            assert close(_np(sel.full_probs), c["full_probs"]), tag
        cfg = _policy(meta)
        mask = L.full_retain_mask(sel, 0, phase) if cfg is None else L.apply_policy(sel, phase, cfg)
        metric = cfg.confidence_metric if cfg is not None else "top1"
        assert close(_np(sel.confidence(metric)), c["conf"]), tag
        keep = np.zeros(c["retained"].shape, dtype=np.uint8)
        keep[_np(mask.retained)] = 1
        assert np.array_equal(keep, c["retained"]), tag
        assert np.array_equal(_np(mask.remap_assigned), c["assigned"]), tag
        assert close(_np(mask.remap_weights), c["weights"]), tag
        assert bool(mask.clipped) == bool(c["clipped"]), tag
        imp = np.zeros(c["important"].shape, dtype=np.uint8)
        if mask.important_tokens is not None:
            imp[_np(mask.important_tokens)] = 1
        assert np.array_equal(imp, c["important"]), tag


def test_golden_through_c_abi_single_launch(selection_golden):
    """lynx_route_select: logits -> softmax/top-k/policy/remap in ONE kernel launch."""
    lib = nat.lib()
    for i, c in enumerate(selection_golden):
        meta = c["meta"]
        tag = (i, meta["tag"])
        z = torch.from_numpy(c["logits"]).cuda()
        T, N = z.shape
        k = meta["k"]
        out = {n: torch.zeros(s, dtype=dt, device="cuda") for n, s, dt in [
            ("ids", (T, k), torch.int32), ("probs", (T, k), torch.float64), ("full", (T, N), torch.float64),
            ("conf", (T,), torch.float64), ("counts", (N,), torch.float64), ("ret", (N,), torch.uint8),
            ("asg", (T, k), torch.int32), ("w", (T, k), torch.float64), ("imp", (T,), torch.uint8),
            ("flags", (1,), torch.int32)]}
        sel = nat.LynxSelection(expert_ids=out["ids"].data_ptr(), probs=out["probs"].data_ptr(),
                                full_probs=out["full"].data_ptr(), conf=out["conf"].data_ptr(),
                                counts=out["counts"].data_ptr(), retained=out["ret"].data_ptr(),
                                assigned=out["asg"].data_ptr(), weights=out["w"].data_ptr(),
                                important=out["imp"].data_ptr(), flags=out["flags"].data_ptr())
        cfg = _policy(meta)
        pol = None if cfg is None else ctypes.cast(ctypes.pointer(cfg.to_native()), ctypes.c_void_p)
        st = lib.lynx_route_select(z.data_ptr(), T, N, k, 1 if meta["phase"] == "decode" else 0, pol,
                                   ctypes.cast(ctypes.pointer(sel), ctypes.c_void_p),
                                   torch.cuda.current_stream().cuda_stream)
        assert st == 0, (tag, st)
        torch.cuda.synchronize()
        assert np.array_equal(_np(out["ids"]), c["expert_ids"]), tag
        assert np.array_equal(_np(out["ret"]), c["retained"]), tag
        assert np.array_equal(_np(out["asg"]), c["assigned"]), tag
        assert close(_np(out["w"]), c["weights"]), tag
        assert np.array_equal(_np(out["imp"]), c["important"]), tag
        assert bool(_np(out["flags"])[0] & nat.FLAG_CLIPPED) == bool(c["clipped"]), tag
        assert np.array_equal(_np(out["counts"]), c["counts"]), tag


def _c_abi_select(c):
    meta = c["meta"]
    z = torch.from_numpy(c["logits"]).cuda()
    T, N = z.shape
    k = meta["k"]
    out = {n: torch.zeros(s, dtype=dt, device="cuda") for n, s, dt in [
        ("ids", (T, k), torch.int32), ("probs", (T, k), torch.float64), ("full", (T, N), torch.float64),
        ("conf", (T,), torch.float64), ("counts", (N,), torch.float64), ("ret", (N,), torch.uint8),
        ("asg", (T, k), torch.int32), ("w", (T, k), torch.float64), ("imp", (T,), torch.uint8),
        ("flags", (1,), torch.int32)]}
    sel = nat.LynxSelection(expert_ids=out["ids"].data_ptr(), probs=out["probs"].data_ptr(),
                            full_probs=out["full"].data_ptr(), conf=out["conf"].data_ptr(),
                            counts=out["counts"].data_ptr(), retained=out["ret"].data_ptr(),
                            assigned=out["asg"].data_ptr(), weights=out["w"].data_ptr(),
                            important=out["imp"].data_ptr(), flags=out["flags"].data_ptr())
    cfg = _policy(meta)
    pol = None if cfg is None else ctypes.cast(ctypes.pointer(cfg.to_native()), ctypes.c_void_p)
    st = nat.lib().lynx_route_select(z.data_ptr(), T, N, k, 1 if meta["phase"] == "decode" else 0, pol,
                                     ctypes.cast(ctypes.pointer(sel), ctypes.c_void_p),
                                     torch.cuda.current_stream().cuda_stream)
    assert st == 0, st
    torch.cuda.synchronize()
    return {n: _np(t) for n, t in out.items()}


def test_neartie64_golden_bit_exact(neartie64_golden):
    """Float64-ulp near-ties (top-2, k/k+1 boundary, random) at the C2/C5/C4
    routing shapes: the reference's order depends on the last bit of
    e / e.sum() (router.py:152-154, 181).  Every output -- ids, probabilities,
    the full softmax, confidences, the policy's decisions and the remap
    weights -- equals the reference's bit for bit, through the C ABI (one
    launch) and through the mirror API."""
    assert len(neartie64_golden) == 60
    for i, c in enumerate(neartie64_golden):
        meta = c["meta"]
        tag = (i, meta["tag"])
        o = _c_abi_select(c)
        assert np.array_equal(o["ids"], c["expert_ids"]), tag
        assert np.array_equal(o["probs"], c["probs"]), tag
        assert np.array_equal(o["full"], c["full_probs"]), tag
        assert np.array_equal(o["ret"], c["retained"]), tag
        assert np.array_equal(o["asg"], c["assigned"]), tag
        assert np.array_equal(o["w"], c["weights"]), tag
        assert np.array_equal(o["imp"], c["important"]), tag
        assert bool(o["flags"][0] & nat.FLAG_CLIPPED) == bool(c["clipped"]), tag
        assert np.array_equal(o["counts"], c["counts"]), tag
        cfg = _policy(meta)
        metric = cfg.confidence_metric if cfg is not None else "top1"
        if cfg is not None:
            assert np.array_equal(o["conf"], c["conf"]), tag
        sel = L.route_batch(L.RoutingLogits(0, L.Phase.DECODE, c["logits"]), meta["k"])
        assert np.array_equal(_np(sel.expert_ids), c["expert_ids"]), tag
        assert np.array_equal(_np(sel.full_probs), c["full_probs"]), tag
        assert np.array_equal(_np(sel.confidence(metric)), c["conf"]), tag
        mask = L.full_retain_mask(sel, 0, L.Phase.DECODE) if cfg is None else L.apply_policy(sel, L.Phase.DECODE, cfg)
        assert np.array_equal(_np(mask.remap_assigned), c["assigned"]), tag
        assert np.array_equal(_np(mask.remap_weights), c["weights"]), tag


def test_golden_probabilities_bit_exact(selection_golden):
    """The 333 reference selection cases: the float64 softmax, top-k
    probabilities and remap weights carry the reference's exact bits."""
    for i, c in enumerate(selection_golden):
        tag = (i, c["meta"]["tag"])
        o = _c_abi_select(c)
        assert np.array_equal(o["probs"], c["probs"]), tag
        if "full_probs" in c:
            assert np.array_equal(o["full"], c["full_probs"]), tag
        assert np.array_equal(o["w"], c["weights"]), tag


@pytest.mark.parametrize("T,N,k", [(2000, 64, 6), (2000, 8, 2), (40, 64, 6)])
def test_deny_rank_selection_scores_confidence_on_full_row(T, N, k):
    """apply_policy on a selection whose rank 0 is NOT the row's arg-max (the
    reference's deny_expert_rank intervention, simulator.py:183-213): the
    confidence is the full row's max / top-2 margin (router.py:125-138), so
    the accuracy policy's important tokens follow the oracle.  T=2000 or
    N=64 run K1's group path on a given selection."""
    rng = np.random.default_rng(T + N)
    z = rng.normal(0, 2.0, size=(T, N))
    ids, probs, full = O.route(z, k)
    den = ids.copy()  # deny rank 0: best unselected expert, slots re-sorted by (p desc, id asc)
    for t in range(T):
        chosen = set(int(e) for e in den[t])
        order = sorted(range(N), key=lambda e: (-full[t, e], e))
        den[t, 0] = next(e for e in order if e not in chosen)
        p = full[t, den[t]]
        den[t] = den[t][np.lexsort((den[t], -p))]
    dprobs = np.take_along_axis(full, den, axis=1)
    sel = L.ExpertSelection(expert_ids=den, probs=dprobs, full_probs=full)
    for metric in ("top1", "margin"):
        assert close(_np(sel.confidence(metric)), O.confidence(full, metric))
        pol = O.Policy(mode="accuracy", confidence_threshold=0.3 if metric == "top1" else 0.1, sample_threshold=8,
                       freq_keep_budget=max(1, N // 4), confidence_metric=metric)
        m = O.apply(den, dprobs, full, pol)
        cfg = L.PolicyConfig(mode="accuracy", confidence_threshold=pol.confidence_threshold, sample_threshold=8,
                             freq_keep_budget=pol.freq_keep_budget, confidence_metric=metric)
        mask = L.apply_policy(sel, L.Phase.DECODE, cfg)
        assert np.array_equal(_np(mask.important_tokens), m.important), metric
        assert np.array_equal(_np(mask.retained), m.retained), metric
        assert np.array_equal(_np(mask.remap_assigned), m.assigned), metric
        assert close(_np(mask.remap_weights), m.weights), metric


def test_remap_golden(remap_golden):
    for i, c in enumerate(remap_golden):
        ids = c["ids"].astype(np.int64)
        full = c["full"]
        sel = L.ExpertSelection(expert_ids=ids, probs=np.take_along_axis(full, ids, axis=1), full_probs=full)
        _, assigned, w = L.remap_tokens(sel, c["keep"])
        assert np.array_equal(_np(assigned), c["assigned"]), i
        assert close(_np(w), c["weights"]), i


@pytest.mark.parametrize("shape", [(16, 8, 2), (32, 8, 2), (128, 64, 6), (256, 8, 2), (1000, 16, 4),
                                   # group path (16 < N <= 64): partial warps, several passes, odd N
                                   (1, 17, 1), (3, 20, 3), (130, 33, 5), (64, 64, 8), (300, 48, 4),
                                   # rows too large to stage in shared memory (global working arrays)
                                   (4096, 8, 2), (2000, 64, 6)])
def test_random_sweep_vs_oracle(shape):
    """Seeded sweeps at the BASELINE shapes (fp32-valued logits as K0 produces)."""
    T, N, k = shape
    rng = np.random.default_rng(T * 131 + N)
    for rep in range(6):
        z = rng.normal(0, 2.0, size=(T, N)).astype(np.float32).astype(np.float64)
        if rep % 3 == 2:
            z = np.round(z * 2) / 2  # exact ties
        for pol in (O.Policy(mode="latency", drop_count=int(rng.integers(0, N))),
                    O.Policy(mode="accuracy", confidence_threshold=0.3, sample_threshold=8,
                             freq_keep_budget=max(1, N // 4))):
            ids, probs, full = O.route(z, k)
            m = O.apply(ids, probs, full, pol)
            cfg = L.PolicyConfig(mode=pol.mode, drop_count=pol.drop_count,
                                 confidence_threshold=pol.confidence_threshold,
                                 sample_threshold=pol.sample_threshold, freq_keep_budget=pol.freq_keep_budget)
            sel = L.route_batch(L.RoutingLogits(0, L.Phase.DECODE, z), k)
            mask = L.apply_policy(sel, L.Phase.DECODE, cfg)
            assert np.array_equal(_np(sel.expert_ids), ids)
            assert np.array_equal(_np(mask.retained), m.retained)
            assert np.array_equal(_np(mask.remap_assigned), m.assigned)
            assert close(_np(mask.remap_weights), m.weights)


class TestRouterKnownAnswers:
    """test_router.py:73-233 through the GPU mirror."""

    def test_two_logit_case(self):
        p = _np(L.softmax_probs(np.array([[np.log(2.0), 0.0]])))
        assert abs(p[0, 0] - 2 / 3) < 1e-12 and abs(p[0, 1] - 1 / 3) < 1e-12

    def test_tie_prefers_smaller_index(self):
        ids, probs = L.top_k_select(np.array([0.1, 0.4, 0.4, 0.1]), 2)
        assert _np(ids).tolist() == [1, 2]
        assert _np(probs).tolist() == [0.4, 0.4]

    def test_margin_metric(self):
        sel = L.route_batch(L.RoutingLogits(0, L.Phase.DECODE, [[np.log(8.0), np.log(2.0), 0.0]]), 2)
        assert abs(_np(sel.confidence("top1"))[0] - 8 / 11) < 1e-12
        assert abs(_np(sel.confidence("margin"))[0] - 6 / 11) < 1e-12

    def test_rejects_nonfinite_device_logits(self):
        z = torch.tensor([[0.0, float("nan")]], dtype=torch.float64, device="cuda")
        with pytest.raises(L.ValidationError):
            L.route_batch(L.RoutingLogits(0, L.Phase.DECODE, z), 1)

    def test_rejects_nonfinite_host_logits(self):
        with pytest.raises(L.ValidationError):
            L.RoutingLogits(0, L.Phase.DECODE, np.array([[0.0, np.inf]]))

    def test_k_out_of_range(self):
        with pytest.raises(L.ValidationError):
            L.route_batch(L.RoutingLogits(0, L.Phase.DECODE, np.zeros((2, 4))), 5)

    def test_min_experts_below_top_k_rejected(self):
        sel = L.route_batch(L.RoutingLogits(0, L.Phase.DECODE, np.random.default_rng(0).normal(size=(4, 8))), 3)
        with pytest.raises(L.ValidationError):
            L.latency_policy(sel, L.Phase.DECODE, L.PolicyConfig(mode="latency", drop_count=2, min_experts=2))

    def test_votes(self):
        ids = np.array([[0, 1], [0, 2]])
        z = np.zeros((2, 4))
        for t in range(2):
            for r in range(2):
                z[t, ids[t, r]] = 2.0 * (2 - r)
        sel = L.route_batch(L.RoutingLogits(0, L.Phase.DECODE, z), 2)
        assert _np(L.vote_expert_frequencies(sel).counts).tolist() == [2, 1, 1, 0]
        assert _np(L.vote_expert_frequencies(sel, rank_weights=(1.0, 0.5)).counts).tolist() == [2.0, 0.5, 0.5, 0.0]


def test_bitwise_deterministic():
    z = np.random.default_rng(5).normal(0, 2, size=(64, 8))
    a = L.route_batch(L.RoutingLogits(0, L.Phase.DECODE, z), 2)
    b = L.route_batch(L.RoutingLogits(0, L.Phase.DECODE, z.copy()), 2)
    assert torch.equal(a.expert_ids, b.expert_ids) and torch.equal(a.full_probs, b.full_probs)
