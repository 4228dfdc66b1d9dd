"""Pin the CPU oracle (oracle/lynx_oracle.py) to the reference's golden vectors.

The fixtures were produced by the reference itself (tests/golden/make_golden.py);
these tests prove the restatement before any CUDA result is compared with it.
"""

from __future__ import annotations

import numpy as np
import pytest

from oracle import lynx_oracle as O


def policy_from(meta):
    cfg = meta["cfg"]
    if cfg is None:
        return None
    rw = cfg["vote_rank_weights"]
    return O.Policy(mode=cfg["mode"], drop_count=cfg["drop_count"],
                    confidence_threshold=cfg["confidence_threshold"],
                    sample_threshold=cfg["sample_threshold"], min_experts=cfg["min_experts"],
                    freq_keep_budget=cfg["freq_keep_budget"],
                    confidence_metric=cfg["confidence_metric"],
                    vote_rank_weights=None if rw is None else tuple(rw))


def oracle_select(case):
    meta = case["meta"]
    k = meta["k"]
    decode = meta["phase"] == "decode"
    ids, probs, full = O.route(case["logits"], k)
    pol = policy_from(meta)
    if pol is None:
        mask = O.identity_mask(ids, probs, full.shape[1])
    else:
        mask = O.apply(ids, probs, full, pol, decode)
    metric = pol.confidence_metric if pol is not None else "top1"
    return ids, probs, full, O.confidence(full, metric), mask


class TestPairwiseSum:
    @pytest.mark.parametrize("n", list(range(1, 140)) + [200, 256, 257, 513])
    def test_matches_numpy_bitwise(self, n):
        rng = np.random.default_rng(n)
        a = np.exp(rng.normal(0, 3, size=(4, n)))
        want = a.sum(axis=-1)
        got = np.array([O.pairwise_sum(r) for r in a])
        assert np.array_equal(want, got)
        assert O.pairwise_sum(a[0]) == a[0].sum()


class TestSelectionGolden:
    def test_case_count(self, selection_golden):
        assert len(selection_golden) > 300

    def test_all_cases(self, selection_golden):
        for i, c in enumerate(selection_golden):
            ids, probs, full, conf, mask = oracle_select(c)
            tag = (i, c["meta"]["tag"])
            assert np.array_equal(ids, c["expert_ids"]), tag
            assert np.allclose(probs, c["probs"], rtol=1e-12, atol=1e-15), tag
            if "full_probs" in c:
                assert np.allclose(full, c["full_probs"], rtol=1e-12, atol=1e-15), tag
            assert np.allclose(conf, c["conf"], rtol=1e-12, atol=1e-15), tag
            keep = np.zeros(full.shape[1], dtype=np.uint8)
            keep[mask.retained] = 1
            assert np.array_equal(keep, c["retained"]), tag
            assert np.array_equal(mask.assigned, c["assigned"]), tag
            assert np.allclose(mask.weights, c["weights"], rtol=1e-12, atol=1e-15), tag
            assert bool(mask.clipped) == bool(c["clipped"]), tag
            imp = np.zeros(full.shape[0], dtype=np.uint8)
            if mask.important is not None:
                imp[mask.important] = 1
            assert np.array_equal(imp, c["important"]), tag
            if mask.counts is not None:
                assert np.array_equal(mask.counts, c["counts"]), tag

    def test_bitwise_on_this_machine(self, selection_golden):
        """Same numpy build as the fixture generator -> exact float64 bits."""
        c = selection_golden[-1]
        _, probs, _, _, mask = oracle_select(c)
        if not np.array_equal(probs, c["probs"]):
            pytest.skip("different numpy exp build than the fixture machine")
        assert np.array_equal(mask.weights, c["weights"])


class TestNumpyExp:
    """The SVML exp restatement (oracle.svml_exp_ha, the same steps as
    csrc/npexp.cuh) against this host's np.exp, bit for bit."""

    def test_matches_numpy_bitwise(self):
        if not O.numpy_uses_svml_exp():
            pytest.skip("this numpy does not dispatch float64 exp to SVML (no AVX512_SKX)")
        rng = np.random.default_rng(7)
        xs = np.concatenate([-np.abs(rng.normal(0, 4, 4000)), -rng.uniform(0, 1e-3, 500),
                             -rng.uniform(0, 700, 500), rng.normal(0, 3, 500),
                             [0.0, -0.0, -1e-300, -5e-324, -1e-17, -np.log(2) / 16, -707.0, 700.0]])
        got = np.array([O.svml_exp_ha(x) for x in xs])
        assert np.array_equal(got, np.exp(xs))

    def test_neartie64_fixtures_bit_exact(self, neartie64_golden):
        """Float64-ulp near-ties: the oracle reproduces the reference's bits."""
        for i, c in enumerate(neartie64_golden):
            ids, probs, full, conf, mask = oracle_select(c)
            tag = (i, c["meta"]["tag"])
            if not np.array_equal(full, c["full_probs"]):
                pytest.skip("different numpy exp build than the fixture machine")
            assert np.array_equal(ids, c["expert_ids"]), tag
            assert np.array_equal(conf, c["conf"]), tag
            assert np.array_equal(mask.assigned, c["assigned"]), tag
            assert np.array_equal(mask.weights, c["weights"]), tag
            keep = np.zeros(full.shape[1], dtype=np.uint8)
            keep[mask.retained] = 1
            assert np.array_equal(keep, c["retained"]), tag


class TestRemapGolden:
    def test_all_cases(self, remap_golden):
        for i, c in enumerate(remap_golden):
            ids = c["ids"].astype(np.int64)
            _, assigned, w = O.remap(ids, c["full"], c["keep"])
            assert np.array_equal(assigned, c["assigned"]), i
            assert np.allclose(w, c["weights"], rtol=1e-12, atol=1e-15), i

    def test_collapse_case(self, remap_golden):
        c = remap_golden[1]
        assert c["assigned"].tolist() == [[0, 0]]

    def test_empty_retained_rejected(self):
        with pytest.raises(O.OracleError):
            O.remap(np.array([[0, 1]]), np.array([[0.5, 0.5]]), [])


class TestForwardGolden:
    def test_tanh2_forward_matches_reference(self, forward_golden):
        for c in forward_golden:
            y = O.forward_tanh2(c["hidden"], c["w1"][None] if c["w1"].ndim == 2 else c["w1"],
                                c["w2"], c["assigned"].astype(np.int64), c["weights"])
            assert np.allclose(y, c["y"], rtol=1e-12, atol=1e-12)

    def test_dispatch_order_and_merged_weights(self, forward_golden):
        for c in forward_golden:
            disp = O.dispatch(c["assigned"].astype(np.int64), c["weights"])
            assert disp.experts == c["order"].tolist()
            for j, (e, rows) in enumerate(zip(disp.experts, disp.rows)):
                ref_rows = [r for r in c["rows"][j].tolist() if r >= 0]
                assert rows.tolist() == ref_rows
                merged = c["merged"][:, e]
                assert np.array_equal(disp.row_weight[j], merged[rows])

    def test_router_logits(self, forward_golden):
        for c in forward_golden:
            z = O.router_logits(c["hidden"], c["router_w"])
            assert np.allclose(z, c["logits"], rtol=1e-12, atol=1e-12)


class TestSwigluOracle:
    def test_single_expert_weight_one(self, rng):
        T, d, ff = 3, 8, 16
        x = rng.normal(size=(T, d)).astype(np.float32)
        w1 = rng.normal(size=(1, ff, d)).astype(np.float32)
        w3 = rng.normal(size=(1, ff, d)).astype(np.float32)
        w2 = rng.normal(size=(1, d, ff)).astype(np.float32)
        assigned = np.zeros((T, 1), dtype=np.int64)
        w = np.ones((T, 1))
        y = O.forward_swiglu(x, w1, w3, w2, assigned, w)
        ref = x + (O.silu(x @ w1[0].T) * (x @ w3[0].T)) @ w2[0].T
        assert np.allclose(y, ref, rtol=1e-5, atol=1e-5)

    def test_bf16_round(self):
        a = np.array([1.0, 1.00390625, 1.001953125, -3.1415926], dtype=np.float32)
        r = O.bf16_round(a)
        import torch
        want = torch.from_numpy(a).to(torch.bfloat16).float().numpy()
        assert np.array_equal(r, want)
