"""The oracle's restatement of simulate() (attention stand-in, KV cache,
decode loop; simulator.py:273-357) pinned to the reference's own outputs
(tests/golden/simulate.npz, made by tests/golden/make_golden_simulate.py):
every routing event bit-exact, hidden states to f64 round-off."""

from __future__ import annotations

import numpy as np

from conftest import load_simulate_golden
from oracle import lynx_oracle as O


def _policy(p):
    if p is None:
        return None
    return O.Policy(mode=p["mode"], drop_count=p["drop_count"], confidence_threshold=p["confidence_threshold"],
                    sample_threshold=p["sample_threshold"], min_experts=p["min_experts"],
                    freq_keep_budget=p["freq_keep_budget"], confidence_metric=p["confidence_metric"],
                    vote_rank_weights=p["vote_rank_weights"])


def test_oracle_simulate_matches_reference():
    meta, w, x, cases = load_simulate_golden()
    L, k = meta["L"], meta["k"]
    attn = [(w["q"][l], w["k"][l], w["v"][l], w["o"][l]) for l in range(L)]
    for case in cases:
        pol = _policy(case["policy"])
        events = []

        def moe(l, phase, flat):
            ids, probs, full = O.route(O.router_logits(flat, w["router"][l]), k)
            if pol is None:
                m = O.identity_mask(ids, probs, full.shape[1])
            else:
                m = O.apply(ids, probs, full, pol, decode=phase == "decode")
            events.append((ids, m))
            return O.forward_tanh2(flat, w["1"][l], w["2"][l], m.assigned, m.weights)

        hidden = O.simulate(x, meta["steps"], L, attn, moe)
        assert len(events) == len(case["events"]), case["name"]
        for (ids, m), ref in zip(events, case["events"]):
            assert np.array_equal(ids, ref["ids"]), (case["name"], ref["event"], ref["layer"])
            assert np.array_equal(m.assigned, ref["assigned"]), (case["name"], ref["event"], ref["layer"])
            assert np.array_equal(np.asarray(m.retained), ref["retained"])
            assert np.allclose(m.weights, ref["weights"], rtol=1e-12, atol=1e-15)
        assert np.allclose(hidden, case["hidden"], rtol=1e-9, atol=1e-9), case["name"]
