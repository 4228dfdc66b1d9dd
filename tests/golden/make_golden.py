"""Generate golden fixtures for the Lynx hot path from the REFERENCE itself.

Run in the build container (the reference is importable only here):

    PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=/root/reference/pkg/src \
        python tests/golden/make_golden.py

It imports ``moetrim`` (the reference, /root/reference/pkg/src/moetrim),
drives its hot-path API -- route_batch (router.py:174), apply_policy
(policy.py:341), remap_tokens (policy.py:151), full_retain_mask
(policy.py:215), forward_layer (simulator.py:86) -- on seeded inputs, and
stores inputs + outputs under tests/golden/*.npz.  The fixtures travel
with the repo; nothing at test time reads /root/reference.

Cases:
  selection.npz  -- logits -> (ids, probs, conf, counts, retained,
                    assigned, weights, important, clipped) for router
                    known-answer rows (test_router.py) and seeded sweeps
                    over the BASELINE shapes (C1 16x8 k2, C2 32x8 k2,
                    C4 128x64 k6, C5 256x8 k2) and random small shapes,
                    both policies, both phases, ties / near-ties /
                    clustered logits.
  selection_neartie64.npz -- float64-ulp near-ties (top-2, k/k+1 boundary,
                    random) at the C2/C5/C4 routing shapes, both policies.
  remap.npz      -- remap_tokens on arbitrary retained sets incl. collapse.
  forward.npz    -- forward_layer (tanh2 reference expert) outputs, plus
                    the per-expert dispatch order and merged weights
                    recovered by instrumenting expert_mlp.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

import moetrim
from moetrim import simulator as sim
from moetrim.policy import ExpertMask, PolicyConfig, apply_policy, full_retain_mask, remap_tokens
from moetrim.router import ExpertSelection, MoEModelSpec, Phase, RoutingLogits, route_batch

HERE = os.path.dirname(os.path.abspath(__file__))


def pack_cfg(cfg: PolicyConfig | None) -> dict | None:
    if cfg is None:
        return None
    return dict(mode=cfg.mode, drop_count=cfg.drop_count,
                confidence_threshold=cfg.confidence_threshold,
                sample_threshold=cfg.sample_threshold, min_experts=cfg.min_experts,
                freq_keep_budget=cfg.freq_keep_budget,
                confidence_metric=cfg.confidence_metric,
                vote_rank_weights=None if cfg.vote_rank_weights is None
                else list(cfg.vote_rank_weights))


def logits_kind(rng, kind, T, N):
    if kind == "normal1":
        return rng.normal(0.0, 1.0, size=(T, N))
    if kind == "normal2":
        return rng.normal(0.0, 2.0, size=(T, N))
    if kind == "normal5":
        return rng.normal(0.0, 5.0, size=(T, N))
    if kind == "fp32":  # what the CUDA router GEMV produces
        return rng.normal(0.0, 2.0, size=(T, N)).astype(np.float32).astype(np.float64)
    if kind == "ties":  # exact ties within rows and duplicated rows
        z = np.round(rng.normal(0.0, 1.5, size=(T, N)) * 2.0) / 2.0
        if T > 2:
            z[T // 2] = z[0]
        return z
    if kind == "neartie":  # fp32-ulp near ties
        z = rng.normal(0.0, 2.0, size=(T, N)).astype(np.float32)
        for t in range(T):
            a, b = rng.choice(N, size=2, replace=False) if N > 1 else (0, 0)
            z[t, b] = np.nextafter(z[t, a], np.float32(np.inf if rng.random() < .5 else -np.inf))
        return z.astype(np.float64)
    if kind == "clustered":  # workloads.py:79-84 recipe
        z = rng.normal(0.0, 1.0, size=(T, N))
        hot = rng.choice(N, size=min(2, N), replace=False)
        z[:, hot] += 2.0
        return z
    if kind == "peaked":  # many confident tokens (accuracy policy truncation)
        z = rng.normal(0.0, 1.0, size=(T, N))
        z[np.arange(T), rng.integers(0, N, size=T)] += 6.0
        return z
    raise ValueError(kind)


def run_selection(z, k, cfg, phase):
    sel = route_batch(RoutingLogits(layer_index=0, phase=phase, values=z), k)
    if cfg is None:
        mask = full_retain_mask(sel, 0, phase)
    else:
        mask = apply_policy(sel, phase, cfg, 0)
    N = z.shape[1]
    metric = cfg.confidence_metric if cfg is not None else "top1"
    if cfg is not None and phase is Phase.DECODE:
        if cfg.mode == "latency":
            counts = moetrim.vote_expert_frequencies(sel, cfg.vote_rank_weights).counts
        else:
            sub = ExpertSelection(expert_ids=sel.expert_ids[mask.important_tokens],
                                  probs=sel.probs[mask.important_tokens],
                                  full_probs=sel.full_probs[mask.important_tokens])
            counts = moetrim.vote_expert_frequencies(sub, cfg.vote_rank_weights).counts
    else:
        counts = np.zeros(N)
    retained = np.zeros(N, dtype=np.uint8)
    retained[mask.retained] = 1
    important = np.zeros(z.shape[0], dtype=np.uint8)
    if mask.important_tokens is not None:
        important[mask.important_tokens] = 1
    return dict(
        logits=z, expert_ids=sel.expert_ids.astype(np.int16), probs=sel.probs,
        full_probs=sel.full_probs, conf=sel.confidence(metric), counts=counts,
        retained=retained, assigned=mask.remap_assigned.astype(np.int16),
        weights=mask.remap_weights, important=important,
        clipped=np.array(bool(mask.clipped)),
    )


def selection_cases():
    rng = np.random.default_rng(20241114)
    cases = []

    def add(z, k, cfg, phase, tag, keep_full=True):
        out = run_selection(np.asarray(z, dtype=np.float64), k, cfg, phase)
        if not keep_full:
            out.pop("full_probs")
        cases.append((dict(k=k, cfg=pack_cfg(cfg), phase=phase.value, tag=tag), out))

    # Router known-answer rows (test_router.py:73-233) as routing-only cases.
    ln = np.log
    known = [
        ([[ln(2.0), 0.0]], 1), ([[4.2] * 8] * 3, 2), ([[0.0, 0.0]], 1),
        ([[30.0, -30.0, -30.0, -30.0], [-30.0, -30.0, -30.0, 30.0]], 1),
        ([[1.0, -0.5, 2.0, 0.0]] * 3, 2), ([[ln(8.0), 0.0, 0.0]], 1),
        ([[0.0] * 8], 2), ([[ln(8.0), ln(2.0), 0.0]], 2),
        ([[1e8, 1e8 - 3.0, 0.0], [-1e8, -1e8 + 1.0, -1e8 + 2.0]], 2),
        (np.log(np.array([[0.1, 0.4, 0.4, 0.1]])), 2),
        (np.log(np.array([[0.05, 0.5, 0.2, 0.25]])), 2),
        ([[0.5, 0.5, 0.5, 0.5]], 4),
    ]
    for rows, k in known:
        add(rows, k, None, Phase.DECODE, "router-known")
        add(rows, k, PolicyConfig(mode="latency", drop_count=1), Phase.DECODE, "router-known-lat")
        add(rows, k, PolicyConfig(mode="accuracy", freq_keep_budget=1,
                                  min_experts=max(k, 1)), Phase.DECODE, "router-known-acc")
        add(rows, k, PolicyConfig(mode="accuracy", confidence_metric="margin"),
            Phase.DECODE, "router-known-acc-margin")

    # Policy known-answer selections (test_policy.py) built like conftest's selection_from_ids.
    def from_ids(ids, N):
        ids = np.asarray(ids)
        z = np.zeros((ids.shape[0], N))
        for t in range(ids.shape[0]):
            for r in range(ids.shape[1]):
                z[t, ids[t, r]] = 2.0 * (ids.shape[1] - r)
        return z

    add(from_ids([[0, 1], [1, 2], [2, 3]], 4), 2, PolicyConfig(mode="latency", drop_count=1),
        Phase.DECODE, "policy-known")
    add(from_ids([[e, (e + 1) % 8] for e in range(8)], 8), 2,
        PolicyConfig(mode="latency", drop_count=2), Phase.DECODE, "policy-known")
    add(from_ids([[0, 1], [1, 2]], 4), 2, PolicyConfig(mode="latency", drop_count=3),
        Phase.PREFILL, "policy-known")
    add(from_ids([[0, 1], [0, 2]], 4), 2, PolicyConfig(mode="latency", drop_count=1,
        vote_rank_weights=(1.0, 0.5)), Phase.DECODE, "policy-known-rankw")
    add(from_ids([[0], [1], [2]], 4), 1, PolicyConfig(mode="accuracy", freq_keep_budget=1,
        min_experts=1), Phase.DECODE, "policy-known")
    add(from_ids([[0], [1], [2]], 8), 1, PolicyConfig(mode="accuracy", freq_keep_budget=6,
        min_experts=1), Phase.DECODE, "policy-known")
    add(from_ids([[2, 0]], 8), 2, PolicyConfig(mode="accuracy", freq_keep_budget=1,
        min_experts=4), Phase.DECODE, "policy-known")
    add(from_ids([[0, 1]] * 12, 8), 2, PolicyConfig(mode="accuracy", freq_keep_budget=4,
        confidence_threshold=0.0), Phase.DECODE, "policy-known")
    add(from_ids([[e % 8, (e + 3) % 8] for e in range(12)], 8), 2,
        PolicyConfig(mode="accuracy", freq_keep_budget=4, confidence_threshold=0.0),
        Phase.DECODE, "policy-known")
    z = np.zeros((12, 4)); z[:, 0] = 3.0 + 0.01 * np.arange(12)[::-1]
    add(z, 2, PolicyConfig(mode="accuracy", sample_threshold=8), Phase.DECODE, "important-truncate")
    z = np.zeros((3, 4)); z[1, 0] = 0.2
    add(z, 2, PolicyConfig(mode="accuracy"), Phase.DECODE, "important-argmax")
    z = np.array([[2.0, 1.9, -8.0, -8.0], [1.0, -4.0, -4.0, -4.0]])
    add(z, 2, PolicyConfig(mode="accuracy", confidence_threshold=0.45), Phase.DECODE, "margin")
    add(z, 2, PolicyConfig(mode="accuracy", confidence_threshold=0.45,
                           confidence_metric="margin"), Phase.DECODE, "margin")

    # Seeded sweeps at the BASELINE shapes.
    shapes = [(16, 8, 2), (32, 8, 2), (128, 64, 6), (256, 8, 2), (64, 8, 2), (8, 8, 2)]
    kinds = ["normal1", "normal2", "fp32", "ties", "neartie", "clustered", "peaked"]
    for (T, N, k) in shapes:
        big = T * N > 4096
        reps = 3 if big else 10
        for rep in range(reps):
            kind = kinds[rep % len(kinds)] if not big else ["normal2", "fp32", "clustered"][rep]
            z = logits_kind(rng, kind, T, N)
            drop = int(rng.integers(0, N + 2))
            add(z, k, PolicyConfig(mode="latency", drop_count=drop), Phase.DECODE,
                f"sweep-{T}x{N}-lat-{kind}", keep_full=not big)
            add(z, k, PolicyConfig(mode="accuracy", confidence_threshold=float(rng.choice([0.1, 0.3, 0.5])),
                                   sample_threshold=int(rng.choice([4, 8, 12])),
                                   freq_keep_budget=int(rng.choice([1, 2, 4, N // 2 or 1])),
                                   confidence_metric=str(rng.choice(["top1", "margin"]))),
                Phase.DECODE, f"sweep-{T}x{N}-acc-{kind}", keep_full=not big)
        add(logits_kind(rng, "normal2", T, N), k, PolicyConfig(mode="latency", drop_count=4),
            Phase.PREFILL, f"sweep-{T}x{N}-prefill", keep_full=not big)

    # Random small shapes, policy invariants style (test_acceptance.py:97-136).
    for rep in range(160):
        T = int(rng.integers(1, 13))
        N = int(rng.integers(2, 17))
        k = int(rng.integers(1, min(4, N) + 1))
        kind = kinds[rep % len(kinds)]
        z = logits_kind(rng, kind, T, N)
        if rng.random() < 0.5:
            mk = None if rng.random() < 0.7 else int(rng.integers(k, N + 1))
            rw = None if rng.random() < 0.8 else tuple(float(x) for x in rng.uniform(0, 1, size=k))
            cfg = PolicyConfig(mode="latency", drop_count=int(rng.integers(0, N + 2)),
                               min_experts=mk, vote_rank_weights=rw)
        else:
            rw = None if rng.random() < 0.8 else tuple(float(x) for x in rng.uniform(0, 1, size=k))
            cfg = PolicyConfig(mode="accuracy", confidence_threshold=float(rng.uniform(0.05, 0.9)),
                               sample_threshold=int(rng.integers(1, 12)),
                               freq_keep_budget=int(rng.integers(1, N + 1)),
                               min_experts=None if rng.random() < 0.7 else int(rng.integers(k, N + 1)),
                               confidence_metric="top1" if rng.random() < 0.7 else "margin",
                               vote_rank_weights=rw)
        phase = Phase.DECODE if rng.random() < 0.85 else Phase.PREFILL
        add(z, k, cfg, phase, f"random-{kind}")
    return cases


def neartie64_cases():
    """Float64-ulp near-ties at the BASELINE routing shapes (own RNG, so the
    other fixtures are unchanged).  Logits one or a few float64 ulps apart --
    at the row max, at the k / k+1 boundary and in random places -- make the
    reference's order depend on the last bit of e / e.sum() (router.py:152-154,
    181), so a device softmax that differs from numpy by one ulp anywhere
    (exp, the row sum, the division) flips ids here."""
    rng = np.random.default_rng(64064)
    cases = []

    def nudge(x, steps, up):
        for _ in range(steps):
            x = np.nextafter(x, np.inf if up else -np.inf)
        return x

    def make(T, N, k, where):
        z = rng.normal(0.0, 2.0, size=(T, N))
        for t in range(T):
            order = np.argsort(-z[t], kind="stable")
            if where == "top":
                a, b = order[0], order[1]
            elif where == "boundary":
                a, b = order[k - 1], order[min(k, N - 1)]
            else:
                a, b = rng.choice(N, size=2, replace=False)
            z[t, b] = nudge(z[t, a], int(rng.integers(0, 3)), bool(rng.random() < 0.5))
            if rng.random() < 0.3 and N > 2:  # a third expert in the same ulp cluster
                c = [e for e in range(N) if e not in (a, b)][int(rng.integers(0, N - 2))]
                z[t, c] = nudge(z[t, a], int(rng.integers(1, 3)), bool(rng.random() < 0.5))
        return z

    shapes = [(32, 8, 2), (256, 8, 2), (64, 8, 2), (16, 16, 4), (128, 64, 6)]
    for (T, N, k) in shapes:
        for where in ("top", "boundary", "random"):
            z = make(T, N, k, where)
            tag = f"neartie64-{T}x{N}-{where}"
            cfgs = [PolicyConfig(mode="latency", drop_count=N // 2),
                    PolicyConfig(mode="accuracy", confidence_threshold=0.3, freq_keep_budget=max(1, N // 4),
                                 confidence_metric="margin"),
                    PolicyConfig(mode="accuracy", confidence_threshold=0.5, freq_keep_budget=max(1, N // 4))]
            for cfg in cfgs:
                out = run_selection(z, k, cfg, Phase.DECODE)
                cases.append((dict(k=k, cfg=pack_cfg(cfg), phase=Phase.DECODE.value, tag=tag), out))
            out = run_selection(z, k, None, Phase.DECODE)
            cases.append((dict(k=k, cfg=None, phase=Phase.DECODE.value, tag=tag + "-identity"), out))
    return cases


def remap_cases():
    rng = np.random.default_rng(77)
    cases = []
    full = np.array([[0.05, 0.3, 0.05, 0.6]]); ids = np.array([[3, 1]])
    cases.append((full, ids, np.array([1, 2])))
    full = np.array([[0.1, 0.2, 0.3, 0.4]]); ids = np.array([[3, 2]])
    cases.append((full, ids, np.array([0])))  # collapse
    for rep in range(60):
        T = int(rng.integers(1, 9)); N = int(rng.integers(2, 9)); k = int(rng.integers(1, min(4, N) + 1))
        sel = route_batch(RoutingLogits(0, Phase.DECODE, rng.normal(0, 2.0, size=(T, N))), k)
        R = int(rng.integers(1, N + 1))
        keep = np.sort(rng.choice(N, size=R, replace=False))
        cases.append((sel.full_probs, sel.expert_ids, keep))
    out = []
    for full, ids, keep in cases:
        sel = ExpertSelection(expert_ids=ids, probs=np.take_along_axis(full, ids, axis=1), full_probs=full)
        orig, assigned, weights = remap_tokens(sel, keep)
        out.append(dict(full=full, ids=ids.astype(np.int16), keep=keep.astype(np.int16),
                        assigned=assigned.astype(np.int16), weights=weights))
    return out


def forward_cases():
    """forward_layer with the reference tanh2 expert + instrumented dispatch."""
    rng = np.random.default_rng(99)
    out = []
    specs = [(4, 2, 16, 32), (8, 2, 32, 64), (8, 2, 32, 64), (4, 1, 8, 16), (8, 3, 16, 32)]
    for i, (N, k, d, ff) in enumerate(specs):
        spec = MoEModelSpec(num_layers=1, num_experts=N, top_k=k, d_model=d, d_ff=ff)
        model = sim.build_model(spec, seed=100 + i)
        T = [16, 16, 32, 5, 12][i]
        hidden = rng.normal(0.0, 1.0, size=(T, d))
        logits = sim.router_logits(model, 0, hidden)
        sel = route_batch(RoutingLogits(0, Phase.DECODE, logits), k)
        cfg = [PolicyConfig(mode="latency", drop_count=4), PolicyConfig(mode="latency", drop_count=4),
               PolicyConfig(mode="accuracy"), None, PolicyConfig(mode="latency", drop_count=2)][i]
        mask = full_retain_mask(sel, 0, Phase.DECODE) if cfg is None else apply_policy(sel, Phase.DECODE, cfg)
        y = sim.forward_layer(hidden, model, 0, mask)
        # Instrumented dispatch: each expert writes a one-hot column so the
        # merged per-row weight is recovered exactly; the token id rides in
        # the last column of the probe input.
        probe = np.zeros((T, N + 1)); probe[:, N] = np.arange(T)
        calls = []
        real = sim.expert_mlp
        def fake(model_, layer, e, x, _calls=calls, _N=N):
            _calls.append((e, x[:, _N].astype(np.int64).tolist()))
            o = np.zeros((x.shape[0], _N + 1)); o[:, e] = 1.0
            return o
        sim.expert_mlp = fake
        try:
            probe_out = sim.forward_layer(probe, model, 0, mask)
        finally:
            sim.expert_mlp = real
        order = np.array([e for e, _ in calls], dtype=np.int16)
        rows = np.full((len(calls), T), -1, dtype=np.int16)
        for j, (_, r) in enumerate(calls):
            rows[j, :len(r)] = r
        out.append(dict(hidden=hidden, router_w=model.router_w[0], w1=model.w1[0], w2=model.w2[0],
                        logits=logits, assigned=mask.remap_assigned.astype(np.int16),
                        weights=mask.remap_weights, y=y, order=order, rows=rows,
                        merged=probe_out[:, :N], k=np.array(k)))
    return out


def save(name, cases, meta=None):
    flat = {}
    for i, c in enumerate(cases):
        d = c[1] if isinstance(c, tuple) else c
        for key, v in d.items():
            flat[f"c{i}_{key}"] = np.asarray(v)
    np.savez_compressed(os.path.join(HERE, name), **flat)
    if meta is not None:
        with open(os.path.join(HERE, name.replace(".npz", ".json")), "w") as f:
            json.dump(meta, f, indent=0)


def main():
    assert moetrim.__version__ == "0.1.0", moetrim.__version__
    sel = selection_cases()
    save("selection.npz", sel, meta=dict(
        source="moetrim 0.1.0 (/root/reference/pkg/src), numpy " + np.__version__,
        cases=[m for m, _ in sel]))
    nt = neartie64_cases()
    save("selection_neartie64.npz", nt, meta=dict(
        source="moetrim 0.1.0 (/root/reference/pkg/src), numpy " + np.__version__,
        cases=[m for m, _ in nt]))
    rem = remap_cases()
    save("remap.npz", rem, meta=dict(n=len(rem)))
    fwd = forward_cases()
    save("forward.npz", fwd, meta=dict(n=len(fwd)))
    print(f"selection {len(sel)} neartie64 {len(nt)} remap {len(rem)} forward {len(fwd)}")


if __name__ == "__main__":
    sys.exit(main())
