"""Golden fixtures for the decode stack from the
REFERENCE itself: moetrim's ``simulate`` (simulator.py:273-357) with its
attention stand-in, tanh expert and a policy intervention, plus the routing
trace its ``trace_sink`` sees (trace.py records).

    PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=/root/reference/pkg/src \\
        python tests/golden/make_golden_simulate.py

The reference model's weights and inputs are rounded to bf16-representable
values first, so the GPU stack (bf16 weights) runs the same model; the
seed is chosen so that every routing decision has a probability margin the
GPU's bf16 hidden states cannot flip.  Writes tests/golden/simulate.npz
(+ .json).  Nothing at test time reads /root/reference.
"""

from __future__ import annotations

import dataclasses
import json
import os
import sys

import numpy as np

from moetrim import simulator as sim
from moetrim.policy import PolicyConfig
from moetrim.router import MoEModelSpec
from moetrim.trace import mask_record_from_event, records_from_event, write_masks_jsonl, write_trace_jsonl

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle.lynx_oracle import bf16_round  # noqa: E402

L, N, K, D_MODEL, D_FF, D_HEAD = 2, 8, 2, 32, 64, 16
B, P, STEPS = 3, 3, 3

CASES = [
    ("latency_drop3", PolicyConfig(mode="latency", drop_count=3)),
    ("accuracy_budget2", PolicyConfig(mode="accuracy", freq_keep_budget=2, confidence_threshold=0.3)),
    ("none", None),
]


def rounded_model(seed):
    m = sim.build_model(MoEModelSpec(L, N, K, D_MODEL, D_FF, 2), seed=seed, d_head=D_HEAD)
    r = lambda a: bf16_round(np.asarray(a, dtype=np.float32)).astype(np.float64)  # noqa: E731
    return dataclasses.replace(m, router_w=r(m.router_w), wq=r(m.wq), wk=r(m.wk), wv=r(m.wv), wo=r(m.wo),
                               w1=r(m.w1), w2=r(m.w2))


def run(model, x, cfg):
    events = []

    def sink(event, layer, phase, selection, mask):
        events.append((event, layer, phase, selection, mask))

    iv = None if cfg is None else sim.Intervention(kind="policy", policy=cfg)
    res = sim.simulate(model, x, STEPS, intervention=iv, trace_sink=sink)
    return res.hidden, events


def min_margin(events):
    """Smallest gap between adjacent sorted probabilities among each token's
    top k+1 (the order of the chosen ids and the top-k boundary)."""
    g = np.inf
    for _, _, _, sel, _ in events:
        s = -np.sort(-sel.full_probs, axis=1)[:, :K + 1]
        g = min(g, float(np.min(s[:, :-1] - s[:, 1:])))
    return g


def main():
    best = None
    for seed in range(2000):
        model = rounded_model(seed)
        x = bf16_round(sim.seeded_inputs(B, P, D_MODEL, seed + 1000).astype(np.float32)).astype(np.float64)
        margins = [min_margin(run(model, x, cfg)[1]) for _, cfg in CASES]
        m = min(margins)
        if best is None or m > best[0]:
            best = (m, seed)
        if m >= 0.03:
            break
    margin, seed = best
    model = rounded_model(seed)
    x = bf16_round(sim.seeded_inputs(B, P, D_MODEL, seed + 1000).astype(np.float32)).astype(np.float64)
    flat = {"w_router": model.router_w, "w_q": model.wq, "w_k": model.wk, "w_v": model.wv, "w_o": model.wo,
            "w_1": model.w1, "w_2": model.w2, "inputs": x}
    meta = {"seed": seed, "min_prob_margin": margin, "L": L, "N": N, "k": K, "d": D_MODEL, "ff": D_FF,
            "d_head": D_HEAD, "B": B, "P": P, "steps": STEPS, "cases": []}
    for ci, (name, cfg) in enumerate(CASES):
        hidden, events = run(model, x, cfg)
        flat[f"c{ci}_hidden"] = hidden
        ev_meta = []
        for ei, (event, layer, phase, sel, mask) in enumerate(events):
            flat[f"c{ci}_e{ei}_ids"] = sel.expert_ids
            flat[f"c{ci}_e{ei}_assigned"] = mask.remap_assigned
            flat[f"c{ci}_e{ei}_weights"] = mask.remap_weights
            flat[f"c{ci}_e{ei}_retained"] = np.asarray(mask.retained, dtype=np.int64)
            rec = [dataclasses.asdict(r) for r in records_from_event("golden", event, layer, phase, sel, mask)]
            mrec = dataclasses.asdict(mask_record_from_event("golden", event, layer, phase, mask))
            ev_meta.append({"event": event, "layer": layer, "phase": phase.value, "clipped": bool(mask.clipped),
                            "trace": rec, "mask": mrec})
        meta["cases"].append({"name": name, "policy": None if cfg is None else dataclasses.asdict(cfg),
                              "events": ev_meta})
    # the reference's own JSONL files for case 0 (byte-level schema check of trace.py)
    _, events = run(model, x, CASES[0][1])
    recs = [r for (e, l, ph, sel, m) in events for r in records_from_event("golden", e, l, ph, sel, m)]
    write_trace_jsonl(os.path.join(HERE, "simulate_trace.jsonl"), recs)
    write_masks_jsonl(os.path.join(HERE, "simulate_trace.masks.jsonl"),
                      [mask_record_from_event("golden", e, l, ph, m) for (e, l, ph, sel, m) in events])
    np.savez_compressed(os.path.join(HERE, "simulate.npz"), **flat)
    with open(os.path.join(HERE, "simulate.json"), "w") as f:
        json.dump(meta, f, indent=0)
    print(f"seed {seed}, min prob margin {margin:.4f}, {sum(len(c['events']) for c in meta['cases'])} events")


if __name__ == "__main__":
    main()
