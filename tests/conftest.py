"""Shared test plumbing.

Markers: ``gpu`` -- needs a B200 (run with ``-m gpu``); everything else
runs on CPU.  The golden fixtures under tests/golden/ were produced from
the reference itself by tests/golden/make_golden.py.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device")


def load_cases(name):
    """Return a list of dicts (one per case) from tests/golden/<name>.npz."""
    data = np.load(os.path.join(GOLDEN, name))
    cases = {}
    for key in data.files:
        idx, field = key.split("_", 1)
        cases.setdefault(int(idx[1:]), {})[field] = data[key]
    meta_path = os.path.join(GOLDEN, name.replace(".npz", ".json"))
    meta = json.load(open(meta_path)) if os.path.exists(meta_path) else {}
    out = []
    for i in sorted(cases):
        c = cases[i]
        if "cases" in meta:
            c["meta"] = meta["cases"][i]
        out.append(c)
    return out


@pytest.fixture(scope="session")
def selection_golden():
    return load_cases("selection.npz")


@pytest.fixture(scope="session")
def neartie64_golden():
    return load_cases("selection_neartie64.npz")


@pytest.fixture(scope="session")
def remap_golden():
    return load_cases("remap.npz")


@pytest.fixture(scope="session")
def forward_golden():
    return load_cases("forward.npz")


@pytest.fixture
def rng():
    return np.random.default_rng(1234)


def has_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def load_simulate_golden():
    """tests/golden/simulate.npz + .json (make_golden_simulate.py): the
    reference's simulate() on a bf16-rounded model, per case and event."""
    data = np.load(os.path.join(GOLDEN, "simulate.npz"))
    meta = json.load(open(os.path.join(GOLDEN, "simulate.json")))
    w = {k[2:]: data[k] for k in data.files if k.startswith("w_")}
    cases = []
    for ci, c in enumerate(meta["cases"]):
        evs = []
        for ei, em in enumerate(c["events"]):
            evs.append(dict(em, **{f: data[f"c{ci}_e{ei}_{f}"] for f in ("ids", "assigned", "weights", "retained")}))
        cases.append(dict(name=c["name"], policy=c["policy"], hidden=data[f"c{ci}_hidden"], events=evs))
    return meta, w, data["inputs"], cases
