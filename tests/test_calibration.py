"""The B200 calibration table (profiles/calibration_b200.csv)
keeps the reference's calibration format (costmodel.py:300-343), so the
reference cost model reads it unchanged."""

from __future__ import annotations

import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TABLE = os.path.join(ROOT, "profiles", "calibration_b200.csv")
REF_SRC = "/root/reference/pkg/src"


def test_table_format():
    lines = [ln for ln in open(TABLE).read().splitlines() if ln.strip() and not ln.startswith("#")]
    assert lines[0] == "batch_size,attn_ms,route_ms,mlp_ms"
    rows = [ln.split(",") for ln in lines[1:]]
    assert [int(r[0]) for r in rows] == [8, 16, 32, 64]
    for r in rows:
        assert all(float(v) > 0 for v in r[1:])


@pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="reference source tree not mounted")
def test_reference_cost_model_reads_table():
    code = ("from moetrim.costmodel import read_calibration_table, calibrate\n"
            "from moetrim.router import MoEModelSpec\n"
            f"rows = read_calibration_table({TABLE!r})\n"
            "p, rep = calibrate(rows, MoEModelSpec(32, 8, 2, 4096, 14336, 2), 4)\n"
            "assert len(rep.rows) == 4 and p.route_ms_per_layer > 0\n"
            "print('ok')\n")
    env = dict(os.environ, PYTHONPATH=REF_SRC, PYTHONDONTWRITEBYTECODE="1")
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, cwd="/tmp")
    assert out.returncode == 0 and out.stdout.strip() == "ok", out.stderr
