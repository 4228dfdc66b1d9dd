"""Trace JSONL in the reference's schema (trace.py:24-199): the reference's
own files (tests/golden/simulate_trace*.jsonl, written by its
write_trace_jsonl / write_masks_jsonl in make_golden_simulate.py) read back
through this package and re-written byte for byte."""

from __future__ import annotations

import os

import pytest

from conftest import GOLDEN

pytest.importorskip("torch")


def test_reference_trace_files_round_trip_byte_exact(tmp_path):
    from paper_2411_08982_b200 import trace as TR
    src = os.path.join(GOLDEN, "simulate_trace.jsonl")
    recs = TR.read_trace_jsonl(src)
    masks = TR.read_masks_jsonl(TR.masks_path_for(src))
    assert len(recs) == 2 * 2 * (9 + 3 * 3) and len(masks) == 2 * 4  # k * L * (prefill B*P + 3 steps * B)
    out = tmp_path / "run.jsonl"
    TR.write_trace_jsonl(out, recs)
    TR.write_masks_jsonl(TR.masks_path_for(out), masks)
    assert open(out).read() == open(src).read()
    assert open(TR.masks_path_for(out)).read() == open(TR.masks_path_for(src)).read()


def test_trace_record_validation():
    from paper_2411_08982_b200 import trace as TR
    from paper_2411_08982_b200.errors import TraceFormatError
    with pytest.raises(TraceFormatError):
        TR.TraceRecord("r", 0, 0, "train", 0, 0, 1, 1, 0.5, 0.5)
    with pytest.raises(TraceFormatError):
        TR.TraceRecord("r", -1, 0, "decode", 0, 0, 1, 1, 0.5, 0.5)


def test_malformed_trace_line_rejected(tmp_path):
    from paper_2411_08982_b200 import trace as TR
    from paper_2411_08982_b200.errors import TraceFormatError
    p = tmp_path / "bad.jsonl"
    p.write_text('{"run_id": "r"}\n')
    with pytest.raises(TraceFormatError):
        TR.read_trace_jsonl(p)
