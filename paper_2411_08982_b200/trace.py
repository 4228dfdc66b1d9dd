"""Routing traces in the reference's JSONL schema (moetrim/trace.py), emitted
from the GPU selection.

Schema (identical to the reference, so ``moetrim analyze`` reads B200 runs
unchanged): one record per (batch event, layer, token, rank) slot with the
fields of ``TRACE_FIELDS`` (trace.py:24-35), plus a sibling
``<stem>.masks.jsonl`` with one record per (batch event, layer) holding the
retained set (trace.py:60-76, 196-199).

``TraceRecorder`` is the B200 part: inside a captured decode step every
layer appends its routing event to a device ring (``lynx_trace_append``, one
launch per layer, slot chosen from the device cache position), so tracing
adds no host synchronisation per step; the ring is drained to host records
when it fills or when the caller asks.
"""

from __future__ import annotations

import json
import os
from dataclasses import asdict, dataclass
from pathlib import Path
from typing import Iterable

from . import _native as nat
from .errors import TraceFormatError
from .router import Phase, ctypes_ref

TRACE_FIELDS = ("run_id", "layer", "batch_id", "phase", "token_id", "rank", "expert_original",
                "expert_assigned", "weight", "confidence")
PHASES = ("prefill", "decode")


def _torch():
    import torch
    return torch


@dataclass(frozen=True)
class TraceRecord:
    """One routed slot (trace.py:38-57)."""

    run_id: str
    layer: int
    batch_id: int
    phase: str
    token_id: int
    rank: int
    expert_original: int
    expert_assigned: int
    weight: float
    confidence: float

    def __post_init__(self) -> None:
        if self.phase not in PHASES:
            raise TraceFormatError(f"phase must be one of {PHASES}, got {self.phase!r}")
        for f in ("layer", "batch_id", "token_id", "rank", "expert_original", "expert_assigned"):
            if int(getattr(self, f)) < 0:
                raise TraceFormatError(f"{f} must be nonnegative")


@dataclass(frozen=True)
class MaskRecord:
    """One (batch event, layer) retained set (trace.py:60-76)."""

    run_id: str
    batch_id: int
    layer: int
    phase: str
    retained: tuple
    clipped: bool
    num_tokens: int
    num_important: int | None = None

    def __post_init__(self) -> None:
        if self.phase not in PHASES:
            raise TraceFormatError(f"phase must be one of {PHASES}, got {self.phase!r}")
        object.__setattr__(self, "retained", tuple(int(e) for e in self.retained))


def _event_records(run_id, batch_id, layer, phase, original, assigned, weights, conf):
    T, k = original.shape
    return [TraceRecord(run_id, int(layer), int(batch_id), phase, t, r, int(original[t, r]), int(assigned[t, r]),
                        float(weights[t, r]), float(conf[t])) for t in range(T) for r in range(k)]


def records_from_event(run_id: str, batch_id: int, layer: int, phase: Phase, selection, mask) -> list:
    """trace.py:81-108 on a GPU selection/mask (arrays copied to the host)."""
    conf = selection.confidence().cpu().numpy()
    return _event_records(run_id, batch_id, layer, phase.value, mask.remap_original.cpu().numpy(),
                          mask.remap_assigned.cpu().numpy(), mask.remap_weights.cpu().numpy(), conf)


def mask_record_from_event(run_id: str, batch_id: int, layer: int, phase: Phase, mask) -> MaskRecord:
    """trace.py:111-125."""
    imp = mask.important_tokens
    return MaskRecord(run_id, int(batch_id), int(layer), phase.value,
                      tuple(int(e) for e in mask.retained.cpu().tolist()), bool(mask.clipped), int(mask.num_tokens),
                      None if imp is None else int(len(imp)))


def _write_lines(path: Path, lines: list) -> None:
    tmp = path.with_suffix(path.suffix + ".tmp")
    tmp.write_text("\n".join(lines) + ("\n" if lines else ""))
    os.replace(tmp, path)


def write_trace_jsonl(path, records: Iterable[TraceRecord]) -> None:
    _write_lines(Path(path), [json.dumps({f: getattr(r, f) for f in TRACE_FIELDS}, separators=(",", ":"))
                              for r in records])


def write_masks_jsonl(path, records: Iterable[MaskRecord]) -> None:
    _write_lines(Path(path), [json.dumps(asdict(r), separators=(",", ":")) for r in records])


def read_trace_jsonl(path) -> list:
    path = Path(path)
    if not path.is_file():
        raise TraceFormatError(f"{path}: no such trace file")
    out = []
    for n, line in enumerate(path.read_text().splitlines(), start=1):
        if not line.strip():
            continue
        try:
            obj = json.loads(line)
        except json.JSONDecodeError as exc:
            raise TraceFormatError(f"{path}:{n}: malformed record: {exc}") from exc
        missing = [f for f in TRACE_FIELDS if f not in obj]
        if missing:
            raise TraceFormatError(f"{path}:{n}: missing fields {missing}")
        try:
            out.append(TraceRecord(**{f: obj[f] for f in TRACE_FIELDS}))
        except (TypeError, TraceFormatError) as exc:
            raise TraceFormatError(f"{path}:{n}: {exc}") from exc
    return out


def read_masks_jsonl(path) -> list:
    path = Path(path)
    if not path.is_file():
        raise TraceFormatError(f"{path}: no such masks file")
    out = []
    for n, line in enumerate(path.read_text().splitlines(), start=1):
        if not line.strip():
            continue
        try:
            obj = json.loads(line)
            obj["retained"] = tuple(int(e) for e in obj["retained"])
            out.append(MaskRecord(**obj))
        except json.JSONDecodeError as exc:
            raise TraceFormatError(f"{path}:{n}: malformed record: {exc}") from exc
        except (TypeError, KeyError) as exc:
            raise TraceFormatError(f"{path}:{n}: {exc}") from exc
    return out


def masks_path_for(trace_path) -> Path:
    """trace.py:196-199."""
    p = Path(trace_path)
    return p.with_name(p.stem + ".masks.jsonl")


class TraceRecorder:
    """Collects every routing event of a DecodeStack run.

    Prefill events are recorded on the host directly (one event, not
    captured).  Decode events go through the device ring: ``capacity`` steps
    of [L, B, k] routing state, drained with one copy when full or on
    ``flush()``.  Batch ids follow simulate(): prefill is event 0, decode
    step s is event 1 + s (simulator.py:344-345).
    """

    def __init__(self, run_id: str, num_layers: int, batch: int, num_experts: int, top_k: int, capacity: int = 256):
        torch = _torch()
        self.run_id, self.L, self.B, self.N, self.k, self.cap = run_id, num_layers, batch, num_experts, top_k, capacity
        dev = "cuda"
        L, B, N, k = num_layers, batch, num_experts, top_k
        self.positions = torch.full((capacity,), -1, dtype=torch.int32, device=dev)
        self.original = torch.zeros((capacity, L, B, k), dtype=torch.int32, device=dev)
        self.assigned = torch.zeros_like(self.original)
        self.weights = torch.zeros((capacity, L, B, k), dtype=torch.float64, device=dev)
        self.conf = torch.zeros((capacity, L, B), dtype=torch.float64, device=dev)
        self.retained = torch.zeros((capacity, L, N), dtype=torch.uint8, device=dev)
        self.important = torch.zeros((capacity, L, B), dtype=torch.uint8, device=dev)
        self.flags = torch.zeros((capacity, L), dtype=torch.int32, device=dev)
        r = nat.LynxTraceRing()
        r.capacity, r.num_layers, r.T, r.k, r.N = capacity, L, B, k, N
        for f in ("positions", "original", "assigned", "weights", "conf", "retained", "important", "flags"):
            setattr(r, f, nat.ptr(getattr(self, f)))
        self._ring = r
        self._ring_ref = ctypes_ref(r)
        self.trace: list = []
        self.masks: list = []
        self.prefill_len = 0
        self._pending = 0
        self._policy_mode: dict = {}

    # --- producers (called by DecodeStack)
    def record(self, layer: int, phase: Phase, lynx_layer, event_offset: int = 0) -> None:
        """Host-side record of a non-captured event (the prefill chunk)."""
        sel_mask = lynx_layer.mask()
        probs = lynx_layer.full_probs.max(dim=1).values.cpu().numpy()
        self.trace.extend(_event_records(self.run_id, event_offset, layer, phase.value,
                                         lynx_layer.expert_ids.cpu().numpy(), lynx_layer.assigned.cpu().numpy(),
                                         lynx_layer.weights.cpu().numpy(), probs))
        self.masks.append(self._mask_record(event_offset, layer, phase.value, sel_mask.retained.cpu().tolist(),
                                            bool(sel_mask.clipped), lynx_layer.T,
                                            self._num_important(lynx_layer, sel_mask.important_tokens.numel())))
        if phase is Phase.PREFILL and layer == 0:
            self.prefill_len = lynx_layer.T // self.B

    def record_device(self, layer: int, lynx_layer, pos) -> None:
        """Append one layer's routing event to the device ring (graph-capturable)."""
        torch = _torch()
        self._policy_mode[layer] = None if lynx_layer._pol is None else lynx_layer._pol.mode
        nat.check(nat.lib().lynx_trace_append(self._ring_ref, pos.data_ptr(), layer, lynx_layer._sel_ref,
                                              torch.cuda.current_stream().cuda_stream), "lynx_trace_append")

    def rewind(self) -> None:
        self.positions.fill_(-1)

    def step_done(self) -> None:
        self._pending += 1
        if self._pending >= self.cap:
            self.flush()

    # --- drain
    def _num_important(self, lynx_layer, count: int):
        pol = lynx_layer._pol
        if pol is None or pol.mode != nat.POLICY_ACCURACY or lynx_layer.phase is not Phase.DECODE:
            return None
        return int(count)

    @staticmethod
    def _mask_record(batch_id, layer, phase, retained, clipped, num_tokens, num_important):
        return MaskRecord("", batch_id, layer, phase, tuple(retained), clipped, num_tokens, num_important)

    def flush(self) -> None:
        """Drain the device ring (one host sync) into host records."""
        if self._pending == 0:
            return
        pos = self.positions.cpu().numpy()
        ori, asg = self.original.cpu().numpy(), self.assigned.cpu().numpy()
        w, conf = self.weights.cpu().numpy(), self.conf.cpu().numpy()
        ret, imp, flags = self.retained.cpu().numpy(), self.important.cpu().numpy(), self.flags.cpu().numpy()
        for slot in sorted(range(self.cap), key=lambda s: pos[s]):
            if pos[slot] < 0:
                continue
            batch_id = 1 + int(pos[slot]) - self.prefill_len
            for l in range(self.L):
                self.trace.extend(_event_records(self.run_id, batch_id, l, "decode", ori[slot, l], asg[slot, l],
                                                 w[slot, l], conf[slot, l]))
                acc = self._policy_mode.get(l) == nat.POLICY_ACCURACY
                self.masks.append(self._mask_record(batch_id, l, "decode",
                                                    [int(e) for e in (ret[slot, l] > 0).nonzero()[0]],
                                                    bool(flags[slot, l] & nat.FLAG_CLIPPED), self.B,
                                                    int(imp[slot, l].sum()) if acc else None))
        self.positions.fill_(-1)
        self._pending = 0

    def records(self) -> list:
        self.flush()
        return list(self.trace)

    def mask_records(self) -> list:
        self.flush()
        return [MaskRecord(self.run_id, m.batch_id, m.layer, m.phase, m.retained, m.clipped, m.num_tokens,
                           m.num_important) for m in self.masks]

    def write(self, path) -> None:
        """Write <path> (slot records) and <stem>.masks.jsonl (retained sets)."""
        write_trace_jsonl(path, self.records())
        write_masks_jsonl(masks_path_for(path), self.mask_records())
