"""Batch-level expert retention on the GPU -- drop-in mirror of moetrim.policy
(policy.py:1-350).

Every policy runs in liblynx_b200's selection kernel (K1): vote tally,
retention order, important-token selection, the retained set, the per-token
remap and renormalised gate weights.  The dataclasses and error behaviour
match the reference; arrays are torch CUDA tensors.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native as nat
from .errors import ValidationError
from .router import ExpertSelection, Phase, ctypes_ref

POLICY_MODES = ("latency", "accuracy")


def _torch():
    import torch
    return torch


@dataclass(frozen=True)
class PolicyConfig:
    """policy.py:26-65 (same defaults and validation)."""

    mode: str = "latency"
    drop_count: int = 0
    confidence_threshold: float = 0.5
    sample_threshold: int = 8
    min_experts: int | None = None
    freq_keep_budget: int = 4
    confidence_metric: str = "top1"
    vote_rank_weights: tuple[float, ...] | None = None

    def __post_init__(self) -> None:
        if self.mode not in POLICY_MODES:
            raise ValidationError(f"mode must be one of {POLICY_MODES}, got {self.mode!r}")
        if self.drop_count < 0:
            raise ValidationError("drop_count must be >= 0")
        if not (0.0 <= self.confidence_threshold <= 1.0):
            raise ValidationError("confidence_threshold must be in [0, 1]")
        if self.sample_threshold < 1:
            raise ValidationError("sample_threshold must be >= 1")
        if self.min_experts is not None and self.min_experts < 1:
            raise ValidationError("min_experts must be >= 1 when given")
        if self.freq_keep_budget < 1:
            raise ValidationError("freq_keep_budget must be >= 1")
        if self.vote_rank_weights is not None and any(w < 0 for w in self.vote_rank_weights):
            raise ValidationError("vote_rank_weights must be nonnegative")

    def resolved_min_experts(self, top_k: int) -> int:
        if self.min_experts is None:
            return top_k
        if self.min_experts < top_k:
            raise ValidationError(f"min_experts ({self.min_experts}) must be >= top_k ({top_k})")
        return self.min_experts

    def to_native(self, mode: str | None = None) -> nat.LynxPolicy:
        """The C struct lynx_policy_t (include/lynx_b200.h)."""
        m = self.mode if mode is None else mode
        p = nat.LynxPolicy()
        p.mode = nat.POLICY_LATENCY if m == "latency" else nat.POLICY_ACCURACY
        p.drop_count = self.drop_count
        p.confidence_threshold = self.confidence_threshold
        p.sample_threshold = self.sample_threshold
        p.min_experts = 0 if self.min_experts is None else self.min_experts
        p.freq_keep_budget = self.freq_keep_budget
        if self.confidence_metric not in ("top1", "margin"):
            raise ValidationError(f"unknown confidence metric {self.confidence_metric!r}")
        p.confidence_metric = nat.CONF_TOP1 if self.confidence_metric == "top1" else nat.CONF_MARGIN
        rw = self.vote_rank_weights
        if rw is not None:
            if len(rw) > nat.MAX_TOPK:
                raise ValidationError(f"at most {nat.MAX_TOPK} rank weights")
            p.n_rank_weights = len(rw)
            for i, w in enumerate(rw):
                p.rank_weights[i] = float(w)
        return p


@dataclass(frozen=True)
class VoteTally:
    """policy.py:68-80."""

    counts: object

    @property
    def num_experts(self) -> int:
        return int(self.counts.shape[0])

    @property
    def total(self) -> float:
        return float(self.counts.sum().item())


@dataclass(frozen=True)
class ExpertMask:
    """A policy decision for one layer-batch (policy.py:83-113)."""

    layer_index: int
    phase: Phase
    retained: object
    remap_original: object
    remap_assigned: object
    remap_weights: object
    clipped: bool = False
    important_tokens: object | None = None

    @property
    def num_retained(self) -> int:
        return int(self.retained.shape[0])

    @property
    def num_tokens(self) -> int:
        return int(self.remap_original.shape[0])

    def displacement_count(self) -> int:
        return int((self.remap_assigned != self.remap_original).sum().item())


@dataclass
class _PolicyRun:
    conf: object
    counts: object
    retained_mask: object
    assigned: object
    weights: object
    important: object
    flags: object


def _run_policy(selection: ExpertSelection, phase: Phase, native, conf_metric: str | None = None,
                check: bool = True) -> _PolicyRun:
    """One launch of the selection kernel on an existing selection."""
    torch = _torch()
    T, N, k = selection.num_tokens, selection.num_experts, selection.top_k
    if native is None and conf_metric is not None:
        native = nat.LynxPolicy()
        native.mode = nat.POLICY_NONE
        native.confidence_metric = nat.CONF_TOP1 if conf_metric == "top1" else nat.CONF_MARGIN
    run = _PolicyRun(
        conf=torch.empty((T,), dtype=torch.float64, device="cuda"),
        counts=torch.zeros((N,), dtype=torch.float64, device="cuda"),
        retained_mask=torch.empty((N,), dtype=torch.uint8, device="cuda"),
        assigned=torch.empty((T, k), dtype=torch.int32, device="cuda"),
        weights=torch.empty((T, k), dtype=torch.float64, device="cuda"),
        important=torch.zeros((T,), dtype=torch.uint8, device="cuda"),
        flags=torch.zeros((1,), dtype=torch.int32, device="cuda"),
    )
    out = nat.LynxSelection(conf=nat.ptr(run.conf), counts=nat.ptr(run.counts),
                            retained=nat.ptr(run.retained_mask), assigned=nat.ptr(run.assigned),
                            weights=nat.ptr(run.weights), important=nat.ptr(run.important),
                            flags=nat.ptr(run.flags))
    pol_ref = ctypes_ref(native) if native is not None else None
    nat.check(nat.lib().lynx_apply_policy(
        nat.ptr(selection.expert_ids), nat.ptr(selection.probs), nat.ptr(selection.full_probs),
        T, N, k, 1 if phase is Phase.DECODE else 0, pol_ref, ctypes_ref(out), nat.stream_handle()),
        "apply_policy")
    if check and native is not None and native.mode != nat.POLICY_NONE and phase is Phase.DECODE:
        if int(run.flags.item()) & nat.FLAG_ZERO_MASS:
            raise ValidationError("token has zero probability mass on the assigned experts")
    return run


def _mask_from_run(selection, run, layer_index, phase, with_important: bool) -> ExpertMask:
    torch = _torch()
    retained = torch.nonzero(run.retained_mask, as_tuple=False).flatten().to(torch.int64)
    important = None
    if with_important:
        important = torch.nonzero(run.important, as_tuple=False).flatten().to(torch.int64)
    flags = int(run.flags.item())
    return ExpertMask(layer_index=layer_index, phase=phase, retained=retained,
                      remap_original=selection.expert_ids.clone(), remap_assigned=run.assigned,
                      remap_weights=run.weights, clipped=bool(flags & nat.FLAG_CLIPPED),
                      important_tokens=important)


def vote_expert_frequencies(selection: ExpertSelection, rank_weights: tuple[float, ...] | None = None) -> VoteTally:
    """policy.py:116-138 on the GPU."""
    torch = _torch()
    T, k, N = selection.num_tokens, selection.top_k, selection.num_experts
    native = None
    if rank_weights is not None:
        if len(rank_weights) != k:
            raise ValidationError(f"rank_weights must have length top_k={k}")
        native = PolicyConfig(vote_rank_weights=tuple(rank_weights)).to_native()
    counts = torch.empty((N,), dtype=torch.float64, device="cuda")
    nat.check(nat.lib().lynx_vote(nat.ptr(selection.expert_ids), T, k, N,
                                  ctypes_ref(native) if native is not None else None,
                                  nat.ptr(counts), nat.stream_handle()), "vote_expert_frequencies")
    return VoteTally(counts=counts)


def _retained_list(retained, N: int) -> list[int]:
    torch = _torch()
    if isinstance(retained, torch.Tensor):
        retained = retained.detach().cpu().numpy()
    ids = sorted(set(int(e) for e in np.asarray(retained).ravel()))
    if not ids:
        raise ValidationError("retained set must be non-empty")
    if ids[0] < 0 or ids[-1] >= N:
        raise ValidationError("retained contains out-of-range expert ids")
    return ids


def remap_tokens(selection: ExpertSelection, retained):
    """policy.py:151-212 -> (original, assigned, weights) CUDA tensors."""
    torch = _torch()
    T, k, N = selection.num_tokens, selection.top_k, selection.num_experts
    ids = _retained_list(retained, N)
    mask = torch.zeros((N,), dtype=torch.uint8)
    mask[ids] = 1
    mask = mask.to("cuda")
    assigned = torch.empty((T, k), dtype=torch.int32, device="cuda")
    weights = torch.empty((T, k), dtype=torch.float64, device="cuda")
    flags = torch.zeros((1,), dtype=torch.int32, device="cuda")
    nat.check(nat.lib().lynx_remap(nat.ptr(selection.expert_ids), nat.ptr(selection.full_probs), T, N, k,
                                   nat.ptr(mask), nat.ptr(assigned), nat.ptr(weights), nat.ptr(flags),
                                   nat.stream_handle()), "remap_tokens")
    if int(flags.item()) & nat.FLAG_ZERO_MASS:
        raise ValidationError("token has zero probability mass on the assigned experts")
    return selection.expert_ids.clone(), assigned, weights


def full_retain_mask(selection: ExpertSelection, layer_index: int, phase: Phase) -> ExpertMask:
    """policy.py:215-229."""
    run = _run_policy(selection, phase, None, conf_metric="top1")
    return _mask_from_run(selection, run, layer_index, phase, with_important=False)


def latency_policy(selection: ExpertSelection, phase: Phase, config: PolicyConfig,
                   layer_index: int = 0) -> ExpertMask:
    """policy.py:232-264."""
    if phase is Phase.PREFILL:
        return full_retain_mask(selection, layer_index, phase)
    config.resolved_min_experts(selection.top_k)
    if config.vote_rank_weights is not None and len(config.vote_rank_weights) != selection.top_k:
        raise ValidationError(f"rank_weights must have length top_k={selection.top_k}")
    run = _run_policy(selection, phase, config.to_native("latency"))
    return _mask_from_run(selection, run, layer_index, phase, with_important=False)


def select_important_tokens(selection: ExpertSelection, config: PolicyConfig):
    """policy.py:267-284 (computed by the accuracy-policy kernel)."""
    torch = _torch()
    if config.confidence_metric not in ("top1", "margin"):
        raise ValidationError(f"unknown confidence metric {config.confidence_metric!r}")
    native = config.to_native("accuracy")
    native.min_experts = 0  # the important set does not depend on the floor
    native.n_rank_weights = 0
    run = _run_policy(selection, Phase.DECODE, native)
    return torch.nonzero(run.important, as_tuple=False).flatten().to(torch.int64)


def accuracy_policy(selection: ExpertSelection, phase: Phase, config: PolicyConfig,
                    layer_index: int = 0) -> ExpertMask:
    """policy.py:287-338."""
    if phase is Phase.PREFILL:
        return full_retain_mask(selection, layer_index, phase)
    config.resolved_min_experts(selection.top_k)
    if config.vote_rank_weights is not None and len(config.vote_rank_weights) != selection.top_k:
        raise ValidationError(f"rank_weights must have length top_k={selection.top_k}")
    run = _run_policy(selection, phase, config.to_native("accuracy"))
    return _mask_from_run(selection, run, layer_index, phase, with_important=True)


def apply_policy(selection: ExpertSelection, phase: Phase, config: PolicyConfig,
                 layer_index: int = 0) -> ExpertMask:
    """policy.py:341-350."""
    if config.mode == "latency":
        return latency_policy(selection, phase, config, layer_index)
    return accuracy_policy(selection, phase, config, layer_index)
