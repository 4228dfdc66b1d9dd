"""Routing math on the GPU -- drop-in mirror of moetrim.router (router.py:1-192).

Same names, argument order, return dataclasses and ValidationError
behaviour as the reference; the arrays are torch CUDA tensors (float64
probabilities, int32 expert ids) produced by liblynx_b200's selection
kernel.  ``tensor.cpu().numpy()`` gives the reference's numpy view.
"""

from __future__ import annotations

from dataclasses import dataclass
from enum import Enum

import numpy as np

from . import _native as nat
from .errors import ValidationError


def _torch():
    import torch
    return torch


class Phase(Enum):
    """router.py:20-22."""

    PREFILL = "prefill"
    DECODE = "decode"


@dataclass(frozen=True)
class MoEModelSpec:
    """Static shape of an MoE stack (router.py:25-54)."""

    num_layers: int
    num_experts: int
    top_k: int
    d_model: int
    d_ff: int
    bytes_per_param: int = 2
    # Builder extension (not in the reference): always-on shared experts of
    # size d_ff applied to every token with weight 1 (DeepSeek-MoE).
    num_shared_experts: int = 0

    def __post_init__(self) -> None:
        if self.num_layers < 1:
            raise ValidationError("num_layers must be >= 1")
        if self.num_experts < 1:
            raise ValidationError("num_experts must be >= 1")
        if not (1 <= self.top_k <= self.num_experts):
            raise ValidationError(
                f"top_k must be in [1, num_experts]; got {self.top_k} with {self.num_experts} experts")
        if self.d_model < 1 or self.d_ff < 1:
            raise ValidationError("d_model and d_ff must be >= 1")
        if self.bytes_per_param < 1:
            raise ValidationError("bytes_per_param must be >= 1")
        if not (0 <= self.num_shared_experts <= nat.MAX_SHARED):
            raise ValidationError(f"num_shared_experts must be in [0, {nat.MAX_SHARED}]")

    @property
    def expert_param_bytes(self) -> int:
        """The reference's two-matrix count (router.py:51-54)."""
        return 2 * self.d_model * self.d_ff * self.bytes_per_param

    @property
    def swiglu_expert_bytes(self) -> int:
        """Bytes one SwiGLU expert (w1, w3, w2) streams: 3*d*ff*bpp."""
        return 3 * self.d_model * self.d_ff * self.bytes_per_param


def _device_f64(values, what: str):
    """2-D float64 CUDA tensor; host inputs are finite-checked here like the reference."""
    torch = _torch()
    if isinstance(values, torch.Tensor):
        v = values
        if v.ndim != 2:
            raise ValidationError(f"{what} must be 2-D, got shape {tuple(v.shape)}")
        if not v.is_cuda:
            host = v.detach().numpy().astype(np.float64)
            if not np.all(np.isfinite(host)):
                raise ValidationError(f"{what} contain non-finite values")
        v = v.to(device="cuda", dtype=torch.float64).contiguous()
    else:
        host = np.asarray(values, dtype=np.float64)
        if host.ndim != 2:
            raise ValidationError(f"{what} must be 2-D, got shape {host.shape}")
        if host.shape[0] >= 1 and host.shape[1] >= 1 and not np.all(np.isfinite(host)):
            raise ValidationError(f"{what} contain non-finite values")
        v = torch.from_numpy(np.ascontiguousarray(host)).to("cuda")
    if v.shape[0] < 1 or v.shape[1] < 1:
        raise ValidationError(f"{what} must be non-empty, got shape {tuple(v.shape)}")
    return v


@dataclass(frozen=True)
class RoutingLogits:
    """Raw router outputs [num_tokens, num_experts] (router.py:57-81).

    Host inputs are checked for NaN/Inf at construction; CUDA inputs are
    checked by the selection kernel and rejected by route_batch.
    """

    layer_index: int
    phase: Phase
    values: object

    def __post_init__(self) -> None:
        object.__setattr__(self, "values", _device_f64(self.values, "logits"))

    @property
    def num_tokens(self) -> int:
        return int(self.values.shape[0])

    @property
    def num_experts(self) -> int:
        return int(self.values.shape[1])


def _ids_tensor(ids):
    torch = _torch()
    if isinstance(ids, torch.Tensor):
        return ids.to(device="cuda", dtype=torch.int32).contiguous()
    return torch.from_numpy(np.ascontiguousarray(np.asarray(ids, dtype=np.int32))).to("cuda")


def _f64_tensor(x):
    torch = _torch()
    if isinstance(x, torch.Tensor):
        return x.to(device="cuda", dtype=torch.float64).contiguous()
    return torch.from_numpy(np.ascontiguousarray(np.asarray(x, dtype=np.float64))).to("cuda")


@dataclass(frozen=True)
class ExpertSelection:
    """Top-k routing decision (router.py:84-138); CUDA tensors."""

    expert_ids: object
    probs: object
    full_probs: object

    def __post_init__(self) -> None:
        ids, probs, full = _ids_tensor(self.expert_ids), _f64_tensor(self.probs), _f64_tensor(self.full_probs)
        if ids.ndim != 2 or full.ndim != 2:
            raise ValidationError("expert_ids and full_probs must be 2-D")
        if tuple(ids.shape) != tuple(probs.shape):
            raise ValidationError(
                f"expert_ids shape {tuple(ids.shape)} does not match probs shape {tuple(probs.shape)}")
        if full.shape[0] != ids.shape[0]:
            raise ValidationError("full_probs must have one row per routed token")
        if ids.shape[1] > full.shape[1]:
            raise ValidationError("more selection slots than experts")
        object.__setattr__(self, "expert_ids", ids)
        object.__setattr__(self, "probs", probs)
        object.__setattr__(self, "full_probs", full)

    @property
    def num_tokens(self) -> int:
        return int(self.expert_ids.shape[0])

    @property
    def top_k(self) -> int:
        return int(self.expert_ids.shape[1])

    @property
    def num_experts(self) -> int:
        return int(self.full_probs.shape[1])

    def confidence(self, metric: str = "top1"):
        """router.py:125-138, computed by the selection kernel."""
        if metric not in ("top1", "margin"):
            raise ValidationError(f"unknown confidence metric {metric!r}")
        from .policy import _run_policy  # local import: policy builds on router
        return _run_policy(self, Phase.DECODE, None, conf_metric=metric).conf


def softmax_probs(logits):
    """Float64 softmax over the last axis (router.py:141-154), on the GPU."""
    torch = _torch()
    if isinstance(logits, torch.Tensor):
        z = logits
        if z.numel() == 0:
            raise ValidationError("softmax input is empty")
    else:
        z = np.asarray(logits, dtype=np.float64)
        if z.size == 0:
            raise ValidationError("softmax input is empty")
        if not np.all(np.isfinite(z)):
            raise ValidationError("softmax input contains non-finite values")
    shape = tuple(z.shape)
    rows = _device_f64(z.reshape(-1, shape[-1]) if len(shape) != 2 else z, "softmax input")
    sel = route_batch(RoutingLogits(0, Phase.DECODE, rows), 1)
    return sel.full_probs.reshape(shape)


def top_k_select(probs, k: int):
    """Indices and values of the k largest entries, ties -> smaller index (router.py:157-171)."""
    torch = _torch()
    p = probs if isinstance(probs, torch.Tensor) else np.asarray(probs, dtype=np.float64)
    if p.ndim != 1:
        raise ValidationError("top_k_select expects a 1-D probability vector")
    n = int(p.shape[0])
    if not (1 <= k <= n):
        raise ValidationError(f"k must be in [1, {n}], got {k}")
    row = _f64_tensor(p).reshape(1, n)
    ids = torch.empty((1, k), dtype=torch.int32, device="cuda")
    vals = torch.empty((1, k), dtype=torch.float64, device="cuda")
    nat.check(nat.lib().lynx_topk(nat.ptr(row), 1, n, k, nat.ptr(ids), nat.ptr(vals), nat.stream_handle()),
              "top_k_select")
    return ids[0].to(torch.int64), vals[0]


def route_batch(logits: RoutingLogits, k: int, check: bool = True) -> ExpertSelection:
    """Softmax + top-k for every token of a layer-batch (router.py:174-187).

    ``check`` reads back the kernel's flag word (one small device->host copy)
    so non-finite CUDA logits raise ValidationError like the reference.
    """
    torch = _torch()
    if not (1 <= k <= logits.num_experts):
        raise ValidationError(f"k must be in [1, {logits.num_experts}], got {k}")
    T, N = logits.num_tokens, logits.num_experts
    ids = torch.empty((T, k), dtype=torch.int32, device="cuda")
    probs = torch.empty((T, k), dtype=torch.float64, device="cuda")
    full = torch.empty((T, N), dtype=torch.float64, device="cuda")
    conf = torch.empty((T,), dtype=torch.float64, device="cuda")
    assigned = torch.empty((T, k), dtype=torch.int32, device="cuda")
    weights = torch.empty((T, k), dtype=torch.float64, device="cuda")
    flags = torch.zeros((1,), dtype=torch.int32, device="cuda")
    sel = nat.LynxSelection(expert_ids=nat.ptr(ids), probs=nat.ptr(probs), full_probs=nat.ptr(full),
                            conf=nat.ptr(conf), assigned=nat.ptr(assigned), weights=nat.ptr(weights),
                            flags=nat.ptr(flags))
    nat.check(nat.lib().lynx_route_select(nat.ptr(logits.values), T, N, k, 1, None, ctypes_ref(sel),
                                          nat.stream_handle()), "route_batch")
    if check and int(flags.item()) & nat.FLAG_NONFINITE:
        raise ValidationError("logits contain non-finite values")
    return ExpertSelection(expert_ids=ids, probs=probs, full_probs=full)


def confidence(selection: ExpertSelection, metric: str = "top1"):
    """Free-function alias for ExpertSelection.confidence (router.py:190-192)."""
    return selection.confidence(metric)


def ctypes_ref(struct):
    import ctypes
    return ctypes.cast(ctypes.pointer(struct), ctypes.c_void_p)
