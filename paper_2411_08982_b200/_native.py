"""ctypes binding of the C ABI in include/lynx_b200.h.

This is the only way the package reaches the GPU: every compute call goes
through liblynx_b200.so.  There is deliberately no CPU or PyTorch fallback;
if the library is missing or no CUDA device is present the call raises.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import NativeLibraryError, ValidationError

LIB_PATH = os.environ.get(
    "LYNX_LIB", os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib", "liblynx_b200.so"))

# include/lynx_b200.h constants
LYNX_OK = 0
ABI_VERSION = 5
STATUS = {
    -1: "invalid shape", -2: "k out of range", -3: "min_experts must be >= top_k",
    -4: "retained set empty or out of range", -5: "token count mismatch", -6: "CUDA error",
    -7: "shape outside build limits", -8: "workspace too small", -9: "invalid policy config",
}
VALIDATION_CODES = {-1, -2, -3, -4, -5, -7, -9}
FLAG_CLIPPED, FLAG_NONFINITE, FLAG_ZERO_MASS = 1, 2, 4
MAX_EXPERTS, MAX_TOPK, MAX_TOKENS, SEG_ROWS, MAX_SHARED, MAX_DHEAD = 64, 8, 4096, 256, 4, 64
MAX_FUSED_ROUTER = 16
POLICY_NONE, POLICY_LATENCY, POLICY_ACCURACY = 0, 1, 2
CONF_TOP1, CONF_MARGIN = 0, 1
ACT_SWIGLU, ACT_TANH2 = 0, 1

_p = ctypes.c_void_p
_i = ctypes.c_int


class LynxPolicy(ctypes.Structure):
    _fields_ = [("mode", ctypes.c_int32), ("drop_count", ctypes.c_int32),
                ("confidence_threshold", ctypes.c_double), ("sample_threshold", ctypes.c_int32),
                ("min_experts", ctypes.c_int32), ("freq_keep_budget", ctypes.c_int32),
                ("confidence_metric", ctypes.c_int32), ("n_rank_weights", ctypes.c_int32),
                ("reserved", ctypes.c_int32), ("rank_weights", ctypes.c_double * MAX_TOPK)]


class LynxSelection(ctypes.Structure):
    _fields_ = [(name, _p) for name in (
        "expert_ids", "probs", "full_probs", "conf", "counts", "retained", "assigned",
        "weights", "important", "flags")]


class LynxLayer(ctypes.Structure):
    _fields_ = [("num_experts", ctypes.c_int32), ("top_k", ctypes.c_int32),
                ("d_model", ctypes.c_int32), ("d_ff", ctypes.c_int32),
                ("activation", ctypes.c_int32), ("num_shared", ctypes.c_int32),
                ("w13", _p), ("w2", _p), ("router_wt", _p)]


class LynxAttention(ctypes.Structure):
    _fields_ = [("d_model", ctypes.c_int32), ("d_head", ctypes.c_int32), ("max_len", ctypes.c_int32),
                ("num_experts", ctypes.c_int32), ("wqkv", _p), ("wo", _p), ("k_cache", _p), ("v_cache", _p),
                ("router_wt", _p), ("logits", _p)]


class LynxTraceRing(ctypes.Structure):
    _fields_ = [("capacity", ctypes.c_int32), ("num_layers", ctypes.c_int32), ("T", ctypes.c_int32),
                ("k", ctypes.c_int32), ("N", ctypes.c_int32), ("reserved", ctypes.c_int32)] + [
        (name, _p) for name in ("positions", "original", "assigned", "weights", "conf", "retained", "important",
                                "flags")]


class LynxEPPeers(ctypes.Structure):
    _fields_ = [("world_size", ctypes.c_int32), ("rank", ctypes.c_int32), ("tokens_per_rank", ctypes.c_int32),
                ("reserved", ctypes.c_int32)] + [
        (name, _p) for name in ("logits", "recv", "back", "flags", "logits_local", "recv_local", "back_local",
                                "flags_local", "counters", "epoch")]


class LynxDispatch(ctypes.Structure):
    _fields_ = [(name, _p) for name in (
        "n_seg", "n_used", "n_rows", "seg_expert", "seg_row", "seg_count", "perm_token", "perm_weight",
        "tok_rows", "tok_weight", "x_perm")]


_SIGS = {
    "lynx_abi_version": (_i, []),
    "lynx_status_string": (ctypes.c_char_p, [_i]),
    "lynx_dispatch_caps": (_i, [_i, _i, _i, _p, _p]),
    "lynx_moe_workspace_bytes": (ctypes.c_size_t, [_p, _i]),
    "lynx_router_logits": (_i, [_p, _p, _i, _i, _i, _p, _p]),
    "lynx_route_select": (_i, [_p, _i, _i, _i, _i, _p, _p, _p]),
    "lynx_apply_policy": (_i, [_p, _p, _p, _i, _i, _i, _i, _p, _p, _p]),
    "lynx_topk": (_i, [_p, _i, _i, _i, _p, _p, _p]),
    "lynx_vote": (_i, [_p, _i, _i, _i, _p, _p, _p]),
    "lynx_remap": (_i, [_p, _p, _i, _i, _i, _p, _p, _p, _p, _p]),
    "lynx_permute": (_i, [_p, _p, _p, _i, _i, _i, _i, _p, _p]),
    "lynx_moe_forward": (_i, [_p, _p, _i, _p, _p, _p, _p, ctypes.c_size_t, _p]),
    "lynx_moe_forward_partial": (_i, [_p, _p, _i, _p, _p, _p, _p, ctypes.c_size_t, _p]),
    "lynx_moe_layer": (_i, [_p, _p, _i, _i, _p, _p, _p, _p, ctypes.c_size_t, _p]),
    "lynx_moe_layer_logits": (_i, [_p, _p, _p, _i, _i, _p, _p, _p, _p, ctypes.c_size_t, _p]),
    "lynx_moe_layer_profiled": (_i, [_p, _p, _i, _i, _p, _p, _p, _p, ctypes.c_size_t, _p, _p, _i]),
    "lynx_moe_ffn_kernel": (_i, [_p, _i, _i, _p, _p]),
    "lynx_pack_w13": (_i, [_p, _p, _i, _i, _i, _p, _p]),
    "lynx_attention_workspace_bytes": (ctypes.c_size_t, [_i, _i]),
    "lynx_attention": (_i, [_p, _p, _i, _i, _i, _p, _p, _p, ctypes.c_size_t, _p]),
    "lynx_advance_position": (_i, [_p, _i, _p]),
    "lynx_trace_append": (_i, [_p, _p, _i, _p, _p]),
    "lynx_enable_peer_access": (_i, [_i]),
    "lynx_ep_p2p_route": (_i, [_p, _p, _i, _i, _p, _p]),
    "lynx_ep_p2p_dispatch": (_i, [_p, _i, _i, _i, _i, _p, _p, _p, _p]),
    "lynx_ep_p2p_expert": (_i, [_p, _i, _p, _p, _p, _p, _p, _p, ctypes.c_size_t, _p]),
    "lynx_ep_p2p_combine": (_i, [_p, _i, _p, _p, _p]),
    "lynx_ep_pack": (_i, [_p, _p, _i, _i, _i, _i, _i, _i, _p, _p]),
    "lynx_ep_local_mask": (_i, [_p, _p, _i, _i, _i, _i, _i, _p, _p, _p]),
    "lynx_ep_combine": (_i, [_p, _p, _i, _i, _i, _p, _p]),
}
EXPORTS = tuple(_SIGS)

_lib = None
_lock = threading.Lock()


def load(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load liblynx_b200.so and declare every exported prototype (no GPU needed)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise NativeLibraryError(
                f"{path} is missing: build it with `python -m paper_2411_08982_b200._build` "
                "(there is no CPU fallback)")
        lib = ctypes.CDLL(path)
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.lynx_abi_version() != ABI_VERSION:
            raise NativeLibraryError("liblynx_b200.so ABI version mismatch")
        _lib = lib
        return lib


def lib() -> ctypes.CDLL:
    return _lib if _lib is not None else load()


def check(status: int, what: str) -> None:
    """Map a lynx_status to the reference's exception type (errors.py:4-5)."""
    if status == LYNX_OK:
        return
    msg = f"{what}: {STATUS.get(status, f'status {status}')}"
    if status in VALIDATION_CODES:
        raise ValidationError(msg)
    raise NativeLibraryError(msg)


def ptr(t) -> int:
    """Device pointer of a CUDA tensor (0 for None)."""
    if t is None:
        return 0
    if not t.is_cuda:
        raise NativeLibraryError("liblynx_b200 takes CUDA tensors (no CPU path)")
    return t.data_ptr()


def stream_handle(stream=None) -> int:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream
