"""CPU checks of the C ABI boundary: the library loads without a GPU and
exports every entry point include/lynx_b200.h declares."""

from __future__ import annotations

import ctypes
import os
import re

import pytest

from conftest import ROOT


def header_symbols():
    text = open(os.path.join(ROOT, "include", "lynx_b200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|size_t|const char \*)\s*\**\s*(lynx_\w+)\s*\(", text, re.M)))


def test_header_declares_expected_entry_points():
    syms = header_symbols()
    for name in ("lynx_route_select", "lynx_apply_policy", "lynx_remap", "lynx_permute", "lynx_moe_forward",
                 "lynx_moe_layer", "lynx_router_logits", "lynx_ep_pack", "lynx_ep_combine"):
        assert name in syms


def test_library_exports_every_header_symbol():
    from paper_2411_08982_b200 import _native
    lib = _native.load()
    for name in header_symbols():
        assert hasattr(lib, name), name
    assert set(header_symbols()) == set(_native.EXPORTS)


def test_status_strings_and_version():
    from paper_2411_08982_b200 import _native
    lib = _native.load()
    assert lib.lynx_abi_version() == _native.ABI_VERSION
    assert lib.lynx_status_string(0) == b"ok"
    assert lib.lynx_status_string(-3) == b"min_experts must be >= top_k"


def test_host_side_validation_needs_no_gpu():
    """Argument validation runs before any CUDA call, mirroring ValidationError sites."""
    from paper_2411_08982_b200 import _native
    lib = _native.load()
    assert lib.lynx_route_select(None, 4, 8, 9, 1, None, None, None) == -2   # k > N (router.py:176)
    assert lib.lynx_route_select(None, 0, 8, 2, 1, None, None, None) == -1   # empty logits
    assert lib.lynx_route_select(None, 4, 65, 2, 1, None, None, None) == -7  # > LYNX_MAX_EXPERTS
    pol = _native.LynxPolicy(mode=1, drop_count=1, confidence_threshold=0.5, sample_threshold=8,
                             min_experts=1, freq_keep_budget=4)
    sel = _native.LynxSelection(expert_ids=1, probs=1, full_probs=1, conf=1, assigned=1, weights=1, flags=1)
    ref = lambda s: ctypes.cast(ctypes.pointer(s), ctypes.c_void_p)  # noqa: E731
    assert lib.lynx_route_select(1, 4, 8, 2, 1, ref(pol), ref(sel), None) == -3  # min_experts < k
    pol.min_experts = 0
    pol.sample_threshold = 0
    assert lib.lynx_route_select(1, 4, 8, 2, 1, ref(pol), ref(sel), None) == -9


def test_dispatch_caps_and_workspace_sizes():
    from paper_2411_08982_b200 import _native
    lib = _native.load()
    ms, rc = ctypes.c_int32(), ctypes.c_int32()
    assert lib.lynx_dispatch_caps(32, 8, 2, ctypes.byref(ms), ctypes.byref(rc)) == 0
    assert ms.value >= 8 and rc.value >= 64 + 15 * 8 and rc.value % 16 == 0
    layer = _native.LynxLayer(num_experts=8, top_k=2, d_model=4096, d_ff=14336, activation=0, w13=1, w2=1)
    ws = lib.lynx_moe_workspace_bytes(ctypes.cast(ctypes.pointer(layer), ctypes.c_void_p), 32)
    assert 0 < ws < 64 << 20


def test_product_path_fails_loudly_without_library(tmp_path):
    from paper_2411_08982_b200 import _native
    from paper_2411_08982_b200.errors import NativeLibraryError
    saved = _native._lib
    _native._lib = None
    try:
        with pytest.raises(NativeLibraryError):
            _native.load(str(tmp_path / "missing.so"))
    finally:
        _native._lib = saved


def test_new_entry_points_validate_without_gpu():
    """Decode-stack, trace-ring and peer-memory EP entry points reject bad
    arguments before touching CUDA."""
    from paper_2411_08982_b200 import _native
    lib = _native.load()
    assert lib.lynx_attention(None, None, 1, 1, 0, None, None, None, 0, None) == -1
    a = _native.LynxAttention(d_model=4096, d_head=128, max_len=8, wqkv=1, wo=1, k_cache=1, v_cache=1)
    ref = lambda s: ctypes.cast(ctypes.pointer(s), ctypes.c_void_p)  # noqa: E731
    assert lib.lynx_attention(ref(a), 1, 2, 1, 0, 1, 1, 1, 1 << 20, None) == -7  # d_head > LYNX_MAX_DHEAD
    a.d_head = 16
    assert lib.lynx_attention(ref(a), 1, 2, 1, 0, 1, 1, 1, 0, None) == -8        # workspace too small
    assert lib.lynx_attention_workspace_bytes(64, 16) >= 64 * 16 * 4
    assert lib.lynx_advance_position(None, 1, None) == -1
    assert lib.lynx_trace_append(None, None, 0, None, None) == -1
    assert lib.lynx_ep_p2p_route(None, None, 4096, 8, None, None) == -1
    p = _native.LynxEPPeers(world_size=2, rank=2, tokens_per_rank=4)
    assert lib.lynx_ep_p2p_combine(1, 4096, 1, ref(p), None) == -1             # rank out of range
    assert lib.lynx_ep_p2p_dispatch(1, 8, 2, 4096, 1, None, None, None, None) == -1
