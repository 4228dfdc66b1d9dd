"""MoE decode layer on the GPU -- mirror of the hot-path part of
moetrim.simulator (simulator.py:26-113, 245-266).

* ``MoEWeights``     -- the per-layer expert/router weights in the layouts the
                        kernels stream (bf16, K-major), i.e. the ``model``
                        argument of ``forward_layer``.
* ``router_logits``  -- simulator.py:82-83 (K0: RMSNorm fused into the GEMV).
* ``forward_layer``  -- simulator.py:86-113 (K2 permute -> K3 grouped expert
                        GEMM on tcgen05 -> K4 combine), same signature.
* ``LynxMoELayer``   -- the whole decode layer (_apply_routing + forward_layer,
                        simulator.py:245-266 + 86-113) as one stream-ordered,
                        graph-capturable C call (lynx_moe_layer).

Expert activations: ``"swiglu"`` (Mixtral's expert, the north-star path) or
``"tanh2"`` (the reference's own ``tanh(x @ w1) @ w2``, simulator.py:77-79).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _native as nat
from .errors import ValidationError
from .policy import ExpertMask, PolicyConfig
from .router import MoEModelSpec, Phase, ctypes_ref


def _torch():
    import torch
    return torch


ACTIVATIONS = {"swiglu": nat.ACT_SWIGLU, "tanh2": nat.ACT_TANH2}


def swiglu_rows(ff: int) -> int:
    """Rows of the packed gate/up matrix per expert (2 * ceil64(ff))."""
    return 2 * ((ff + 63) // 64) * 64


def w13_row_of(f: int, up: bool) -> int:
    """Packed row holding feature f of w1 (up=False) or w3 (up=True) -- lynx_pack_w13."""
    return 128 * (f // 64) + 32 * ((f % 64) // 16) + (16 if up else 0) + f % 16


def unpack_w13(w13, ff: int):
    """Inverse of lynx_pack_w13: packed [N, rows, d] -> (w1, w3) each [N, ff, d]."""
    torch = _torch()
    f = torch.arange(ff)
    gate = 128 * (f // 64) + 32 * ((f % 64) // 16) + f % 16
    idx = gate.to(w13.device)
    return w13[:, idx], w13[:, idx + 16]


def pack_w13(w1, w3):
    """HF gate/up projections [N, ff, d] (bf16, CUDA) -> packed w13 (lynx_pack_w13 kernel)."""
    torch = _torch()
    N, ff, d = w1.shape
    w13 = torch.empty((N, swiglu_rows(ff), d), dtype=torch.bfloat16, device=w1.device)
    nat.check(nat.lib().lynx_pack_w13(nat.ptr(w1.contiguous()), nat.ptr(w3.contiguous()), N, ff, d,
                                      nat.ptr(w13), nat.stream_handle()), "pack_w13")
    return w13


@dataclass
class MoEWeights:
    """Device weights of an MoE stack, per layer (the ``model`` of forward_layer).

    swiglu: w13[l] packed [N, 2*ceil64(ff), d], w2[l] [N, d, ff]
    tanh2:  w13[l] = w1^T [N, ff, d], w2[l] = w2^T [N, d, ff]
    router_wt[l] = router_w^T [N, d]; all bf16, contiguous, CUDA.
    """

    spec: MoEModelSpec
    activation: str
    w13: list
    w2: list
    router_wt: list
    _native: dict = field(default_factory=dict, repr=False)

    def native_layer(self, layer: int) -> nat.LynxLayer:
        if layer not in self._native:
            s = self.spec
            L = nat.LynxLayer()
            L.num_experts, L.top_k, L.d_model, L.d_ff = s.num_experts, s.top_k, s.d_model, s.d_ff
            L.activation = ACTIVATIONS[self.activation]
            L.num_shared = s.num_shared_experts
            L.w13 = nat.ptr(self.w13[layer])
            L.w2 = nat.ptr(self.w2[layer])
            L.router_wt = nat.ptr(self.router_wt[layer]) if self.router_wt[layer] is not None else 0
            self._native[layer] = L
        return self._native[layer]

    def expert_bytes(self) -> int:
        """Bytes streamed per used expert per layer (all three projections, bf16)."""
        s = self.spec
        return 3 * s.d_model * s.d_ff * 2 if self.activation == "swiglu" else 2 * s.d_model * s.d_ff * 2


def build_swiglu_model(spec: MoEModelSpec, seed: int = 0, router_gain: float = 2.0, expert_gain: float = 1.0,
                       device: str = "cuda") -> MoEWeights:
    """Random-init SwiGLU stack (SURVEY 8d recipe, after simulator.py:44-74):
    router ~ N(0, (gain/sqrt(d))^2), W1, W3 ~ N(0, 1/d), W2 ~ N(0, (expert_gain *
    out_damp / sqrt(ff))^2) with the reference's depth damping out_damp =
    1/sqrt(2L) (simulator.py:64-73), so a deep stack keeps bounded hidden
    norms; bf16.  Shared experts (spec.num_shared_experts) are experts
    N..N+S-1 of w13/w2."""
    torch = _torch()
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    N, d, ff = spec.num_experts, spec.d_model, spec.d_ff
    E = N + spec.num_shared_experts
    w13s, w2s, routers = [], [], []
    for _ in range(spec.num_layers):
        w13 = torch.randn((E, swiglu_rows(ff), d), generator=g, device=device, dtype=torch.bfloat16)
        w13.mul_(1.0 / np.sqrt(d))
        if ff % 64:  # zero the padding features of the packed layout
            f = torch.arange(ff, swiglu_rows(ff) // 2)
            for up in (False, True):
                rows = 128 * (f // 64) + 32 * ((f % 64) // 16) + (16 if up else 0) + f % 16
                w13[:, rows.to(device)] = 0
        w2 = torch.randn((E, d, ff), generator=g, device=device, dtype=torch.bfloat16)
        w2.mul_(expert_gain / np.sqrt(2.0 * spec.num_layers) / np.sqrt(ff))
        r = torch.randn((N, d), generator=g, device=device, dtype=torch.bfloat16)
        r.mul_(router_gain / np.sqrt(d))
        w13s.append(w13)
        w2s.append(w2)
        routers.append(r)
    return MoEWeights(spec, "swiglu", w13s, w2s, routers)


def from_hf_swiglu(spec: MoEModelSpec, w1: list, w3: list, w2: list, router: list) -> MoEWeights:
    """Per-layer HF Mixtral tensors: w1/w3 [N, ff, d], w2 [N, d, ff], router [N, d]."""
    torch = _torch()
    cast = lambda t: t.to(device="cuda", dtype=torch.bfloat16).contiguous()  # noqa: E731
    return MoEWeights(spec, "swiglu", [pack_w13(cast(a), cast(b)) for a, b in zip(w1, w3)],
                      [cast(t) for t in w2], [cast(t) for t in router])


def from_reference(model) -> MoEWeights:
    """A moetrim.simulator.SyntheticMoE (simulator.py:30-41) as bf16 tanh2 weights.

    Duck-typed: needs ``spec``, ``router_w [L,d,N]``, ``w1 [L,N,d,ff]``, ``w2 [L,N,ff,d]``.
    """
    torch = _torch()
    s = model.spec
    spec = MoEModelSpec(s.num_layers, s.num_experts, s.top_k, s.d_model, s.d_ff, s.bytes_per_param)
    bf = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).to(  # noqa: E731
        "cuda").to(torch.bfloat16).contiguous()
    w1t = [bf(np.transpose(model.w1[l], (0, 2, 1))) for l in range(s.num_layers)]
    w2t = [bf(np.transpose(model.w2[l], (0, 2, 1))) for l in range(s.num_layers)]
    rt = [bf(np.transpose(model.router_w[l])) for l in range(s.num_layers)]
    return MoEWeights(spec, "tanh2", w1t, w2t, rt)


# ----------------------------------------------------------------- workspace
_WS: dict = {}


def _workspace(layer: nat.LynxLayer, T: int):
    torch = _torch()
    nbytes = int(nat.lib().lynx_moe_workspace_bytes(ctypes_ref(layer), T))
    key = (torch.cuda.current_device(), nbytes)
    buf = _WS.get(key)
    if buf is None:
        buf = torch.empty((nbytes,), dtype=torch.uint8, device="cuda")
        _WS[key] = buf
    return buf


def _hidden_bf16(hidden, d: int):
    torch = _torch()
    if isinstance(hidden, torch.Tensor):
        h = hidden.to(device="cuda", dtype=torch.bfloat16)
    else:
        h = torch.from_numpy(np.ascontiguousarray(np.asarray(hidden, dtype=np.float32))).to("cuda").to(
            torch.bfloat16)
    if h.ndim != 2 or h.shape[1] != d:
        raise ValidationError(f"hidden must be [T, {d}], got {tuple(h.shape)}")
    return h.contiguous()


def router_logits(model: MoEWeights, layer: int, hidden):
    """rms_norm(hidden) @ router_w (simulator.py:26-27, 82-83) -> float64 [T, N]."""
    torch = _torch()
    s = model.spec
    h = _hidden_bf16(hidden, s.d_model)
    out = torch.empty((h.shape[0], s.num_experts), dtype=torch.float64, device="cuda")
    nat.check(nat.lib().lynx_router_logits(nat.ptr(h), nat.ptr(model.router_wt[layer]), h.shape[0], s.d_model,
                                           s.num_experts, nat.ptr(out), nat.stream_handle()), "router_logits")
    return out


def forward_layer(hidden, model: MoEWeights, layer_index: int, mask: ExpertMask):
    """MoE sublayer: residual + weighted sum of the assigned experts (simulator.py:86-113).

    Returns bf16 [T, d] on the GPU.  Only experts with at least one assigned
    slot are read from HBM.
    """
    torch = _torch()
    s = model.spec
    h = _hidden_bf16(hidden, s.d_model)
    if h.shape[0] != mask.num_tokens:
        raise ValidationError(f"mask covers {mask.num_tokens} tokens but hidden has {h.shape[0]}")
    T = int(h.shape[0])
    layer = model.native_layer(layer_index)
    assigned = mask.remap_assigned.to(device="cuda", dtype=torch.int32).contiguous()
    weights = mask.remap_weights.to(device="cuda", dtype=torch.float64).contiguous()
    ws = _workspace(layer, T)
    out = torch.empty_like(h)
    nat.check(nat.lib().lynx_moe_forward(ctypes_ref(layer), nat.ptr(h), T, nat.ptr(assigned), nat.ptr(weights),
                                         nat.ptr(out), nat.ptr(ws), ws.numel(), nat.stream_handle()),
              "forward_layer")
    return out


def forward_partial(hidden, model: MoEWeights, layer_index: int, assigned, weights):
    """f32 sum of expert outputs without the residual; assigned < 0 skipped (EP helper)."""
    torch = _torch()
    s = model.spec
    h = _hidden_bf16(hidden, s.d_model)
    T = int(h.shape[0])
    layer = model.native_layer(layer_index)
    ws = _workspace(layer, T)
    out = torch.empty((T, s.d_model), dtype=torch.float32, device="cuda")
    nat.check(nat.lib().lynx_moe_forward_partial(ctypes_ref(layer), nat.ptr(h), T, nat.ptr(assigned),
                                                 nat.ptr(weights), nat.ptr(out), nat.ptr(ws), ws.numel(),
                                                 nat.stream_handle()), "forward_partial")
    return out


class LynxMoELayer:
    """The whole decode MoE layer as one C call (lynx_moe_layer):

        K0 router GEMV + RMSNorm -> K1 route + Lynx policy + remap ->
        K2 histogram/scan permutation + gather -> K3 grouped expert GEMM
        (tcgen05, used experts only) -> K4 weighted combine + residual.

    Shapes are fixed at construction; buffers are preallocated, so calls
    never synchronise the host and can be captured into a CUDA graph.
    The selection/mask outputs stay on the device (``.expert_ids``,
    ``.assigned``, ``.weights``, ``.retained_mask``, ``.flags`` ...).
    """

    def __init__(self, model: MoEWeights, layer_index: int, num_tokens: int,
                 policy: PolicyConfig | None = None, phase: Phase = Phase.DECODE, workspace=None):
        torch = _torch()
        s = model.spec
        self.model, self.layer_index, self.T = model, layer_index, int(num_tokens)
        self.phase = phase
        if policy is not None:
            if phase is Phase.DECODE:
                policy.resolved_min_experts(s.top_k)
            self._pol = policy.to_native()
        else:
            self._pol = None
        self._layer = model.native_layer(layer_index)
        nbytes = int(nat.lib().lynx_moe_workspace_bytes(ctypes_ref(self._layer), self.T))
        if workspace is not None and workspace.numel() >= nbytes:
            self.workspace = workspace  # shared by layers that run in stream order
        else:
            # zero-filled once: the fused front's barrier words start at zero (every call leaves them zero)
            self.workspace = torch.zeros((nbytes,), dtype=torch.uint8, device="cuda")
        T, N, k = self.T, s.num_experts, s.top_k
        dev = "cuda"
        self.expert_ids = torch.empty((T, k), dtype=torch.int32, device=dev)
        self.probs = torch.empty((T, k), dtype=torch.float64, device=dev)
        self.full_probs = torch.empty((T, N), dtype=torch.float64, device=dev)
        self.conf = torch.empty((T,), dtype=torch.float64, device=dev)
        self.counts = torch.empty((N,), dtype=torch.float64, device=dev)
        self.retained_mask = torch.empty((N,), dtype=torch.uint8, device=dev)
        self.assigned = torch.empty((T, k), dtype=torch.int32, device=dev)
        self.weights = torch.empty((T, k), dtype=torch.float64, device=dev)
        self.important = torch.empty((T,), dtype=torch.uint8, device=dev)
        self.flags = torch.zeros((1,), dtype=torch.int32, device=dev)
        self._sel = nat.LynxSelection(
            expert_ids=nat.ptr(self.expert_ids), probs=nat.ptr(self.probs), full_probs=nat.ptr(self.full_probs),
            conf=nat.ptr(self.conf), counts=nat.ptr(self.counts), retained=nat.ptr(self.retained_mask),
            assigned=nat.ptr(self.assigned), weights=nat.ptr(self.weights), important=nat.ptr(self.important),
            flags=nat.ptr(self.flags))
        self._lib = nat.lib()
        self._sel_ref = ctypes_ref(self._sel)
        self._layer_ref = ctypes_ref(self._layer)
        self._pol_ref = ctypes_ref(self._pol) if self._pol is not None else None

    def __call__(self, hidden, out=None, logits=None):
        """The layer on device-resident ``hidden`` [T, d] bf16.  ``logits``
        (f64 [T, N], e.g. from the decode stack's fused router) skips K0."""
        torch = _torch()
        if hidden.dtype != torch.bfloat16 or not hidden.is_cuda or tuple(hidden.shape) != (
                self.T, self.model.spec.d_model):
            raise ValidationError(f"hidden must be a CUDA bf16 tensor of shape [{self.T}, "
                                  f"{self.model.spec.d_model}]")
        if out is None:
            out = torch.empty_like(hidden)
        decode = 1 if self.phase is Phase.DECODE else 0
        stream = torch.cuda.current_stream().cuda_stream
        if logits is not None:
            st = self._lib.lynx_moe_layer_logits(self._layer_ref, hidden.data_ptr(), logits.data_ptr(), self.T,
                                                 decode, self._pol_ref, out.data_ptr(), self._sel_ref,
                                                 self.workspace.data_ptr(), self.workspace.numel(), stream)
            nat.check(st, "lynx_moe_layer_logits")
            return out
        st = self._lib.lynx_moe_layer(self._layer_ref, hidden.data_ptr(), self.T, decode, self._pol_ref,
                                      out.data_ptr(), self._sel_ref, self.workspace.data_ptr(),
                                      self.workspace.numel(), stream)
        nat.check(st, "lynx_moe_layer")
        return out

    def host_step(self, hidden_host, out_host):
        """One decode-layer step on PINNED HOST buffers: host->device copy of
        ``hidden_host`` [T, d] bf16, the layer (K0..K4), device->host copy into
        ``out_host``.  The three are captured once per buffer pair into a CUDA
        graph and replayed on the current stream, so a step costs one graph
        launch.  Returns ``out_host``; it is valid after the stream syncs."""
        torch = _torch()
        d = self.model.spec.d_model
        for t in (hidden_host, out_host):
            if t.is_cuda or t.dtype != torch.bfloat16 or tuple(t.shape) != (self.T, d) or not t.is_pinned():
                raise ValidationError(f"host_step takes pinned host bf16 tensors of shape [{self.T}, {d}]")
        key = (hidden_host.data_ptr(), out_host.data_ptr())
        graphs = self.__dict__.setdefault("_host_graphs", {})
        if key not in graphs:
            dev_in = torch.empty((self.T, d), dtype=torch.bfloat16, device="cuda")
            dev_out = torch.empty_like(dev_in)
            side = torch.cuda.Stream()
            side.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(side):  # warm-up outside capture (lazy init, TMA descriptors)
                dev_in.copy_(hidden_host, non_blocking=True)
                self(dev_in, dev_out)
            torch.cuda.current_stream().wait_stream(side)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                dev_in.copy_(hidden_host, non_blocking=True)
                self(dev_in, dev_out)
                out_host.copy_(dev_out, non_blocking=True)
            graphs[key] = (g, dev_in, dev_out)
        graphs[key][0].replay()
        return out_host

    def stream_host(self, hidden_hosts, out_hosts):
        """Run the layer over a sequence of PINNED HOST batches with the PCIe
        copies overlapped: while the layer (one graph replay) computes batch
        i, a copy stream moves batch i+1 host->device and batch i-1's output
        device->host.  Double-buffered device slots; every batch's own H2D and
        D2H still happens, they just hide behind the neighbouring batches'
        expert streams.  Results land in ``out_hosts``; the current stream
        is ordered after the last copy on return (no host sync)."""
        torch = _torch()
        n = len(hidden_hosts)
        if n != len(out_hosts):
            raise ValidationError("stream_host needs one output buffer per input batch")
        d = self.model.spec.d_model
        for t in list(hidden_hosts) + list(out_hosts):
            if t.is_cuda or t.dtype != torch.bfloat16 or tuple(t.shape) != (self.T, d) or not t.is_pinned():
                raise ValidationError(f"stream_host takes pinned host bf16 tensors of shape [{self.T}, {d}]")
        st = self.__dict__.get("_stream_state")
        if st is None:
            dev_in = [torch.empty((self.T, d), dtype=torch.bfloat16, device="cuda") for _ in range(2)]
            dev_out = [torch.empty_like(dev_in[0]) for _ in range(2)]
            side = torch.cuda.Stream()
            side.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(side):
                for s_ in range(2):
                    self(dev_in[s_], dev_out[s_])  # warm-up outside capture
            torch.cuda.current_stream().wait_stream(side)
            graphs = []
            for s_ in range(2):
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    self(dev_in[s_], dev_out[s_])
                graphs.append(g)
            st = dict(dev_in=dev_in, dev_out=dev_out, graphs=graphs, copy=torch.cuda.Stream())
            self._stream_state = st
        cs, xs = torch.cuda.current_stream(), st["copy"]
        ev = lambda: torch.cuda.Event()  # noqa: E731
        in_ready, computed, out_copied = [ev(), ev()], [ev(), ev()], [ev(), ev()]
        xs.wait_stream(cs)
        with torch.cuda.stream(xs):
            st["dev_in"][0].copy_(hidden_hosts[0], non_blocking=True)
            in_ready[0].record(xs)
        for i in range(n):
            s_ = i % 2
            if i + 1 < n:  # next input into the other slot once batch i-1 is done reading it
                with torch.cuda.stream(xs):
                    if i >= 1:
                        xs.wait_event(computed[1 - s_])
                    st["dev_in"][1 - s_].copy_(hidden_hosts[i + 1], non_blocking=True)
                    in_ready[1 - s_].record(xs)
            cs.wait_event(in_ready[s_])
            if i >= 2:
                cs.wait_event(out_copied[s_])  # batch i-2's output has left this slot
            st["graphs"][s_].replay()
            computed[s_].record(cs)
            with torch.cuda.stream(xs):
                xs.wait_event(computed[s_])
                out_hosts[i].copy_(st["dev_out"][s_], non_blocking=True)
                out_copied[s_].record(xs)
        cs.wait_stream(xs)
        return out_hosts

    def profiled(self, hidden, events, out=None):
        """__call__ that records 6 torch.cuda.Events around K0..K4 (lynx_moe_layer_profiled)."""
        torch = _torch()
        if out is None:
            out = torch.empty_like(hidden)
        stream = torch.cuda.current_stream()
        handles = (ctypes.c_void_p * 6)()
        for i, ev in enumerate(events):
            if not ev.cuda_event:
                ev.record(stream)  # torch creates CUDA events lazily
            handles[i] = ev.cuda_event
        st = self._lib.lynx_moe_layer_profiled(self._layer_ref, hidden.data_ptr(), self.T,
                                               1 if self.phase is Phase.DECODE else 0, self._pol_ref,
                                               out.data_ptr(), self._sel_ref, self.workspace.data_ptr(),
                                               self.workspace.numel(), stream.cuda_stream,
                                               ctypes.cast(handles, ctypes.c_void_p), 6)
        nat.check(st, "lynx_moe_layer_profiled")
        return out

    def ffn_kernel(self) -> str:
        """The K3 kernel this layer launches: "ffn_pair_kernel" (tcgen05
        cta_group::2, wide expert segments) or "ffn_kernel" (lynx_moe_ffn_kernel)."""
        rows = ctypes.c_int32()
        r = self._lib.lynx_moe_ffn_kernel(self._layer_ref, self.T, 1 if self.phase is Phase.DECODE else 0,
                                          self._pol_ref, ctypes.byref(rows))
        if r < 0:
            nat.check(r, "lynx_moe_ffn_kernel")
        return "ffn_pair_kernel" if r == 1 else "ffn_kernel"

    def used_experts(self) -> int:
        """Experts streamed by the last call: routed experts with >= 1 assigned
    slot plus the shared experts (host sync; reporting only)."""
        torch = _torch()
        s = self.model.spec
        used = torch.bincount(self.assigned.flatten().long(), minlength=s.num_experts) > 0
        return int(used.sum().item()) + s.num_shared_experts

    def mask(self) -> ExpertMask:
        """The last call's ExpertMask (host sync)."""
        torch = _torch()
        flags = int(self.flags.item())
        return ExpertMask(layer_index=self.layer_index, phase=self.phase,
                          retained=torch.nonzero(self.retained_mask).flatten().long(),
                          remap_original=self.expert_ids.clone(), remap_assigned=self.assigned.clone(),
                          remap_weights=self.weights.clone(), clipped=bool(flags & nat.FLAG_CLIPPED),
                          important_tokens=torch.nonzero(self.important).flatten().long())
