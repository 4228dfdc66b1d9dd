"""The decode loop around the MoE layer -- mirror of moetrim.simulator.simulate
(simulator.py:273-357) on the GPU.

Per layer and routing event the reference does

    h = h + attention(layer, h, offset)           simulator.py:333
    selection, mask = _apply_routing(...)         simulator.py:335-337
    h = forward_layer(h, model, layer, mask)      simulator.py:340

over a prefill chunk (all B*P tokens, Phase.PREFILL) and then one token per
sequence per decode step (Phase.DECODE), each decode step fed rms_norm of
the previous step's final state (simulator.py:351-355).

Here every layer is two attention kernels (lynx_attention: the single-head
stand-in with its KV cache and residual) followed by the whole Lynx MoE
decode layer (lynx_moe_layer: K0..K4).  A decode step of all layers is
captured ONCE into a CUDA graph and replayed; the cache position lives in
device memory and is advanced inside the graph, so a step is one graph
launch with no host work.  Hidden states between layers are bf16.

The retention policy plays the reference's ``Intervention(kind="policy")``
(simulator.py:114-170): it applies to the layers in ``policy_layers``
(default all) during decode; prefill always uses the identity mask
(the policies are identity for PREFILL, policy.py:244-245, 300-301).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native as nat
from .errors import ValidationError
from .moe import LynxMoELayer, MoEWeights
from .policy import PolicyConfig
from .router import Phase, ctypes_ref


def _torch():
    import torch
    return torch


@dataclass
class AttentionWeights:
    """Per-layer attention stand-in weights (simulator.py:35-38), bf16 on the GPU.

    wqkv[l] = [wq^T; wk^T; wv^T]  [3*dh, d];  wo[l] = wo  [dh, d].
    """

    d_head: int
    wqkv: list
    wo: list


def build_attention(num_layers: int, d_model: int, d_head: int = 16, seed: int = 0, attn_gain: float = 1.5,
                    device: str = "cuda") -> AttentionWeights:
    """Random-init attention weights with the reference's scales (simulator.py:62-71):
    wq, wk, wv ~ N(0, 1/d); wo ~ N(0, (attn_gain / sqrt(2L) / sqrt(dh))^2)."""
    torch = _torch()
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    out_damp = 1.0 / np.sqrt(2.0 * num_layers)
    wqkv, wo = [], []
    for _ in range(num_layers):
        a = torch.randn((3 * d_head, d_model), generator=g, device=device, dtype=torch.float32)
        wqkv.append((a / np.sqrt(d_model)).to(torch.bfloat16).contiguous())
        o = torch.randn((d_head, d_model), generator=g, device=device, dtype=torch.float32)
        wo.append((o * (attn_gain * out_damp / np.sqrt(d_head))).to(torch.bfloat16).contiguous())
    return AttentionWeights(d_head, wqkv, wo)


def attention_from_reference(model) -> AttentionWeights:
    """A moetrim SyntheticMoE's wq/wk/wv [L, d, dh] and wo [L, dh, d] as bf16 device weights."""
    torch = _torch()
    L = model.spec.num_layers
    bf = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).to(  # noqa: E731
        "cuda").to(torch.bfloat16).contiguous()
    wqkv = [bf(np.concatenate([model.wq[l].T, model.wk[l].T, model.wv[l].T], axis=0)) for l in range(L)]
    wo = [bf(model.wo[l]) for l in range(L)]
    return AttentionWeights(int(model.d_head), wqkv, wo)


@dataclass
class SimResult:
    """simulator.py:240-244: final-layer states per position [B, P + D, d]."""

    hidden: object
    prefill_len: int
    decode_steps: int


class DecodeStack:
    """simulate() for one batch of B sequences on one GPU.

    ``prefill(inputs)`` runs the prefill chunk; ``step()`` one decode step
    (a CUDA-graph replay after the first call); ``simulate(inputs, steps)``
    both, returning the reference's SimResult layout.  ``trace`` (optional,
    a ``trace.TraceRecorder``) records every routing event on the device.
    """

    def __init__(self, moe: MoEWeights, attn: AttentionWeights, batch: int, max_len: int,
                 policy: PolicyConfig | None = None, policy_layers=None, graph: bool = True, trace=None,
                 probe=None):
        torch = _torch()
        s = moe.spec
        if len(attn.wqkv) != s.num_layers:
            raise ValidationError("attention weights and MoE weights have different layer counts")
        self.moe, self.attn, self.B, self.max_len = moe, attn, int(batch), int(max_len)
        self.L, self.d = s.num_layers, s.d_model
        self.policy = policy
        self.policy_layers = None if policy_layers is None else frozenset(int(l) for l in policy_layers)
        self.graph_enabled = graph
        self.trace = trace
        # probe(layer, phase, h_in, h_mid, h_out, lynx_layer): eager-only hook
        # on every layer's input, post-attention and output (tests)
        self.probe = probe
        if probe is not None:
            self.graph_enabled = False
        dev = "cuda"
        self.k_cache = torch.zeros((self.L, self.B, self.max_len, attn.d_head), dtype=torch.float32, device=dev)
        self.v_cache = torch.zeros_like(self.k_cache)
        self.pos = torch.zeros((1,), dtype=torch.int32, device=dev)
        # Decode steps fuse the next MoE layer's router into the attention
        # output kernel: logits come out with h, K0 drops out.
        self.fused_router = (s.num_experts <= nat.MAX_FUSED_ROUTER and self.d <= 8192 and
                             all(r is not None for r in moe.router_wt))
        self.logits = torch.empty((self.B, s.num_experts), dtype=torch.float64, device=dev)
        self._attn, self._attn_dec = [], []
        for l in range(self.L):
            for fused, lst in ((False, self._attn), (self.fused_router, self._attn_dec)):
                a = nat.LynxAttention()
                a.d_model, a.d_head, a.max_len = self.d, attn.d_head, self.max_len
                a.wqkv, a.wo = nat.ptr(attn.wqkv[l]), nat.ptr(attn.wo[l])
                a.k_cache, a.v_cache = nat.ptr(self.k_cache[l]), nat.ptr(self.v_cache[l])
                if fused:
                    a.num_experts, a.router_wt, a.logits = s.num_experts, nat.ptr(moe.router_wt[l]), nat.ptr(self.logits)
                lst.append(a)
        self._attn_refs = [ctypes_ref(a) for a in self._attn]
        self._attn_dec_refs = [ctypes_ref(a) for a in self._attn_dec]
        # one MoE workspace shared by every layer (they run in stream order)
        self._decode_layers = self._make_layers(self.B, Phase.DECODE)
        self.prev = torch.zeros((self.B, self.d), dtype=torch.bfloat16, device=dev)
        self._mid = torch.empty_like(self.prev)
        self._alt = [torch.empty_like(self.prev), torch.empty_like(self.prev)]
        # zeroed: holds the fused router's per-row arrival counters (kernel re-arms them)
        self._attn_ws = torch.zeros((int(nat.lib().lynx_attention_workspace_bytes(self.B, attn.d_head)),),
                                    dtype=torch.uint8, device=dev)
        self._graph = None
        self.steps_done = 0

    # ------------------------------------------------------------ helpers
    def _layer_policy(self, l: int, phase: Phase):
        if self.policy is None or phase is not Phase.DECODE:
            return None
        if self.policy_layers is not None and l not in self.policy_layers:
            return None
        return self.policy

    def _make_layers(self, T: int, phase: Phase):
        torch = _torch()
        layers, ws = [], None
        for l in range(self.L):
            layer = LynxMoELayer(self.moe, l, T, policy=self._layer_policy(l, phase), phase=phase, workspace=ws)
            ws = layer.workspace
            layers.append(layer)
        torch.cuda.synchronize()
        return layers

    def _attention(self, l: int, h_in, T_new: int, norm_input: bool, h_out, ws, fused: bool = False):
        torch = _torch()
        ref = self._attn_dec_refs[l] if fused else self._attn_refs[l]
        st = nat.lib().lynx_attention(ref, h_in.data_ptr(), self.B, T_new, 1 if norm_input else 0,
                                      self.pos.data_ptr(), h_out.data_ptr(), ws.data_ptr(), ws.numel(),
                                      torch.cuda.current_stream().cuda_stream)
        nat.check(st, "lynx_attention")

    def _advance(self, by: int):
        torch = _torch()
        nat.check(nat.lib().lynx_advance_position(self.pos.data_ptr(), by, torch.cuda.current_stream().cuda_stream),
                  "lynx_advance_position")

    # ------------------------------------------------------------ prefill
    def prefill(self, inputs):
        """The prefill chunk (simulator.py:349-350): inputs [B, P, d] -> final states [B, P, d] (bf16)."""
        torch = _torch()
        x = inputs if isinstance(inputs, torch.Tensor) else torch.from_numpy(np.asarray(inputs, dtype=np.float32))
        if x.ndim != 3 or x.shape[0] != self.B or x.shape[2] != self.d:
            raise ValidationError(f"inputs must be [{self.B}, prefill_len, {self.d}]")
        P = int(x.shape[1])
        if P < 1:
            raise ValidationError("prefill_len must be >= 1")
        if P > self.max_len:
            raise ValidationError("prefill_len exceeds the cache capacity")
        h = x.to(device="cuda", dtype=torch.bfloat16).reshape(self.B * P, self.d).contiguous()
        layers = self._make_layers(self.B * P, Phase.PREFILL)
        ws = torch.empty((int(nat.lib().lynx_attention_workspace_bytes(self.B * P, self.attn.d_head)),),
                         dtype=torch.uint8, device="cuda")
        self.pos.zero_()
        self.steps_done = 0
        mid, out = torch.empty_like(h), torch.empty_like(h)
        for l in range(self.L):
            self._attention(l, h, P, False, mid, ws)
            layers[l](mid, out)
            if self.probe is not None:
                self.probe(l, Phase.PREFILL, h, mid, out, layers[l])
            if self.trace is not None:
                self.trace.record(l, Phase.PREFILL, layers[l], event_offset=0)
            h, out = out, h
        self._advance(P)
        self.prefill_len = P
        hp = h.reshape(self.B, P, self.d)
        self.prev.copy_(hp[:, -1])
        return hp

    # ------------------------------------------------------------ decode
    def _step_body(self):
        h = self.prev
        for l in range(self.L):
            self._attention(l, h, 1, l == 0, self._mid, self._attn_ws, fused=self.fused_router)
            dst = self.prev if l == self.L - 1 else self._alt[l % 2]
            if self.probe is not None:
                h_in = h.clone()
            self._decode_layers[l](self._mid, dst, logits=self.logits if self.fused_router else None)
            if self.probe is not None:
                self.probe(l, Phase.DECODE, h_in, self._mid, dst, self._decode_layers[l])
            if self.trace is not None:
                self.trace.record_device(l, self._decode_layers[l], self.pos)
            h = dst
        self._advance(1)

    def step(self):
        """One decode step over all layers; returns the final states [B, d]
        (``self.prev``, overwritten by the next step)."""
        torch = _torch()
        if self.graph_enabled:
            if self._graph is None:
                # capture from a scratch copy of the state, then restore it
                saved = (self.prev.clone(), self.pos.clone(), self.k_cache.clone(), self.v_cache.clone())
                side = torch.cuda.Stream()
                side.wait_stream(torch.cuda.current_stream())
                with torch.cuda.stream(side):
                    self._step_body()  # warm-up outside capture
                torch.cuda.current_stream().wait_stream(side)
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    self._step_body()
                self.prev.copy_(saved[0])
                self.pos.copy_(saved[1])
                self.k_cache.copy_(saved[2])
                self.v_cache.copy_(saved[3])
                if self.trace is not None:
                    self.trace.rewind()
                del saved
                self._graph = g
            self._graph.replay()
        else:
            self._step_body()
        if self.trace is not None:
            self.trace.step_done()
        self.steps_done += 1
        return self.prev

    def profile_step(self) -> dict:
        """One eager decode step with CUDA events around every kernel group;
        returns milliseconds per step split the way the reference's cost
        model calibration table is (costmodel.py:300-343): attention,
        routing (router GEMV + selection), MLP (gather + expert FFN +
        combine).  Event records serialise the programmatic launches, so
        the parts sum to slightly more than a graphed step."""
        torch = _torch()
        ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
        marks = []
        h = self.prev
        for l in range(self.L):
            a0, a1 = ev(), ev()
            k = [ev() for _ in range(6)]
            a0.record()
            self._attention(l, h, 1, l == 0, self._mid, self._attn_ws)  # unfused: K0 timed as routing
            a1.record()
            dst = self.prev if l == self.L - 1 else self._alt[l % 2]
            self._decode_layers[l].profiled(self._mid, k, dst)
            marks.append((a0, a1, k))
            h = dst
        self._advance(1)
        torch.cuda.synchronize()
        attn = sum(a0.elapsed_time(a1) for a0, a1, _ in marks)
        route = sum(k[0].elapsed_time(k[2]) for _, _, k in marks)
        mlp = sum(k[2].elapsed_time(k[5]) for _, _, k in marks)
        self.steps_done += 1
        return {"attn_ms": attn, "route_ms": route, "mlp_ms": mlp}

    def simulate(self, inputs, decode_steps: int) -> SimResult:
        """simulator.py:273-357 for one batch: prefill then decode_steps greedy steps."""
        torch = _torch()
        if decode_steps < 0:
            raise ValidationError("decode_steps must be >= 0")
        hp = self.prefill(inputs)
        P = hp.shape[1]
        if P + decode_steps > self.max_len:
            raise ValidationError("prefill_len + decode_steps exceeds the cache capacity")
        out = torch.empty((self.B, P + decode_steps, self.d), dtype=torch.bfloat16, device="cuda")
        out[:, :P] = hp
        for s in range(decode_steps):
            out[:, P + s] = self.step()
        return SimResult(hidden=out, prefill_len=P, decode_steps=decode_steps)
