"""Expert parallelism over NCCL: one process per GPU, rank g
owns experts [g*N/G, (g+1)*N/G), decode tokens are data-parallel (T_local
rows per rank).

Per layer step:
  1. K0 router GEMV on the local rows                       -> logits [T_l, N]
  2. all_gather of float64 logits                           -> logits [T, N]
  3. K1 route + Lynx policy on the GLOBAL batch; every rank computes the
     identical selection, so the batch vote is global and no count
     exchange is needed
  4. pack: row i goes to peer p iff token (rank, i) has a slot on one of
     p's experts (fixed capacity T_l rows per peer)
  5. all_to_all (dispatch) of bf16 rows                     -> [T, d] in global token order
  6. K2+K3+K4 on the local experts only (mask renumbered, others -1),
     f32 partial sums without residual
  7. all_to_all (combine) of f32 partials back to the owning rank
  8. residual + sum over peers in rank order (= experts ascending)

The collectives are torch.distributed calls (NCCL on GPUs, gloo in the CPU
tests); the compute steps are an ``EPOps`` object.  ``NativeEPOps`` runs
liblynx_b200 kernels; the CPU tests plug in oracle-backed ops to exercise
the same orchestration with world_size 2.
"""

from __future__ import annotations

from dataclasses import dataclass

from . import _native as nat
from .policy import PolicyConfig
from .router import ctypes_ref


def _torch():
    import torch
    return torch


@dataclass(frozen=True)
class EPShape:
    num_experts: int
    top_k: int
    d_model: int
    d_ff: int
    tokens_per_rank: int
    world_size: int
    rank: int

    @property
    def experts_per_rank(self) -> int:
        return self.num_experts // self.world_size

    @property
    def tokens(self) -> int:
        return self.tokens_per_rank * self.world_size


class EPOps:
    """Compute steps of an EP layer (overridden by the native and test backends)."""

    def router(self, hidden_local):  # -> float64 [T_l, N]
        raise NotImplementedError

    def select(self, logits_all):  # -> (assigned int32 [T,k], weights f64 [T,k])
        raise NotImplementedError

    def pack(self, hidden_local, assigned):  # -> bf16 [G*T_l, d]
        raise NotImplementedError

    def local_mask(self, assigned, weights):  # -> (assigned_local, weights_local)
        raise NotImplementedError

    def forward_partial(self, recv, assigned_local, weights_local):  # -> f32 [T, d]
        raise NotImplementedError

    def combine(self, hidden_local, back):  # -> bf16 [T_l, d]
        raise NotImplementedError


def ep_layer(shape: EPShape, ops: EPOps, hidden_local, group=None, mark=None):
    """One expert-parallel MoE decode layer (steps 1-8 above).  ``mark(i)``
    (optional, e.g. a CUDA event record) is called at the 8 phase
    boundaries: before the router (0), the logits all-gather (1), select +
    pack (2), the dispatch all-to-all (3), the expert FFN (4), the return
    all-to-all (5), the combine (6) and after it (7)."""
    torch = _torch()
    import torch.distributed as dist
    mark = mark or (lambda i: None)
    G, Tl, N, d = shape.world_size, shape.tokens_per_rank, shape.num_experts, shape.d_model
    mark(0)
    logits_local = ops.router(hidden_local)
    logits_all = torch.empty((G * Tl, N), dtype=logits_local.dtype, device=logits_local.device)
    mark(1)
    dist.all_gather_into_tensor(logits_all, logits_local.contiguous(), group=group)
    mark(2)
    assigned, weights = ops.select(logits_all)
    send = ops.pack(hidden_local, assigned)
    recv = torch.empty_like(send)
    mark(3)
    dist.all_to_all_single(recv, send, group=group)
    mark(4)
    assigned_local, weights_local = ops.local_mask(assigned, weights)
    partial = ops.forward_partial(recv.view(G * Tl, d), assigned_local, weights_local)
    back = torch.empty_like(partial)
    mark(5)
    dist.all_to_all_single(back, partial.contiguous(), group=group)
    mark(6)
    out = ops.combine(hidden_local, back.view(G, Tl, d))
    mark(7)
    return out


class NativeEPOps(EPOps):
    """EP compute on liblynx_b200 (all buffers preallocated; graph-safe).

    router_wt: the full router [N, d] (replicated); w13/w2: this rank's
    experts only ([N/G, rows, d], [N/G, d, ff]).
    """

    def __init__(self, shape: EPShape, router_wt, w13, w2, policy: PolicyConfig | None,
                 activation: int = nat.ACT_SWIGLU):
        torch = _torch()
        self.s = shape
        self.lib = nat.lib()
        s = shape
        T, Tl, N, k, d, G = s.tokens, s.tokens_per_rank, s.num_experts, s.top_k, s.d_model, s.world_size
        self.router_wt = router_wt
        self.pol = policy.to_native() if policy is not None else None
        self.pol_ref = ctypes_ref(self.pol) if self.pol is not None else None
        self.layer = nat.LynxLayer(num_experts=s.experts_per_rank, top_k=k, d_model=d, d_ff=s.d_ff,
                                   activation=activation, w13=w13.data_ptr(), w2=w2.data_ptr(), router_wt=0)
        self.layer_ref = ctypes_ref(self.layer)
        self._keep = (router_wt, w13, w2)
        dev = "cuda"
        self.logits = torch.empty((Tl, N), dtype=torch.float64, device=dev)
        self.ids = torch.empty((T, k), dtype=torch.int32, device=dev)
        self.probs = torch.empty((T, k), dtype=torch.float64, device=dev)
        self.full = torch.empty((T, N), dtype=torch.float64, device=dev)
        self.conf = torch.empty((T,), dtype=torch.float64, device=dev)
        self.assigned = torch.empty((T, k), dtype=torch.int32, device=dev)
        self.weights = torch.empty((T, k), dtype=torch.float64, device=dev)
        self.flags = torch.zeros((1,), dtype=torch.int32, device=dev)
        self.sel = nat.LynxSelection(expert_ids=self.ids.data_ptr(), probs=self.probs.data_ptr(),
                                     full_probs=self.full.data_ptr(), conf=self.conf.data_ptr(),
                                     assigned=self.assigned.data_ptr(), weights=self.weights.data_ptr(),
                                     flags=self.flags.data_ptr())
        self.sel_ref = ctypes_ref(self.sel)
        self.send = torch.empty((G * Tl, d), dtype=torch.bfloat16, device=dev)
        self.assigned_local = torch.empty((T, k), dtype=torch.int32, device=dev)
        self.weights_local = torch.empty((T, k), dtype=torch.float64, device=dev)
        self.partial = torch.empty((T, d), dtype=torch.float32, device=dev)
        self.out = torch.empty((Tl, d), dtype=torch.bfloat16, device=dev)
        nbytes = int(self.lib.lynx_moe_workspace_bytes(self.layer_ref, T))
        self.ws = torch.empty((nbytes,), dtype=torch.uint8, device=dev)

    @staticmethod
    def _stream():
        return _torch().cuda.current_stream().cuda_stream

    def router(self, hidden_local):
        s = self.s
        nat.check(self.lib.lynx_router_logits(hidden_local.data_ptr(), self.router_wt.data_ptr(),
                                              s.tokens_per_rank, s.d_model, s.num_experts,
                                              self.logits.data_ptr(), self._stream()), "ep router")
        return self.logits

    def select(self, logits_all):
        s = self.s
        nat.check(self.lib.lynx_route_select(logits_all.data_ptr(), s.tokens, s.num_experts, s.top_k, 1,
                                             self.pol_ref, self.sel_ref, self._stream()), "ep select")
        return self.assigned, self.weights

    def pack(self, hidden_local, assigned):
        s = self.s
        nat.check(self.lib.lynx_ep_pack(hidden_local.data_ptr(), assigned.data_ptr(), s.tokens_per_rank, s.top_k,
                                        s.num_experts, s.world_size, s.d_model, s.rank, self.send.data_ptr(),
                                        self._stream()), "ep pack")
        return self.send

    def local_mask(self, assigned, weights):
        s = self.s
        nat.check(self.lib.lynx_ep_local_mask(assigned.data_ptr(), weights.data_ptr(), s.tokens, s.top_k,
                                              s.num_experts, s.world_size, s.rank, self.assigned_local.data_ptr(),
                                              self.weights_local.data_ptr(), self._stream()), "ep local mask")
        return self.assigned_local, self.weights_local

    def forward_partial(self, recv, assigned_local, weights_local):
        s = self.s
        nat.check(self.lib.lynx_moe_forward_partial(self.layer_ref, recv.data_ptr(), s.tokens,
                                                    assigned_local.data_ptr(), weights_local.data_ptr(),
                                                    self.partial.data_ptr(), self.ws.data_ptr(), self.ws.numel(),
                                                    self._stream()), "ep forward")
        return self.partial

    def combine(self, hidden_local, back):
        s = self.s
        nat.check(self.lib.lynx_ep_combine(hidden_local.data_ptr(), back.data_ptr(), s.tokens_per_rank,
                                           s.world_size, s.d_model, self.out.data_ptr(), self._stream()),
                  "ep combine")
        return self.out


def shard_experts(tensor, rank: int, world_size: int):
    """Rows [rank*N/G, (rank+1)*N/G) of an expert-major weight tensor."""
    n = tensor.shape[0] // world_size
    return tensor[rank * n:(rank + 1) * n].contiguous()
