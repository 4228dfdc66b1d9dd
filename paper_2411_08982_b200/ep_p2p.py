"""Expert parallelism over NVLink peer memory -- the fused
alternative to ``ep.ep_layer``'s NCCL collectives.

The kernels that produce the data store it straight into the peers'
symmetric buffers and release a flag per peer; the consuming kernels
acquire-wait on the flags (include/lynx_b200.h, ``lynx_ep_p2p_*``):

  route     K0 on the local rows -> logits rows written into every rank
  dispatch  wait logits; K1 on the GLOBAL batch (identical on every rank,
            so the Lynx vote is global); this rank's rows into their expert
            owners' recv buffers
  expert    wait rows; this rank's experts (K2..K3); K4 stores every
            token's partial sum into its owner's back buffer
  combine   wait partials; residual + sum over ranks (rank order)

Buffers are shared across processes over CUDA IPC (``ipc_peers``: one GPU
per rank over NVLink, or several processes on one GPU), or through
``torch.distributed._symmetric_memory`` (``symmetric_peers``, distinct GPUs
only).  For single-process tests, G simulated ranks share ordinary device
allocations (``simulated_peers``) and are driven phase by phase.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

from . import _native as nat
from .errors import ValidationError
from .policy import PolicyConfig
from .router import ctypes_ref


def _torch():
    import torch
    return torch


@dataclass
class PeerSet:
    """One rank's view: the C struct plus the tensors it points into."""

    struct: nat.LynxEPPeers
    keep: tuple  # tensors that must outlive the struct

    @property
    def ref(self):
        return ctypes_ref(self.struct)


def _ptr_array(ptrs):
    torch = _torch()
    return torch.tensor([int(p) for p in ptrs], dtype=torch.int64, device="cuda")


def _make(G, rank, Tl, bufs, arrays, counters, epoch):
    torch = _torch()
    s = nat.LynxEPPeers()
    s.world_size, s.rank, s.tokens_per_rank = G, rank, Tl
    s.logits, s.recv, s.back, s.flags = (arrays[n].data_ptr() for n in ("logits", "recv", "back", "flags"))
    s.logits_local, s.recv_local, s.back_local, s.flags_local = (
        bufs[n].data_ptr() for n in ("logits", "recv", "back", "flags"))
    s.counters, s.epoch = counters.data_ptr(), epoch.data_ptr()
    del torch
    return PeerSet(s, (bufs, arrays, counters, epoch))


def _buffers(alloc, G, Tl, N, d):
    torch = _torch()
    return {"logits": alloc((G * Tl, N), torch.float64), "recv": alloc((G * Tl, d), torch.bfloat16),
            "back": alloc((G * Tl, d), torch.float32), "flags": alloc((3 * G,), torch.int32)}


def simulated_peers(G: int, Tl: int, N: int, d: int) -> list:
    """G ranks' buffers on the current GPU, wired to each other like peers."""
    torch = _torch()
    zeros = lambda shape, dt: torch.zeros(shape, dtype=dt, device="cuda")  # noqa: E731
    bufs = [_buffers(zeros, G, Tl, N, d) for _ in range(G)]
    arrays = {n: _ptr_array([b[n].data_ptr() for b in bufs]) for n in ("logits", "recv", "back", "flags")}
    return [_make(G, r, Tl, bufs[r], arrays, zeros((4,), torch.int32), zeros((1,), torch.int32)) for r in range(G)]


def symmetric_peers(group, Tl: int, N: int, d: int) -> PeerSet:
    """This process's rank over torch symmetric memory (one GPU per rank)."""
    torch = _torch()
    import torch.distributed as dist
    import torch.distributed._symmetric_memory as symm
    G, rank = dist.get_world_size(group), dist.get_rank(group)

    def alloc(shape, dt):
        t = symm.empty(shape, dtype=dt, device="cuda")
        t.zero_()
        return t

    bufs = _buffers(alloc, G, Tl, N, d)
    arrays = {}
    for n, t in bufs.items():
        h = symm.rendezvous(t, group)
        arrays[n] = _ptr_array(h.buffer_ptrs)
    dist.barrier(group)
    zeros = lambda shape, dt: torch.zeros(shape, dtype=dt, device="cuda")  # noqa: E731
    return _make(G, rank, Tl, bufs, arrays, zeros((4,), torch.int32), zeros((1,), torch.int32))


def _device_uuid(dev: int) -> str:
    return str(_torch().cuda.get_device_properties(dev).uuid)


def _local_ordinal(uuid: str) -> int:
    """This process's ordinal of the GPU with `uuid`; -1 if it is not visible
    (e.g. per-rank CUDA_VISIBLE_DEVICES isolation)."""
    torch = _torch()
    for i in range(torch.cuda.device_count()):
        if _device_uuid(i) == uuid:
            return i
    return -1


def ipc_peers(group, Tl: int, N: int, d: int) -> PeerSet:
    """This process's rank with buffers shared over CUDA IPC (cudaIpc*MemHandle
    through torch's storage sharing): works across GPUs of one node (the
    opened peer allocations are reached over NVLink) and for several
    processes on one GPU, which is how it is tested here.

    Collective and all-or-nothing: every rank of `group` calls it, and it
    either succeeds on every rank or raises ValidationError on every rank,
    so callers can fall back (to NCCL) together without a hang.  Peer GPUs
    are identified by UUID, not by the owner's device ordinal (ordinals are
    per process: under CUDA_VISIBLE_DEVICES isolation every rank is device 0).
    """
    torch = _torch()
    import torch.distributed as dist
    G, rank = dist.get_world_size(group), dist.get_rank(group)
    zeros = lambda shape, dt: torch.zeros(shape, dtype=dt, device="cuda")  # noqa: E731
    mine, bufs = {}, None
    try:
        bufs = _buffers(zeros, G, Tl, N, d)
        torch.cuda.synchronize()
        mine = {"uuid": _device_uuid(torch.cuda.current_device()),
                "h": {n: t.untyped_storage()._share_cuda_() for n, t in bufs.items()}}
    except Exception as e:  # still join the exchange below, so no rank is left waiting
        mine = {"error": f"rank {rank}: {type(e).__name__}: {e}"}
    allh = [None] * G
    dist.all_gather_object(allh, mine, group=group)
    errors = [a["error"] for a in allh if "error" in a]
    opened, arrays, err = [], {}, None
    if not errors:
        try:
            here = torch.cuda.current_device()
            local = []
            for r in range(G):
                dev = _local_ordinal(allh[r]["uuid"])
                if dev < 0:
                    raise ValidationError(f"rank {r}'s GPU {allh[r]['uuid']} is not visible to rank {rank} "
                                          "(per-rank device isolation?): peer memory needs every GPU visible")
                local.append(dev)
            # Opened IPC allocations are mapped for their owner's device; our
            # kernels run on this rank's device and store into them over NVLink.
            for dev in sorted(set(local) - {here}):
                nat.check(nat.lib().lynx_enable_peer_access(int(dev)), "lynx_enable_peer_access")
            for n, t in bufs.items():
                ptrs = []
                for r in range(G):
                    if r == rank:
                        ptrs.append(t.data_ptr())
                        continue
                    h = allh[r]["h"][n]
                    st = torch.UntypedStorage._new_shared_cuda(local[r], *h[1:])
                    opened.append(st)
                    ptrs.append(st.data_ptr())
                arrays[n] = _ptr_array(ptrs)
            torch.cuda.synchronize()
        except Exception as e:
            err = f"rank {rank}: {type(e).__name__}: {e}"
    status = [None] * G
    dist.all_gather_object(status, err, group=group)
    errors += [e for e in status if e]
    if errors:
        raise ValidationError("CUDA-IPC peer buffers unavailable: " + "; ".join(errors))
    dist.barrier(group)
    ps = _make(G, rank, Tl, bufs, arrays, zeros((4,), torch.int32), zeros((1,), torch.int32))
    ps.keep = ps.keep + (opened,)
    return ps


class P2PEPLayer:
    """One rank's expert-parallel Lynx MoE decode layer over peer memory.

    router_wt: full router [N, d]; w13/w2: this rank's N/G experts.  All
    buffers are preallocated; every call is stream-ordered with no host
    sync, so a full layer (``__call__``) can be captured into a CUDA graph.
    """

    def __init__(self, peers: PeerSet, router_wt, w13, w2, num_experts: int, top_k: int, d_ff: int,
                 policy: PolicyConfig | None, activation: int = nat.ACT_SWIGLU):
        torch = _torch()
        P = peers.struct
        G, Tl = P.world_size, P.tokens_per_rank
        if num_experts % G:
            raise ValidationError(f"{num_experts} experts do not shard over {G} ranks")
        self.peers, self.N, self.k = peers, num_experts, top_k
        self.d = int(router_wt.shape[1])
        self.router_wt = router_wt.contiguous()
        self.layer = nat.LynxLayer(num_experts=num_experts // G, top_k=top_k, d_model=self.d, d_ff=d_ff,
                                   activation=activation, w13=w13.data_ptr(), w2=w2.data_ptr(), router_wt=0)
        self.layer_ref = ctypes_ref(self.layer)
        self._keep = (w13, w2)
        self.pol = policy.to_native() if policy is not None else None
        self.pol_ref = ctypes_ref(self.pol) if self.pol is not None else None
        T, N, k, dev = G * Tl, num_experts, top_k, "cuda"
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
        self.assigned_local = torch.empty((T, k), dtype=torch.int32, device=dev)
        self.weights_local = torch.empty((T, k), dtype=torch.float64, device=dev)
        self.out = torch.empty((Tl, self.d), dtype=torch.bfloat16, device=dev)
        nbytes = int(nat.lib().lynx_moe_workspace_bytes(self.layer_ref, T))
        self.ws = torch.empty((nbytes,), dtype=torch.uint8, device=dev)
        self.lib = nat.lib()

    @staticmethod
    def _stream():
        return _torch().cuda.current_stream().cuda_stream

    def route(self, hidden_local):
        nat.check(self.lib.lynx_ep_p2p_route(self.router_wt.data_ptr(), hidden_local.data_ptr(), self.d, self.N,
                                             self.peers.ref, self._stream()), "ep_p2p_route")

    def dispatch(self, hidden_local, decode: bool = True):
        nat.check(self.lib.lynx_ep_p2p_dispatch(hidden_local.data_ptr(), self.N, self.k, self.d, 1 if decode else 0,
                                                self.pol_ref, self.sel_ref, self.peers.ref, self._stream()),
                  "ep_p2p_dispatch")

    def expert(self):
        nat.check(self.lib.lynx_ep_p2p_expert(self.layer_ref, self.N, self.assigned.data_ptr(),
                                              self.weights.data_ptr(), self.assigned_local.data_ptr(),
                                              self.weights_local.data_ptr(), self.peers.ref, self.ws.data_ptr(),
                                              self.ws.numel(), self._stream()), "ep_p2p_expert")

    def combine(self, hidden_local, out=None):
        out = self.out if out is None else out
        nat.check(self.lib.lynx_ep_p2p_combine(hidden_local.data_ptr(), self.d, out.data_ptr(), self.peers.ref,
                                               self._stream()), "ep_p2p_combine")
        return out

    def __call__(self, hidden_local, out=None):
        self.route(hidden_local)
        self.dispatch(hidden_local)
        self.expert()
        return self.combine(hidden_local, out)


def run_simulated(layers: list, hiddens: list) -> list:
    """Drive G simulated ranks (one GPU) phase by phase; returns each rank's output."""
    for phase in ("route", "dispatch", "expert"):
        for lay, h in zip(layers, hiddens):
            if phase == "expert":
                lay.expert()
            else:
                getattr(lay, phase)(h)
    return [lay.combine(h) for lay, h in zip(layers, hiddens)]


__all__ = ["P2PEPLayer", "PeerSet", "simulated_peers", "symmetric_peers", "ipc_peers", "run_simulated"]
del ctypes
