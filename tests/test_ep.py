"""Expert-parallel orchestration (paper_2411_08982_b200/ep.py).

CPU: world_size 2 over gloo with oracle-backed compute ops -- checks that the
all-gather / all-to-all plumbing, packing, local masks and the combine
reproduce the single-device layer exactly.
GPU: the native ops at world_size 1 over NCCL match LynxMoELayer.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest

from conftest import has_gpu
from oracle import lynx_oracle as O


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


class OracleEPOps:
    """Test-only EPOps backed by the CPU oracle (float32, exact bookkeeping)."""

    def __init__(self, shape, router_w, w1, w3, w2, pol):
        self.s, self.router_w, self.w1, self.w3, self.w2, self.pol = shape, router_w, w1, w3, w2, pol

    def router(self, hidden_local):
        import torch
        z = O.router_logits(hidden_local.numpy().astype(np.float64), self.router_w)
        return torch.from_numpy(z)

    def select(self, logits_all):
        import torch
        ids, probs, full = O.route(logits_all.numpy(), self.s.top_k)
        m = O.apply(ids, probs, full, self.pol)
        return torch.from_numpy(m.assigned.astype(np.int32)), torch.from_numpy(m.weights)

    def pack(self, hidden_local, assigned):
        import torch
        s = self.s
        per = s.num_experts // s.world_size
        send = torch.zeros((s.world_size * s.tokens_per_rank, s.d_model), dtype=hidden_local.dtype)
        for p in range(s.world_size):
            for i in range(s.tokens_per_rank):
                t = s.rank * s.tokens_per_rank + i
                if any(int(e) // per == p for e in assigned[t]):
                    send[p * s.tokens_per_rank + i] = hidden_local[i]
        return send

    def local_mask(self, assigned, weights):
        s = self.s
        per = s.num_experts // s.world_size
        a = assigned.clone()
        own = (a // per) == s.rank
        a[own] -= s.rank * per
        a[~own] = -1
        return a, weights

    def forward_partial(self, recv, assigned_local, weights_local):
        import torch
        x = recv.numpy().astype(np.float64)
        a = assigned_local.numpy()
        w = weights_local.numpy()
        out = np.zeros_like(x)
        per = self.s.num_experts // self.s.world_size
        for e in range(per):
            ge = self.s.rank * per + e
            for t in range(x.shape[0]):
                wt = sum(float(w[t, c]) for c in range(a.shape[1]) if a[t, c] == e)
                if any(a[t, c] == e for c in range(a.shape[1])):
                    h = O.silu(x[t] @ self.w1[ge].T) * (x[t] @ self.w3[ge].T)
                    out[t] += wt * (h @ self.w2[ge].T)
        return torch.from_numpy(out)

    def combine(self, hidden_local, back):
        return hidden_local + back.sum(dim=0)


def _ep_worker(rank, world, port, result_path):
    import torch
    import torch.distributed as dist

    from paper_2411_08982_b200 import ep as EP
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(0)
    N, k, d, ff, Tl = 4, 2, 16, 24, 5
    router_w = rng.normal(0, 2 / np.sqrt(d), size=(d, N))
    w1 = rng.normal(0, 1 / np.sqrt(d), size=(N, ff, d))
    w3 = rng.normal(0, 1 / np.sqrt(d), size=(N, ff, d))
    w2 = rng.normal(0, 1 / np.sqrt(ff), size=(N, d, ff))
    hidden_all = rng.normal(size=(world * Tl, d))
    pol = O.Policy(mode="latency", drop_count=2)
    shape = EP.EPShape(num_experts=N, top_k=k, d_model=d, d_ff=ff, tokens_per_rank=Tl, world_size=world, rank=rank)
    ops = OracleEPOps(shape, router_w, w1, w3, w2, pol)
    h_local = torch.from_numpy(hidden_all[rank * Tl:(rank + 1) * Tl].copy())
    out = EP.ep_layer(shape, ops, h_local)
    outs = [torch.empty_like(out) for _ in range(world)]
    dist.all_gather(outs, out)
    if rank == 0:
        got = torch.cat(outs).numpy()
        ids, probs, full = O.route(O.router_logits(hidden_all, router_w), k)
        m = O.apply(ids, probs, full, pol)
        want = O.forward_swiglu(hidden_all, w1, w3, w2, m.assigned, m.weights, dtype=np.float64)
        np.save(result_path, np.stack([got, want]))
    dist.destroy_process_group()


def test_ep_orchestration_gloo_world2(tmp_path):
    import torch.multiprocessing as mp
    path = str(tmp_path / "ep.npy")
    mp.spawn(_ep_worker, args=(2, _free_port(), path), nprocs=2, join=True)
    got, want = np.load(path)
    # grouping differs only by float64 association (per-rank partial sums)
    assert np.max(np.abs(got - want)) < 1e-10


@pytest.mark.gpu
def test_ep_native_world1_matches_layer():
    import torch
    import torch.distributed as dist

    import paper_2411_08982_b200 as L
    from paper_2411_08982_b200 import ep as EP
    if not has_gpu():
        pytest.skip("no GPU")
    if not dist.is_initialized():
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(_free_port())
        dist.init_process_group("nccl", rank=0, world_size=1)
    spec = L.MoEModelSpec(1, 8, 2, 256, 512)
    model = L.build_swiglu_model(spec, seed=3)
    T = 32
    hidden = torch.randn((T, 256), device="cuda").to(torch.bfloat16)
    cfg = L.PolicyConfig(mode="latency", drop_count=4)
    shape = EP.EPShape(8, 2, 256, 512, T, 1, 0)
    ops = EP.NativeEPOps(shape, model.router_wt[0], model.w13[0], model.w2[0], cfg)
    out = EP.ep_layer(shape, ops, hidden)
    layer = L.LynxMoELayer(model, 0, T, policy=cfg)
    ref = layer(hidden)
    torch.cuda.synchronize()
    assert torch.equal(ops.assigned, layer.assigned)
    # fp32 partial + residual in the EP combine vs fused bf16 combine: within bf16 rounding
    err = (out.float() - ref.float()).abs().max().item() / ref.float().abs().max().item()
    assert err < 1e-2
    dist.destroy_process_group()


@pytest.mark.gpu
def test_forward_partial_empty_shard_is_zero():
    import torch

    import paper_2411_08982_b200 as L
    if not has_gpu():
        pytest.skip("no GPU")
    spec = L.MoEModelSpec(1, 2, 2, 128, 256)
    model = L.build_swiglu_model(spec, seed=0)
    T = 8
    hidden = torch.randn((T, 128), device="cuda").to(torch.bfloat16)
    assigned = torch.full((T, 2), -1, dtype=torch.int32, device="cuda")
    weights = torch.zeros((T, 2), dtype=torch.float64, device="cuda")
    out = L.forward_partial(hidden, model, 0, assigned, weights)
    assert torch.count_nonzero(out).item() == 0


@pytest.mark.gpu
@pytest.mark.parametrize("G,N,policy", [(2, 8, ("latency", 4)), (4, 8, ("accuracy", 3)), (8, 8, ("latency", 4)),
                                        (4, 16, ("latency", 6))])
def test_p2p_ep_simulated_ranks_match_single_device(G, N, policy):
    """Peer-memory EP (lynx_ep_p2p_*) with G ranks simulated on one GPU:
    every rank's selection is bit-identical to the single-device layer on the
    global batch, and its output rows match that layer's rows (bf16 tol; the
    cross-rank sum reorders the fp32 additions)."""
    import torch

    import paper_2411_08982_b200 as L
    from paper_2411_08982_b200 import ep as EP
    from paper_2411_08982_b200 import ep_p2p as P2P
    Tl, k, d, ff = 16, 2, 256, 512
    spec = L.MoEModelSpec(1, N, k, d, ff)
    model = L.build_swiglu_model(spec, seed=G + N)
    mode, x = policy
    cfg = L.PolicyConfig(mode=mode, drop_count=x if mode == "latency" else 0,
                         freq_keep_budget=x if mode == "accuracy" else 4)
    hidden = torch.randn((G * Tl, d), device="cuda").to(torch.bfloat16)
    ref_layer = L.LynxMoELayer(model, 0, G * Tl, policy=cfg)
    ref = ref_layer(hidden)
    peers = P2P.simulated_peers(G, Tl, N, d)
    layers = [P2P.P2PEPLayer(peers[r], model.router_wt[0], EP.shard_experts(model.w13[0], r, G),
                             EP.shard_experts(model.w2[0], r, G), N, k, ff, cfg) for r in range(G)]
    hs = [hidden[r * Tl:(r + 1) * Tl].contiguous() for r in range(G)]
    for step in range(2):  # second step exercises the epoch advance
        outs = P2P.run_simulated(layers, hs)
        torch.cuda.synchronize()
        for r in range(G):
            assert torch.equal(layers[r].assigned, ref_layer.assigned), (step, r)
            assert O.norm_rel_err(outs[r].float().cpu().numpy(), ref[r * Tl:(r + 1) * Tl].float().cpu().numpy()) <= 1e-2
            delta = (outs[r].float() - hs[r].float()).cpu().numpy()
            ref_delta = (ref[r * Tl:(r + 1) * Tl].float() - hs[r].float()).cpu().numpy()
            assert O.norm_rel_err(delta, ref_delta) <= 3e-2, (step, r)


@pytest.mark.gpu
def test_p2p_ep_two_processes_one_gpu():
    """The multi-process wiring (CUDA-IPC buffer exchange, cross-process
    release/acquire flags, epochs): two torchrun ranks on one GPU run three
    layer steps of the peer-memory EP layer against the single-device layer."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.join(root, "scripts",
                                                                                          "p2p_two_proc.py")]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=240, cwd=root)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-2000:]
    assert "rank 0: ok" in out.stdout and "rank 1: ok" in out.stdout


@pytest.mark.gpu
@pytest.mark.parametrize("config,transport,batch", [("c2", "p2p", 32), ("c5", "p2p", 256), ("c5", "nccl", 256)])
def test_bench_multi_rank_path_runs(config, transport, batch):
    """bench.py --gpus 4 WITHOUT torchrun: it re-launches itself with four
    local ranks (here all on GPU 0: --share-gpu, gloo), runs the EP step at
    the config's fixed global batch (C5: decode batch 256 = 64 rows per rank)
    and prints one JSON line with the per-rank / critical-path / aggregate
    bytes and the EP output's error against the single-device layer.  Per-rank statistics differ between ranks, so every collective
    must use one dtype on all ranks."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, os.path.join(root, "bench.py"), "--gpus", "4", "--share-gpu", "--config", config,
           "--ep-transport", transport, "--steps", "4", "--warmup", "3"]
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=root, env=env)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 4 and d["scaling"] == "strong" and d["value"] > 0
    assert d["config"]["parallelism"] == "ep4"
    assert d["config"]["global_batch"] == batch and d["config"]["tokens_per_gpu"] == batch // 4
    run = d["run"]
    assert len(run["used_experts_per_rank"]) == 4
    assert run["critical_path_bytes"] == max(run["expert_bytes_per_rank"])
    assert abs(run["aggregate_bytes"] - sum(run["expert_bytes_per_rank"])) < 1
    assert ("nccl" in run["transport"].lower()) == (transport == "nccl")
    # the EP output against the single-device layer on the same global batch (bench checks it too)
    assert run["parity_max_rel_err_vs_single_device"] <= 1e-2
    if transport == "nccl":
        assert 0 <= run["comm_share"] <= 1
