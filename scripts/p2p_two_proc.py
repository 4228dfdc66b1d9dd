"""Two processes on ONE GPU driving the peer-memory EP layer over CUDA-IPC
shared buffers: checks the multi-process wiring of ep_p2p.ipc_peers end to
end against the single-device layer.
    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 scripts/p2p_two_proc.py"""
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_08982_b200 as L  # noqa: E402
from oracle import lynx_oracle as O  # noqa: E402
from paper_2411_08982_b200 import ep as EP  # noqa: E402
from paper_2411_08982_b200 import ep_p2p as P2P  # noqa: E402


def main():
    backend = os.environ.get("BACKEND", "gloo")
    dist.init_process_group(backend)
    rank, G = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(0)
    Tl, N, k, d, ff = 16, 8, 2, 256, 512
    spec = L.MoEModelSpec(1, N, k, d, ff)
    model = L.build_swiglu_model(spec, seed=3)
    cfg = L.PolicyConfig(mode="latency", drop_count=4)
    g = torch.Generator(device="cuda").manual_seed(7)
    hidden = torch.randn((G * Tl, d), generator=g, device="cuda").to(torch.bfloat16)
    ref_layer = L.LynxMoELayer(model, 0, G * Tl, policy=cfg)
    ref = ref_layer(hidden)
    peers = P2P.ipc_peers(dist.group.WORLD, Tl, N, d)
    layer = P2P.P2PEPLayer(peers, model.router_wt[0], EP.shard_experts(model.w13[0], rank, G),
                           EP.shard_experts(model.w2[0], rank, G), N, k, ff, cfg)
    h = hidden[rank * Tl:(rank + 1) * Tl].contiguous()
    for step in range(3):
        out = layer(h)
        torch.cuda.synchronize()
        assert torch.equal(layer.assigned, ref_layer.assigned), step
        err = O.norm_rel_err(out.float().cpu().numpy(), ref[rank * Tl:(rank + 1) * Tl].float().cpu().numpy())
        assert err <= 1e-2, err
    print(f"rank {rank}: ok (rel err {err:.2e})", flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
