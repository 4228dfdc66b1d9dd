"""B200 calibration table for the reference cost model.

Runs the Mixtral-shaped 32-layer decode stack (attention stand-in + Lynx MoE
layer, 4 active experts = latency policy drop 4, the reference table's
calibration_active_experts) at batch 8/16/32/64 and writes per-step
attn/route/mlp milliseconds in the format of the reference's
sample_configs/calibration_a100.csv (costmodel.py:300-343), so
`moetrim costmodel` can be calibrated against B200 numbers unchanged.

    python scripts/calibrate_b200.py [out.csv]      (GPU)
"""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_08982_b200 as L  # noqa: E402


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else "profiles/calibration_b200.csv"
    nl, d, ff, N, k = 32, 4096, 14336, 8, 2
    spec = L.MoEModelSpec(nl, N, k, d, ff)
    model = L.build_swiglu_model(spec, seed=0)
    attn = L.build_attention(nl, d, 16, seed=1)
    pol = L.PolicyConfig(mode="latency", drop_count=4)
    P, reps = 16, 8
    rows = []
    for B in (8, 16, 32, 64):
        stack = L.DecodeStack(model, attn, B, max_len=P + 4 * reps + 8, policy=pol)
        x = torch.randn((B, P, d), generator=torch.Generator().manual_seed(B)).to(torch.bfloat16)
        stack.prefill(x)
        for _ in range(2):
            stack.profile_step()
        samples = [stack.profile_step() for _ in range(reps)]
        used = statistics.mean(layer.used_experts() for layer in stack._decode_layers)
        # graphed step time for the same shape (what a deployment pays)
        for _ in range(3):
            stack.step()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            stack.step()
        e1.record()
        torch.cuda.synchronize()
        row = {key: statistics.median(s[key] for s in samples) for key in ("attn_ms", "route_ms", "mlp_ms")}
        row.update(batch_size=B, used=used, graph_ms=e0.elapsed_time(e1) / reps)
        rows.append(row)
        print(row, flush=True)
        del stack
        torch.cuda.empty_cache()
    os.makedirs(os.path.dirname(os.path.abspath(out)), exist_ok=True)
    with open(out, "w") as f:
        f.write("# Measured per-step decode cost breakdown on one B200 (sm_100a), Mixtral-8x7B shape\n")
        f.write("# (32 layers, 8 experts, top-2, d=4096, ff=14336, bf16), Lynx latency policy with 4 active\n")
        f.write("# experts, prefill 16 then decode; milliseconds per 32-layer step, each part summed over\n")
        f.write("# layers from CUDA events around its kernels (serialised; graphed step = "
                + ", ".join(f"{r['graph_ms']:.3f} ms @ {r['batch_size']}" for r in rows) + ").\n")
        f.write("# Made by scripts/calibrate_b200.py; same columns as the reference's calibration_a100.csv.\n")
        f.write("batch_size,attn_ms,route_ms,mlp_ms\n")
        for r in rows:
            f.write(f"{r['batch_size']},{r['attn_ms']:.3f},{r['route_ms']:.3f},{r['mlp_ms']:.3f}\n")
    print("wrote", out)


if __name__ == "__main__":
    main()
