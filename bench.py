#!/usr/bin/env python
"""Lynx MoE decode layer benchmark (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl lynx|reference] [--config c2]

One step = one full MoE decode layer call on one batch: router GEMV+RMSNorm
(K0) -> route + Lynx policy + remap (K1) -> permutation/gather (K2) ->
grouped SwiGLU expert GEMM over the used experts on tcgen05 (K3) -> weighted
combine + residual (K4).  Default workload (configs[1]): Mixtral-8x7B layer
shape, d=4096, ff=14336, 8 experts, top-2, bf16, decode batch 32, Lynx
latency policy dropping 4 experts.

N > 1: expert parallel, rank g owns N_experts/N experts.  The config's batch
is the GLOBAL batch (fixed as N grows, scaling "strong"; T/N rows per rank);
--scaling weak keeps T rows per rank instead.  The exchanges run over NVLink
peer memory inside the producing kernels (--ep-transport p2p, the product
path) or as NCCL all-gather + all-to-all (--ep-transport nccl, the baseline).
Without torchrun, --gpus N re-launches itself through torch.distributed.run
with N local ranks (127.0.0.1).

--impl reference: the reference's CPU algorithm (the oracle port of moetrim's
route_batch + apply_policy + forward_layer with a SwiGLU expert, numpy/BLAS
on all host cores) on the same workload; rank 0 only.  Both arms also time
the reference as shipped -- the same calls with its own float64
tanh(x w1) w2 expert (simulator.py:77-113) -- as cpu_baseline_f64_tanh2.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "MoE decode layer µs/step & tokens/s (Mixtral shape, bs32); % of HBM roofline"

CONFIGS = {
    # configs[1] of BASELINE.json -- the headline
    "c2": dict(workload="mixtral-8x7b-moe-layer-decode-bs32-lynx-latency-drop4", d=4096, ff=14336, N=8, k=2,
               T=32, mode="latency", drop=4, rotate=4),
    "c2-nolynx": dict(workload="mixtral-8x7b-moe-layer-decode-bs32-no-lynx", d=4096, ff=14336, N=8, k=2, T=32,
                      mode="latency", drop=0, rotate=4),
    "c2-acc": dict(workload="mixtral-8x7b-moe-layer-decode-bs32-lynx-accuracy", d=4096, ff=14336, N=8, k=2,
                   T=32, mode="accuracy", drop=0, rotate=4),
    # configs[2]: Mixtral-8x7B full 32-layer decode step (attention stand-in + MoE layer per layer, one CUDA
    # graph per step), batch 64, kept-expert budget swept 8 -> 4 (latency policy drop 0..4); headline = budget 4
    "c3": dict(workload="mixtral-8x7b-32-layer-decode-step-bs64-lynx-latency-budget-sweep", d=4096, ff=14336, N=8,
               k=2, T=64, layers=32, mode="latency", drop=4, sweep=(0, 1, 2, 3, 4), prefill=16, d_head=16),
    # configs[3]: DeepSeek-MoE-16B shape, 64 routed + 2 shared experts, top-6, dynamic (accuracy) selection
    "c4": dict(workload="deepseek-moe-16b-layer-decode-bs128-lynx-accuracy-budget16", d=2048, ff=1408, N=64, S=2,
               k=6, T=128, mode="accuracy", drop=0, budget=16, rotate=6),
    # configs[4]: Mixtral-8x22B shape, decode batch 256 (the global batch: T/G rows per rank under EP)
    "c5": dict(workload="mixtral-8x22b-moe-layer-decode-bs256-lynx-latency-drop4", d=6144, ff=16384, N=8, k=2,
               T=256, mode="latency", drop=4, rotate=3),
    # the same layer at 32 tokens (C5's per-GPU batch at EP8)
    "c5-bs32": dict(workload="mixtral-8x22b-moe-layer-decode-bs32-lynx-latency-drop4", d=6144, ff=16384, N=8, k=2,
                    T=32, mode="latency", drop=4, rotate=3),
}

SWIGLU_BYTES = lambda c: 3 * c["d"] * c["ff"] * 2  # noqa: E731


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ----------------------------------------------------------------- clocks
class ClockSampler:
    """NVML sampling of SM clock + throttle reasons during the timed region."""

    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, device_index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception as e:  # pragma: no cover - reporting only
            log("clock sampler unavailable:", e)
            self.nv = None

    def _poll_once(self):
        nv = self.nv
        self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
        try:
            r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        except Exception:
            r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
        for bit, name in self.REASONS.items():
            if r & bit:
                self.reasons.add(name)

    def _run(self):
        while not self._stop.is_set():
            self._poll_once()
            time.sleep(0.002)

    def __enter__(self):
        if self.nv is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *exc):
        if self.nv is not None:
            self._stop.set()
            self._t.join()
            if not self.samples:
                self._poll_once()

    def summary(self):
        if self.nv is None:
            return None
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy read+write)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(cfg_name):
    """ncu DRAM bytes of ONE launch of this config's FFN kernel (profiles/ffn_traffic.json, written by
    scripts/summarize_round.py from the round's --set full captures); None when the config was not captured."""
    path = os.path.join(ROOT, "profiles", "ffn_traffic.json")
    if os.path.exists(path):
        with open(path) as f:
            return json.load(f).get(cfg_name)
    return None


# ------------------------------------------------------------- CPU oracle
def cpu_layer_setup(c, seed=0):
    """Host-side C2 layer for the oracle port: fp32 weights of the experts the
    sampled batches use (others are never read by the reference either)."""
    import numpy as np

    from oracle import lynx_oracle as O
    rng = np.random.default_rng(seed)
    T, d, ff, N, k = c["T"], c["d"], c["ff"], c["N"], c["k"]
    router_w = (rng.standard_normal((d, N), dtype=np.float32) * (2.0 / np.sqrt(d))).astype(np.float32)
    batches = [rng.standard_normal((T, d), dtype=np.float32) for _ in range(2)]
    pol = O.Policy(mode=c["mode"], drop_count=c["drop"], freq_keep_budget=c.get("budget", 4))
    used = set(range(N, N + c.get("S", 0)))
    for h in batches:
        ids, probs, full = O.route(O.router_logits(h, router_w).astype(np.float64), k)
        m = O.apply(ids, probs, full, pol)
        used.update(int(e) for e in np.unique(m.assigned))
    w1, w3, w2 = {}, {}, {}
    for e in sorted(used):
        w1[e] = rng.standard_normal((ff, d), dtype=np.float32) / np.float32(np.sqrt(d))
        w3[e] = rng.standard_normal((ff, d), dtype=np.float32) / np.float32(np.sqrt(d))
        w2[e] = rng.standard_normal((d, ff), dtype=np.float32) / np.float32(np.sqrt(ff))
    return dict(router_w=router_w, batches=batches, pol=pol, w1=w1, w3=w3, w2=w2, k=k,
                shared=range(N, N + c.get("S", 0)))


def cpu_layer_step(st, i):
    import numpy as np

    from oracle import lynx_oracle as O
    h = st["batches"][i % len(st["batches"])]
    ids, probs, full = O.route(O.router_logits(h, st["router_w"]).astype(np.float64), st["k"])
    m = O.apply(ids, probs, full, st["pol"])
    return O.forward_swiglu(h, st["w1"], st["w3"], st["w2"], m.assigned, m.weights, shared=st["shared"])


def cpu_tanh2_setup(c, seed=0):
    """The reference as shipped (simulator.py:77-113): float64 router, route_batch,
    apply_policy and forward_layer with its tanh(x @ w1) @ w2 expert; weights
    [d, ff] / [ff, d] float64 of the experts the sampled batches use."""
    import numpy as np

    from oracle import lynx_oracle as O
    rng = np.random.default_rng(seed)
    T, d, ff, N, k = c["T"], c["d"], c["ff"], c["N"], c["k"]
    router_w = rng.standard_normal((d, N)) * (2.0 / np.sqrt(d))
    batches = [rng.standard_normal((T, d)) for _ in range(2)]
    pol = O.Policy(mode=c["mode"], drop_count=c["drop"], freq_keep_budget=c.get("budget", 4))
    used = set()
    for h in batches:
        ids, probs, full = O.route(O.router_logits(h, router_w), k)
        used.update(int(e) for e in np.unique(O.apply(ids, probs, full, pol).assigned))
    w1, w2 = {}, {}
    for e in sorted(used):
        w1[e] = rng.standard_normal((d, ff), dtype=np.float32).astype(np.float64) / np.sqrt(d)
        w2[e] = rng.standard_normal((ff, d), dtype=np.float32).astype(np.float64) / np.sqrt(ff)
    return dict(router_w=router_w, batches=batches, pol=pol, w1=w1, w2=w2, k=k)


def cpu_tanh2_step(st, i):
    from oracle import lynx_oracle as O
    h = st["batches"][i % len(st["batches"])]
    ids, probs, full = O.route(O.router_logits(h, st["router_w"]), st["k"])
    m = O.apply(ids, probs, full, st["pol"])
    return O.forward_tanh2(h, st["w1"], st["w2"], m.assigned, m.weights)


def cpu_baseline_tanh2(c, steps=2):
    if c.get("S", 0):
        return {"skipped": "the reference has no shared experts (DeepSeek-MoE extension)"}
    st = cpu_tanh2_setup(c)
    cpu_tanh2_step(st, 0)
    t0 = time.perf_counter()
    for i in range(steps):
        cpu_tanh2_step(st, i)
    nl = c.get("layers", 1)
    dt = (time.perf_counter() - t0) / steps
    return {"value": c["T"] / (dt * nl), "unit": "tokens/s", "cores": cpu_threads(), "kind": "port",
            "ms_per_step": dt * 1e3 * nl,
            "sample": f"{steps} layer steps (T={c['T']}) of the reference as shipped: float64 router, route_batch, "
                      f"apply_policy, forward_layer with tanh(x w1) w2 experts (simulator.py:77-113) restated in "
                      f"oracle/lynx_oracle.py, numpy/OpenBLAS" + (f"; x {nl} layers" if nl > 1 else "")}


def config_dict(c, world=1, scaling="strong"):
    """The workload description, identical in both arms (no run-specific data)."""
    T = c["T"]
    per_gpu = T // world if scaling == "strong" else T
    out = {"workload": c["workload"], "d_model": c["d"], "d_ff": c["ff"], "experts": c["N"], "top_k": c["k"],
           "shared_experts": c.get("S", 0), "global_batch": per_gpu * world, "tokens_per_gpu": per_gpu,
           "policy": policy_name(c), "parallelism": "single" if world == 1 else f"ep{world}",
           "scaling": scaling}
    if "layers" in c:
        out.update(layers=c["layers"], prefill_len=c["prefill"], d_head=c["d_head"])
    return out


def policy_name(c):
    if c["mode"] == "accuracy":
        return f"accuracy tau 0.5 sample 8 budget {c.get('budget', 4)}"
    return f"latency drop {c['drop']}"


def cpu_threads():
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()


def cpu_baseline(c, steps=3):
    st = cpu_layer_setup(c)
    cpu_layer_step(st, 0)
    t0 = time.perf_counter()
    for i in range(steps):
        cpu_layer_step(st, i)
    dt = (time.perf_counter() - t0) / steps
    nl = c.get("layers", 1)
    sample = (f"{steps} full layer steps (T={c['T']}, router+route+{c['mode']} policy+SwiGLU fp32 over "
              f"the used experts) of the oracle port oracle/lynx_oracle.py, numpy/OpenBLAS")
    if nl > 1:
        sample += f"; the {nl}-layer step is timed as {nl} x one layer (attention stand-in not included)"
    return {"value": c["T"] / (dt * nl), "unit": "tokens/s", "cores": cpu_threads(), "kind": "port",
            "sample": sample, "ms_per_step": dt * 1e3 * nl}


# -------------------------------------------------------------- reference arm
def run_reference(args, c):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    st = cpu_layer_setup(c)
    for i in range(args.warmup):
        cpu_layer_step(st, i)
    t0 = time.perf_counter()
    for i in range(args.steps):
        cpu_layer_step(st, i)
    dt = (time.perf_counter() - t0) / args.steps * c.get("layers", 1)  # C3: layers x one layer step
    value = c["T"] / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": config_dict(c, args.gpus, args.scaling),
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": cpu_threads(), "kind": "port",
                         "sample": f"each step = one full layer step (global batch T={c['T']}) of the oracle port "
                                   "(moetrim's route_batch/apply_policy/forward_layer restated, SwiGLU fp32), "
                                   "numpy/OpenBLAS on every host core"},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if not args.no_cpu_baseline:
        line["cpu_baseline_f64_tanh2"] = cpu_baseline_tanh2(c)
    print(json.dumps(line), flush=True)
    return 0


# -------------------------------------------------------------- GPU arm
def run_single(args, c):
    import torch

    import paper_2411_08982_b200 as L
    T, d, ff, N, k, n = c["T"], c["d"], c["ff"], c["N"], c["k"], c["rotate"]
    spec = L.MoEModelSpec(num_layers=n, num_experts=N, top_k=k, d_model=d, d_ff=ff,
                          num_shared_experts=c.get("S", 0))
    model = L.build_swiglu_model(spec, seed=0)
    pol = L.PolicyConfig(mode=c["mode"], drop_count=c["drop"], freq_keep_budget=c.get("budget", 4))
    layers = [L.LynxMoELayer(model, l, T, policy=pol) for l in range(n)]
    g = torch.Generator(device="cuda").manual_seed(1)
    hid = [torch.randn((T, d), generator=g, device="cuda").to(torch.bfloat16) for _ in range(n)]
    outs = [torch.empty_like(h) for h in hid]

    for i in range(max(args.warmup, n)):
        layers[i % n](hid[i % n], outs[i % n])
    torch.cuda.synchronize()
    used = [layers[l].used_experts() for l in range(n)]
    ffn_kernel = layers[0].ffn_kernel()

    # CUDA graphs: all rotating layer copies captured back to back in ONE
    # graph (a deployment runs its layers inside one graph, so no graph
    # launch gap per layer; programmatic dependent launch spans the layer
    # boundaries), plus one single-layer graph per copy for remainders.
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        for l in range(n):
            layers[l](hid[l], outs[l])
    torch.cuda.current_stream().wait_stream(side)
    g_all = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g_all):
        for l in range(n):
            layers[l](hid[l], outs[l])
    graphs = []
    for l in range(n):
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr):
            layers[l](hid[l], outs[l])
        graphs.append(gr)
    g_all.replay()
    for gr in graphs:
        gr.replay()
    torch.cuda.synchronize()

    # (A) timed region: exactly K layer steps (K // n replays of the n-layer
    # graph + K % n single-layer replays), device-timed
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(torch.cuda.current_device()) as clocks:
        torch.cuda.synchronize()
        e0.record()
        for _ in range(args.steps // n):
            g_all.replay()
        for i in range(args.steps % n):
            graphs[i].replay()
        e1.record()
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps

    # (B) per-kernel device time on the launching stream (events between K0..K4)
    kp = min(args.steps, 100)
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(6)] for _ in range(kp)]
    for i in range(kp):
        layers[i % n].profiled(hid[i % n], evs[i], outs[i % n])
    torch.cuda.synchronize()
    names = ["router", "select_plan", "gather", "ffn", "combine"]
    kern = {nm: statistics.mean(evs[i][j].elapsed_time(evs[i][j + 1]) for i in range(kp))
            for j, nm in enumerate(names)}
    step_b = statistics.mean(evs[i][0].elapsed_time(evs[i][5]) for i in range(kp))

    # (C) end to end through the public API with pinned host buffers: every
    # step copies its own input host->device and its output device->host.
    # LynxMoELayer.stream_host overlaps those PCIe copies with the
    # neighbouring steps' expert streams (copy stream + double-buffered
    # device slots, one graph replay per step).
    h_host = [h.cpu().pin_memory() for h in hid]
    xs_host = [h_host[i % n] for i in range(args.steps)]
    os_host = [torch.empty_like(h_host[0]).pin_memory() for _ in range(args.steps)]
    layer0 = layers[0]
    layer0.stream_host(xs_host[:4], os_host[:4])  # capture + warm
    torch.cuda.synchronize()
    c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    c0.record()
    layer0.stream_host(xs_host, os_host)
    c1.record()
    torch.cuda.synchronize()
    ms_e2e = c0.elapsed_time(c1) / args.steps
    ref0 = layers[0](hid[0].clone()).cpu()
    assert torch.equal(os_host[0], ref0), "stream_host output differs from the device-resident call"
    # single-step host API (H2D + layer + D2H as one graph, no overlap) for reference
    o1 = torch.empty_like(h_host[0]).pin_memory()
    layer0.host_step(h_host[0], o1)
    torch.cuda.synchronize()
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record()
    for _ in range(20):
        layer0.host_step(h_host[0], o1)
    s1.record()
    torch.cuda.synchronize()
    ms_host_step = s0.elapsed_time(s1) / 20

    # (D) this GPU's achievable READ bandwidth, measured live (a read-only
    # reduction over 4 GiB, best of 5): the expert stream only reads, and a
    # read can beat MEASURED_PEAKS.json's copy figure (read + write)
    xbuf = torch.empty(4 << 30, dtype=torch.uint8, device="cuda").view(torch.int64)
    xbuf.fill_(1)
    best_rd = 1e9
    for _ in range(5):
        r0, r1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        r0.record()
        torch.amax(xbuf)
        r1.record()
        torch.cuda.synchronize()
        best_rd = min(best_rd, r0.elapsed_time(r1))
    read_peak = (4 << 30) / (best_rd * 1e-3) / 1e9
    del xbuf
    torch.cuda.empty_cache()

    # algorithmic bytes of one layer step (used experts only) and of one FFN launch
    mean_used = statistics.mean(used[i % n] for i in range(kp))
    ffn_bytes = mean_used * SWIGLU_BYTES(c)
    step_bytes = ffn_bytes + N * d * 2 + 2 * T * d * 2
    peak, peak_src = measured_peaks()
    achieved = ffn_bytes / (kern["ffn"] * 1e-3) / 1e9
    traffic = ncu_traffic(args.config)
    result = {
        "metric": METRIC, "value": T / (ms * 1e-3), "unit": "tokens/s", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "us_per_step": ms * 1e3, "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic: random-init Mixtral-shaped bf16 weights, N(0,1) hidden",
        "config": config_dict(c),
        "run": {"weight_copies": n,
                "graph": f"{n} layer calls (one per rotating weight copy) per CUDA-graph replay",
                "l2": f"inputs > L2: {n} rotating layer copies "
                      f"({n * (N + c.get('S', 0)) * SWIGLU_BYTES(c) / 1e9:.1f} GB) >> 126 MB L2",
                "used_experts_per_copy": used, "mean_used_experts": mean_used, "ffn_kernel": ffn_kernel},
        "roofline": {"bound": "hbm", "kernel": f"{ffn_kernel} (K3, tcgen05 grouped SwiGLU)",
                     "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "peak_source": peak_src,
                     "frac_of_8TBs": achieved / 8000.0,
                     "read_peak_gbs": read_peak, "frac_of_read_peak": achieved / read_peak,
                     "read_peak_source": "measured live in this run: torch.amax over 4 GiB (read-only), best of 5",
                     "algorithmic_bytes_per_launch": ffn_bytes,
                     "traffic": traffic.get("dram_bytes_per_launch") if traffic else None,
                     "traffic_source": traffic.get("source") if traffic else None,
                     "ffn_share_of_step": kern["ffn"] / step_b,
                     "step_bytes": step_bytes, "step_achieved_gbs": step_bytes / (ms * 1e-3) / 1e9},
        "kernel_ms": kern, "profiled_step_ms": step_b,
        "e2e": {"value": T / (ms_e2e * 1e-3), "unit": "tokens/s", "ms_per_step": ms_e2e,
                "h2d_bytes_per_step": T * d * 2, "d2h_bytes_per_step": T * d * 2,
                "api": "paper_2411_08982_b200.LynxMoELayer.stream_host (per-step H2D + lynx_moe_layer graph + D2H, "
                       "copies overlapped with neighbouring steps)",
                "single_step_host_api_ms": ms_host_step},
        # kernels per layer step: the fused front (N <= 8, T <= 256, no shared experts) + K3 + K4,
        # else K0 + K1 + K2 + K3 + K4
        "gpu_launches": (3 if (N <= 8 and T <= 256 and not c.get("S", 0)
                               and os.environ.get("LYNX_FUSED_FRONT") != "0") else 5) * args.steps,
        "clocks": clocks.summary(),
    }
    return result


def run_stack(args, c):
    """C3: the full decode step (simulate's decode loop, simulator.py:351-355) over
    all layers, replayed as one CUDA graph per step, for each kept-expert budget."""
    import torch

    import paper_2411_08982_b200 as L
    B, d, ff, N, k, nl = c["T"], c["d"], c["ff"], c["N"], c["k"], c["layers"]
    spec = L.MoEModelSpec(num_layers=nl, num_experts=N, top_k=k, d_model=d, d_ff=ff)
    model = L.build_swiglu_model(spec, seed=0)
    attn = L.build_attention(nl, d, c["d_head"], seed=1)
    P = c["prefill"]
    x = torch.randn((B, P, d), generator=torch.Generator().manual_seed(2)).to(torch.bfloat16)
    sweep = {}
    clocks = None
    for drop in c["sweep"]:
        pol = L.PolicyConfig(mode="latency", drop_count=drop)
        stack = L.DecodeStack(model, attn, B, max_len=P + args.warmup + args.steps + 4, policy=pol)
        stack.prefill(x)
        for _ in range(args.warmup):
            stack.step()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with ClockSampler(torch.cuda.current_device()) as cs:
            e0.record()
            for _ in range(args.steps):
                stack.step()
            e1.record()
            torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.steps
        assert bool(torch.isfinite(stack.prev.float()).all()), "decode stack produced non-finite states"
        flags = [int(layer.flags.item()) for layer in stack._decode_layers]
        assert not any(f & 2 for f in flags), "non-finite router logits"
        used = [layer.used_experts() for layer in stack._decode_layers]
        sweep[N - drop] = {"ms_per_step": ms, "tokens_per_s": B / (ms * 1e-3), "us_per_layer": ms * 1e3 / nl,
                           "mean_used_experts": statistics.mean(used),
                           "step_bytes": sum(used) * SWIGLU_BYTES(c),
                           "achieved_gbs": sum(used) * SWIGLU_BYTES(c) / (ms * 1e-3) / 1e9}
        if drop == c["drop"]:
            clocks = cs.summary()
            head = stack
        else:
            del stack
        log(f"budget {N - drop}: {ms:.3f} ms/step, used {statistics.mean(used):.2f}")
    best = sweep[N - c["drop"]]
    # e2e: the caller's host-side view per step -- the step's input state
    # host->device (pinned), one graphed step, the step's output device->host
    h_host = torch.randn((B, d)).to(torch.bfloat16).pin_memory()
    o_host = torch.empty_like(h_host).pin_memory()
    torch.cuda.synchronize()
    c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n_e2e = min(args.steps, 20)
    head.prefill(x)
    c0.record()
    for _ in range(n_e2e):
        head.prev.copy_(h_host, non_blocking=True)
        o_host.copy_(head.step(), non_blocking=True)
    c1.record()
    torch.cuda.synchronize()
    ms_e2e = c0.elapsed_time(c1) / n_e2e
    peak, peak_src = measured_peaks()
    return {
        "metric": METRIC, "value": best["tokens_per_s"], "unit": "tokens/s", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": best["ms_per_step"], "us_per_step": best["ms_per_step"] * 1e3,
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic: random-init Mixtral-shaped bf16 weights (32 layers, 90 GB), N(0,1) prefill inputs",
        "config": config_dict(c),
        "run": {"l2": "inputs > L2: each step streams every layer's used experts (>= 45 GB) >> 126 MB L2",
                "kept_budget": N - c["drop"], "budget_sweep": sweep},
        "roofline": {"bound": "hbm", "kernel": "whole decode step (32 x [attention + fused router, K1..K4])",
                     "achieved": best["achieved_gbs"], "peak": peak, "unit": "GB/s",
                     "frac": best["achieved_gbs"] / peak, "peak_source": peak_src,
                     "frac_of_8TBs": best["achieved_gbs"] / 8000.0, "algorithmic_bytes_per_step": best["step_bytes"],
                     "traffic": None},
        "e2e": {"value": B / (ms_e2e * 1e-3), "unit": "tokens/s", "ms_per_step": ms_e2e,
                "h2d_bytes_per_step": B * d * 2, "d2h_bytes_per_step": B * d * 2,
                "api": "paper_2411_08982_b200.DecodeStack.step (one CUDA graph per step)"},
        # per layer: the decode attention (one clustered kernel for d <= 8192, else attn_qkv + attn_out),
        # the fused front, K3, K4; per step: the position advance
        "gpu_launches": (nl * ((1 if d <= 8192 and os.environ.get("LYNX_ATTN_CLUSTER") != "0" else 2) + 3) + 1)
                        * args.steps,
        "clocks": clocks,
    }


def _ep_stats(used_local, world, c, ms, phase_ms, phase_names):
    """Per-rank / critical-path / aggregate expert bytes and the phase split, reduced over ranks."""
    import torch
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    mine = torch.tensor([float(statistics.mean(used_local))], dtype=torch.float64, device=dev)
    per_rank = [torch.zeros_like(mine) for _ in range(world)]
    dist.all_gather(per_rank, mine)
    used = [float(t.item()) for t in per_rank]
    ph = torch.tensor(phase_ms, dtype=torch.float64, device=dev)
    dist.all_reduce(ph, op=dist.ReduceOp.MAX)
    eb = SWIGLU_BYTES(c)
    return {
        "used_experts_per_rank": used,
        "expert_bytes_per_rank": [u * eb for u in used],
        "critical_path_bytes": max(used) * eb,
        "aggregate_bytes": sum(used) * eb,
        "phase_ms_max_over_ranks": dict(zip(phase_names, [float(x) for x in ph.tolist()])),
    }


def _ep_parity(c, rank, world, Tl, pol, out_local):
    """The EP step against the single-device layer on the same global batch:
    layer copy 0 (seed 100) rebuilt whole on every rank, every rank's first
    input regenerated from its seed; this rank's rows of the reference vs its
    EP output, norm-wise max |y - y_ref| / max |y_ref|, max over ranks.  The
    EP sum runs in rank order, the single-device combine in expert order: the
    same experts, another association, so a tolerance (1e-2), not equality."""
    import torch

    import paper_2411_08982_b200 as L
    d, ff, N, k = c["d"], c["ff"], c["N"], c["k"]
    spec = L.MoEModelSpec(num_layers=1, num_experts=N, top_k=k, d_model=d, d_ff=ff)
    full = L.build_swiglu_model(spec, seed=100)
    xs = []
    for r in range(world):
        g = torch.Generator(device="cuda").manual_seed(1000 + r)
        xs.append(torch.randn((Tl, d), generator=g, device="cuda").to(torch.bfloat16))
    ref = L.LynxMoELayer(full, 0, Tl * world, policy=pol)(torch.cat(xs))[rank * Tl:(rank + 1) * Tl].float()
    torch.cuda.synchronize()
    err = float((out_local.float() - ref).abs().max() / ref.abs().max().clamp_min(1e-30))
    del full, ref, xs
    torch.cuda.empty_cache()
    err = _max_over_ranks(err)
    if not err <= 1e-2:
        raise RuntimeError(f"EP output differs from the single-device layer: max rel err {err:.3e}")
    return err


def _ep_result(args, c, world, Tl, ms, ms_e2e, stats, transport, kernel_note, launches, clocks):
    peak, peak_src = measured_peaks()
    crit = stats["critical_path_bytes"]
    Tg = Tl * world
    return {
        "metric": METRIC, "value": Tg / (ms * 1e-3), "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "us_per_step": ms * 1e3, "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic: random-init Mixtral-shaped bf16 weights, N(0,1) hidden",
        "config": config_dict(c, world, args.scaling),
        "run": dict(stats, transport=transport, weight_copies=c["rotate"]),
        "roofline": {"bound": "hbm", "kernel": kernel_note,
                     "achieved": crit / (ms * 1e-3) / 1e9, "peak": peak, "unit": "GB/s",
                     "frac": crit / (ms * 1e-3) / 1e9 / peak, "peak_source": peak_src,
                     "note": "critical-path expert bytes (max over ranks) / whole step time, exchanges included",
                     "aggregate_achieved_gbs": stats["aggregate_bytes"] / (ms * 1e-3) / 1e9,
                     "traffic": None},
        "e2e": {"value": Tg / (ms_e2e * 1e-3), "unit": "tokens/s", "ms_per_step": ms_e2e,
                "h2d_bytes_per_step": Tl * c["d"] * 2, "d2h_bytes_per_step": Tl * c["d"] * 2,
                "note": "per rank: its T/G input rows in, its output rows out"},
        "gpu_launches": launches * args.steps,
        "clocks": clocks.summary(),
    }


def run_ep_p2p(args, c, rank, world, local_rank, peers):
    """Expert parallel over NVLink peer memory (ep_p2p.P2PEPLayer): the logits
    all-gather, dispatch and return are stores issued by the producing
    kernels into the peers' CUDA-IPC-shared buffers; one CUDA graph per step."""
    import torch
    import torch.distributed as dist

    import paper_2411_08982_b200 as L
    from paper_2411_08982_b200 import ep as EP
    from paper_2411_08982_b200 import ep_p2p as P2P
    Tl = c["T"] // world if args.scaling == "strong" else c["T"]
    d, ff, N, k, n = c["d"], c["ff"], c["N"], c["k"], c["rotate"]
    spec = L.MoEModelSpec(num_layers=1, num_experts=N, top_k=k, d_model=d, d_ff=ff)
    pol = L.PolicyConfig(mode=c["mode"], drop_count=c["drop"], freq_keep_budget=c.get("budget", 4))
    layers = []
    for l in range(n):
        full = L.build_swiglu_model(spec, seed=100 + l)  # same seed on every rank -> identical model
        layers.append(P2P.P2PEPLayer(peers, full.router_wt[0].contiguous(), EP.shard_experts(full.w13[0], rank, world),
                                     EP.shard_experts(full.w2[0], rank, world), N, k, ff, pol))
        del full
        torch.cuda.empty_cache()
    g = torch.Generator(device="cuda").manual_seed(1000 + rank)
    hid = [torch.randn((Tl, d), generator=g, device="cuda").to(torch.bfloat16) for _ in range(n)]
    outs = [torch.empty_like(h) for h in hid]
    # every rank's layers are built before any rank waits on a peer's flags
    # (the peer waits have a watchdog)
    torch.cuda.synchronize()
    dist.barrier()
    for i in range(max(args.warmup, n)):
        layers[i % n](hid[i % n], outs[i % n])
    torch.cuda.synchronize()
    dist.barrier()
    used_local = []
    for l in range(n):
        a = layers[l].assigned_local
        used_local.append(int((torch.bincount(a[a >= 0].long(), minlength=N // world) > 0).sum()))
    # phase split (eager, events between the four calls; serialises the programmatic launches)
    names = ["route", "dispatch", "expert", "combine"]
    reps = min(20, args.steps)
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in range(reps)]
    dist.barrier()
    for i in range(reps):
        lay, h = layers[i % n], hid[i % n]
        evs[i][0].record()
        lay.route(h)
        evs[i][1].record()
        lay.dispatch(h)
        evs[i][2].record()
        lay.expert()
        evs[i][3].record()
        lay.combine(h, outs[i % n])
        evs[i][4].record()
    torch.cuda.synchronize()
    phase = [statistics.mean(evs[i][j].elapsed_time(evs[i][j + 1]) for i in range(reps)) for j in range(4)]
    g_all = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g_all):
        for l in range(n):
            layers[l](hid[l], outs[l])
    dist.barrier()
    g_all.replay()
    torch.cuda.synchronize()
    dist.barrier()
    reps = max(1, args.steps // n)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(torch.cuda.current_device()) as clocks:
        dist.barrier()
        torch.cuda.synchronize()
        e0.record()
        for _ in range(reps):
            g_all.replay()
        e1.record()
        torch.cuda.synchronize()
        dist.barrier()
    steps = reps * n
    ms = _max_over_ranks(e0.elapsed_time(e1) / steps)
    stats = _ep_stats(used_local, world, c, ms, phase, names)
    # e2e: pinned host input/output per step around the same layers
    h_host = [h.cpu().pin_memory() for h in hid]
    o_host = torch.empty((Tl, d), dtype=torch.bfloat16).pin_memory()
    dist.barrier()
    torch.cuda.synchronize()
    c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    c0.record()
    for i in range(steps):
        l = i % n
        hid[l].copy_(h_host[l], non_blocking=True)
        layers[l](hid[l], outs[l])
        o_host.copy_(outs[l], non_blocking=True)
    c1.record()
    torch.cuda.synchronize()
    ms_e2e = _max_over_ranks(c0.elapsed_time(c1) / steps)
    args.steps = steps
    layers[0](hid[0], outs[0])
    stats["parity_max_rel_err_vs_single_device"] = _ep_parity(c, rank, world, Tl, pol, outs[0])
    return _ep_result(args, c, world, Tl, ms, ms_e2e, stats,
                      "nvlink peer memory (lynx_ep_p2p_*, CUDA-IPC shared buffers; stores issued by K0 / the "
                      "dispatch kernel / K4, release-acquire flags)",
                      "ffn_kernel per rank (critical path)", 11, clocks)


def _max_over_ranks(v):
    import torch
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([float(v)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def run_ep(args, c, rank, world, local_rank):
    """Expert parallel with NCCL collectives (ep.ep_layer): all-gather of the
    logits, all-to-all dispatch and return around the same kernels."""
    import torch
    import torch.distributed as dist

    import paper_2411_08982_b200 as L
    from paper_2411_08982_b200 import ep as EP
    Tl = c["T"] // world if args.scaling == "strong" else c["T"]
    d, ff, N, k, n = c["d"], c["ff"], c["N"], c["k"], c["rotate"]
    shape = EP.EPShape(num_experts=N, top_k=k, d_model=d, d_ff=ff, tokens_per_rank=Tl, world_size=world, rank=rank)
    spec = L.MoEModelSpec(num_layers=1, num_experts=N, top_k=k, d_model=d, d_ff=ff)
    pol = L.PolicyConfig(mode=c["mode"], drop_count=c["drop"], freq_keep_budget=c.get("budget", 4))
    ops = []
    for l in range(n):
        full = L.build_swiglu_model(spec, seed=100 + l)  # same seed on every rank -> identical model
        w13 = EP.shard_experts(full.w13[0], rank, world)
        w2 = EP.shard_experts(full.w2[0], rank, world)
        ops.append(EP.NativeEPOps(shape, full.router_wt[0].contiguous(), w13, w2, pol))
        del full
        torch.cuda.empty_cache()
    g = torch.Generator(device="cuda").manual_seed(1000 + rank)
    hid = [torch.randn((Tl, d), generator=g, device="cuda").to(torch.bfloat16) for _ in range(n)]
    for i in range(max(args.warmup, n)):
        EP.ep_layer(shape, ops[i % n], hid[i % n])
    torch.cuda.synchronize()
    used_local = []
    for l in range(n):
        EP.ep_layer(shape, ops[l], hid[l])
        a = ops[l].assigned_local
        used_local.append(int((torch.bincount(a[a >= 0].long(), minlength=shape.experts_per_rank) > 0).sum()))
    # phase split: events around the three collectives (comm) and the compute between them
    names = ["router", "allgather_logits", "select_pack", "alltoall_dispatch", "expert", "alltoall_return",
             "combine"]
    reps = min(20, args.steps)
    marks = [[torch.cuda.Event(enable_timing=True) for _ in range(8)] for _ in range(reps)]
    dist.barrier()
    for i in range(reps):
        EP.ep_layer(shape, ops[i % n], hid[i % n], mark=lambda j, _i=i: marks[_i][j].record())
    torch.cuda.synchronize()
    phase = [statistics.mean(marks[i][j].elapsed_time(marks[i][j + 1]) for i in range(reps)) for j in range(7)]
    dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(torch.cuda.current_device()) as clocks:
        dist.barrier()
        torch.cuda.synchronize()
        e0.record()
        for i in range(args.steps):
            EP.ep_layer(shape, ops[i % n], hid[i % n])
        e1.record()
        torch.cuda.synchronize()
        dist.barrier()
    ms = _max_over_ranks(e0.elapsed_time(e1) / args.steps)
    stats = _ep_stats(used_local, world, c, ms, phase, names)
    pm = stats["phase_ms_max_over_ranks"]
    comm = pm["allgather_logits"] + pm["alltoall_dispatch"] + pm["alltoall_return"]
    stats["comm_share"] = comm / sum(pm.values())
    # e2e: host-resident inputs/outputs per step
    h_host = [h.cpu().pin_memory() for h in hid]
    o_host = torch.empty((Tl, d), dtype=torch.bfloat16).pin_memory()
    dist.barrier()
    torch.cuda.synchronize()
    c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    c0.record()
    for i in range(args.steps):
        l = i % n
        hid[l].copy_(h_host[l], non_blocking=True)
        out = EP.ep_layer(shape, ops[l], hid[l])
        o_host.copy_(out, non_blocking=True)
    c1.record()
    torch.cuda.synchronize()
    ms_e2e = _max_over_ranks(c0.elapsed_time(c1) / args.steps)
    stats["parity_max_rel_err_vs_single_device"] = _ep_parity(c, rank, world, Tl, pol,
                                                              EP.ep_layer(shape, ops[0], hid[0]))
    return _ep_result(args, c, world, Tl, ms, ms_e2e, stats, "NCCL all_gather + all_to_all_single (torch.distributed)",
                      "ffn_kernel per rank (critical path)", 6, clocks)


def self_launch(args) -> int:
    """--gpus N without torchrun: re-run this script under torch.distributed.run
    with N local ranks (rendezvous on 127.0.0.1)."""
    import socket
    import subprocess
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    log("launching", " ".join(cmd))
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["lynx", "reference"], default="lynx")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="c2")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--share-gpu", action="store_true",
                    help="N>1 on ONE GPU (gloo + CUDA IPC): functional check only, not a measurement")
    ap.add_argument("--ep-transport", choices=["p2p", "nccl"], default="p2p",
                    help="N>1: expert-parallel exchange over NVLink peer memory or NCCL collectives")
    ap.add_argument("--scaling", choices=["strong", "weak"], default="strong",
                    help="N>1: strong = the config's batch is the global batch (T/N rows per rank); "
                         "weak = T rows per rank")
    ap.add_argument("--tokens", type=int, default=None, help="override the config's batch (diagnostics)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    c = dict(CONFIGS[args.config])
    if args.tokens:
        c["T"] = args.tokens
        c["workload"] += f"-T{args.tokens}"
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.impl == "reference":
        return run_reference(args, c)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return self_launch(args)
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    if world > 1 and (c["N"] % world or (args.scaling == "strong" and c["T"] % world)):
        raise SystemExit(f"{c['N']} experts / batch {c['T']} do not shard over {world} GPUs")
    if world > 1 and "layers" in c:
        raise SystemExit("the 32-layer stack (c3) runs on one GPU")

    import torch
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.share_gpu:  # functional check of the N>1 path with every rank on GPU 0 (timings meaningless)
        local_rank = 0
    torch.cuda.set_device(local_rank)
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if args.share_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        peers = None
        if args.ep_transport == "p2p":
            from paper_2411_08982_b200 import ep_p2p as P2P
            Tl = c["T"] // world if args.scaling == "strong" else c["T"]
            try:  # collective: every rank gets the same outcome, so every rank takes the same branch
                peers = P2P.ipc_peers(dist.group.WORLD, Tl, c["N"], c["d"])
            except Exception as e:
                log(f"peer-memory EP unavailable ({type(e).__name__}: {e}); using NCCL collectives")
        if peers is not None:
            result = run_ep_p2p(args, c, rank, world, local_rank, peers)
        else:
            result = run_ep(args, c, rank, world, local_rank)
    elif "layers" in c:
        result = run_stack(args, c)
    else:
        result = run_single(args, c)
    if rank == 0:
        if world == 1 and not args.no_cpu_baseline:
            result["cpu_baseline"] = cpu_baseline(c)
            result["cpu_baseline_f64_tanh2"] = cpu_baseline_tanh2(c)
        print(json.dumps(result), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
