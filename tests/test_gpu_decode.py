"""GPU parity of the decode stack around the MoE layer:
the attention stand-in kernels, the graphed multi-layer decode step and the
device trace ring, against the CPU oracle's restatement of simulate()
(simulator.py:273-357).

Per layer the stack is teacher-forced: each layer's GPU input is fed to the
oracle, so selections are compared bit-exactly on the kernel's own logits
and outputs within the bf16 tolerance, with no drift across layers.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import has_gpu
from oracle import lynx_oracle as O

pytestmark = pytest.mark.gpu

TOL = 1e-2

if has_gpu():
    import torch

    import paper_2411_08982_b200 as L
    from paper_2411_08982_b200 import _native as nat


def f64(t):
    return t.detach().float().cpu().numpy().astype(np.float64)


def attn_host(attn, l):
    """(wq, wk, wv, wo) of layer l as the oracle takes them ([d, dh] x3, [dh, d])."""
    w = f64(attn.wqkv[l])
    dh = attn.d_head
    return w[:dh].T, w[dh:2 * dh].T, w[2 * dh:].T, f64(attn.wo[l])


def test_attention_chunk_vs_oracle():
    """lynx_attention on a chunk of Tn tokens over a pre-filled cache prefix."""
    B, d, dh, S0, max_len = 3, 256, 16, 5, 32
    attn = L.build_attention(1, d, dh, seed=3)
    k_cache = torch.zeros((B, max_len, dh), dtype=torch.float32, device="cuda")
    v_cache = torch.zeros_like(k_cache)
    k_cache[:, :S0] = torch.randn((B, S0, dh), device="cuda")
    v_cache[:, :S0] = torch.randn((B, S0, dh), device="cuda")
    a = nat.LynxAttention()
    a.d_model, a.d_head, a.max_len = d, dh, max_len
    a.wqkv, a.wo, a.k_cache, a.v_cache = (nat.ptr(attn.wqkv[0]), nat.ptr(attn.wo[0]), nat.ptr(k_cache),
                                          nat.ptr(v_cache))
    for Tn, norm in ((1, False), (4, False), (1, True)):
        h = torch.randn((B * Tn, d), device="cuda").to(torch.bfloat16) * 3
        out = torch.empty_like(h)
        pos = torch.tensor([S0], dtype=torch.int32, device="cuda")
        ws = torch.empty((int(nat.lib().lynx_attention_workspace_bytes(B * Tn, dh)),), dtype=torch.uint8,
                         device="cuda")
        keys0, vals0 = f64(k_cache[:, :S0]), f64(v_cache[:, :S0])
        st = nat.lib().lynx_attention(L.router.ctypes_ref(a), h.data_ptr(), B, Tn, int(norm), pos.data_ptr(),
                                      out.data_ptr(), ws.data_ptr(), ws.numel(), torch.cuda.current_stream().cuda_stream)
        assert st == 0
        torch.cuda.synchronize()
        x = f64(h).reshape(B, Tn, d)
        if norm:
            x = O.rms_norm(x)
        ref, keys, vals = O.attention(x, *attn_host(attn, 0), keys0, vals0, S0)
        assert O.norm_rel_err(f64(out).reshape(B, Tn, d), x + ref) <= TOL
        assert O.norm_rel_err(f64(out).reshape(B, Tn, d) - x, ref) <= 5e-2  # attention part alone
        assert np.allclose(f64(k_cache[:, :S0 + Tn]), keys, rtol=1e-3, atol=1e-4)
        assert np.allclose(f64(v_cache[:, :S0 + Tn]), vals, rtol=1e-3, atol=1e-4)


def _stack(L_layers=3, N=8, k=2, d=128, ff=256, B=4, policy=None, seed=0, **kw):
    spec = L.MoEModelSpec(L_layers, N, k, d, ff)
    moe = L.build_swiglu_model(spec, seed=seed)
    attn = L.build_attention(L_layers, d, 16, seed=seed + 1)
    return spec, moe, attn, L.DecodeStack(moe, attn, B, max_len=16, policy=policy, **kw)


def test_decode_stack_teacher_forced_vs_oracle():
    """Every layer of prefill + 3 decode steps: attention output and cache
    entries vs the oracle, selection bit-exact vs the oracle on the GPU
    logits, MoE output vs the fp32 SwiGLU oracle."""
    pol = L.PolicyConfig(mode="latency", drop_count=3)
    seen = []

    def probe(l, phase, h_in, mid, out, layer):
        fused = phase is L.Phase.DECODE and stack.fused_router
        seen.append((l, phase, h_in.clone(), mid.clone(), out.clone(), layer.mask(),
                     layer.expert_ids.clone(), int(stack.pos.item()),
                     stack.k_cache[l].clone(), stack.v_cache[l].clone(),
                     stack.logits.clone() if fused else None))

    spec, moe, attn, stack = _stack(policy=pol, probe=probe)
    B, P, d = 4, 3, spec.d_model
    x = np.random.default_rng(0).normal(size=(B, P, d))
    stack.simulate(x, 3)
    assert len(seen) == spec.num_layers * 4
    assert stack.fused_router
    for l, phase, h_in, mid, out, mask, ids, pos, kc, vc, fused_logits in seen:
        decode = phase is L.Phase.DECODE
        Tn = 1 if decode else P
        xin = f64(h_in).reshape(B, Tn, d)
        if decode and l == 0:
            xin = O.rms_norm(xin)  # the step input is rms_norm(prev)
        ref_a, keys, vals = O.attention(xin, *attn_host(attn, l), f64(kc[:, :pos]), f64(vc[:, :pos]), pos)
        assert O.norm_rel_err(f64(mid).reshape(B, Tn, d), xin + ref_a) <= TOL, (l, phase)
        assert np.allclose(f64(kc[:, :pos + Tn]), keys, rtol=1e-3, atol=1e-4), (l, phase)
        # routing on the kernel's logits (decode: the router fused into the
        # attention kernel; prefill: K0): bit-exact decisions
        k0_logits = f64(L.router_logits(moe, l, mid))
        if fused_logits is not None:
            logits = f64(fused_logits)
            assert np.allclose(logits, k0_logits, rtol=1e-5, atol=1e-5), (l, phase)
        else:
            logits = k0_logits
        r_ids, r_probs, r_full = O.route(logits, spec.top_k)
        opol = O.Policy(mode="latency", drop_count=3)
        ref_mask = O.apply(r_ids, r_probs, r_full, opol, decode=decode)
        assert np.array_equal(ids.cpu().numpy(), r_ids), (l, phase)
        assert np.array_equal(mask.remap_assigned.cpu().numpy(), ref_mask.assigned), (l, phase)
        if decode:
            assert len(mask.retained) == spec.num_experts - 3
        w1, w3 = L.unpack_w13(moe.w13[l], spec.d_ff)
        ref = O.forward_swiglu(f64(mid).astype(np.float32), f64(w1), f64(w3), f64(moe.w2[l]), ref_mask.assigned,
                               ref_mask.weights, round_h_bf16=True)
        assert O.norm_rel_err(f64(out), ref) <= TOL, (l, phase)


def test_decode_graph_replay_matches_eager():
    """The captured decode step (one graph launch per step) is bit-identical
    to the eager layer-by-layer path."""
    pol = L.PolicyConfig(mode="accuracy", freq_keep_budget=2)
    x = np.random.default_rng(1).normal(size=(4, 2, 128))
    _, _, _, eager = _stack(policy=pol, graph=False, seed=5)
    a = eager.simulate(x, 4).hidden
    _, _, _, graphed = _stack(policy=pol, graph=True, seed=5)
    b = graphed.simulate(x, 4).hidden
    assert torch.equal(a, b)
    # and a second simulate on the same graphed stack restarts cleanly
    c = graphed.simulate(x, 4).hidden
    assert torch.equal(a, c)


def test_trace_ring_matches_host_records(tmp_path):
    """Device trace ring (graphed decode) == host-side records of the same
    events taken through the eager probe path; JSONL round trip."""
    pol = L.PolicyConfig(mode="accuracy", freq_keep_budget=3)
    x = np.random.default_rng(2).normal(size=(4, 2, 128))
    host_trace, host_masks = [], []

    def probe(l, phase, h_in, mid, out, layer):
        event = 0 if phase is L.Phase.PREFILL else 1 + int(stack_e.pos.item()) - 2
        sel = L.ExpertSelection(expert_ids=layer.expert_ids.clone(), probs=layer.probs.clone(),
                                full_probs=layer.full_probs.clone())
        m = layer.mask()
        host_trace.extend(L.trace.records_from_event("run", event, l, phase, sel, m))
        if phase is L.Phase.PREFILL:
            m = L.ExpertMask(layer_index=l, phase=phase, retained=m.retained, remap_original=m.remap_original,
                             remap_assigned=m.remap_assigned, remap_weights=m.remap_weights, clipped=m.clipped,
                             important_tokens=None)
        host_masks.append(L.trace.mask_record_from_event("run", event, l, phase, m))

    _, _, _, stack_e = _stack(policy=pol, probe=probe, seed=7)
    stack_e.simulate(x, 3)
    spec, moe, attn, _ = _stack(seed=7)
    rec = L.TraceRecorder("run", spec.num_layers, 4, spec.num_experts, spec.top_k, capacity=2)
    stack_g = L.DecodeStack(moe, attn, 4, max_len=16, policy=pol, trace=rec)
    stack_g.simulate(x, 3)
    got = rec.records()
    key = lambda r: (r.batch_id, r.layer, r.token_id, r.rank)  # noqa: E731
    assert sorted(got, key=key) == sorted(host_trace, key=key)
    gm = sorted(rec.mask_records(), key=lambda m: (m.batch_id, m.layer))
    hm = sorted(host_masks, key=lambda m: (m.batch_id, m.layer))
    assert gm == hm
    path = tmp_path / "run.jsonl"
    rec.write(path)
    assert L.read_trace_jsonl(path) == got
    assert L.read_masks_jsonl(L.masks_path_for(path)) == rec.mask_records()


def test_decode_stack_vs_reference_simulate():
    """The whole GPU decode stack (attention stand-in + Lynx layer, graphed
    decode steps, device trace ring) on the reference's own model against
    the reference's simulate() output (tests/golden/simulate.npz): every
    routing event's expert ids, assignment and retained set bit-exact, weights
    to 1e-2 (they come from bf16-state logits), final states within the bf16
    tolerance of the f64 reference."""
    from conftest import load_simulate_golden
    meta, w, x, cases = load_simulate_golden()
    Ln, N, k, d, ff = meta["L"], meta["N"], meta["k"], meta["d"], meta["ff"]

    class Ref:  # duck-typed moetrim SyntheticMoE
        pass
    ref = Ref()
    ref.spec = L.MoEModelSpec(Ln, N, k, d, ff)
    ref.router_w, ref.w1, ref.w2 = w["router"], w["1"], w["2"]
    ref.wq, ref.wk, ref.wv, ref.wo, ref.d_head = w["q"], w["k"], w["v"], w["o"], meta["d_head"]
    moe = L.from_reference(ref)
    attn = L.attention_from_reference(ref)
    for case in cases:
        p = case["policy"]
        pol = None if p is None else L.PolicyConfig(**{f: (tuple(v) if isinstance(v, list) else v)
                                                       for f, v in p.items()})
        rec = L.TraceRecorder("golden", Ln, meta["B"], N, k, capacity=8)
        stack = L.DecodeStack(moe, attn, meta["B"], max_len=16, policy=pol, trace=rec)
        out = stack.simulate(x, meta["steps"]).hidden
        assert O.norm_rel_err(f64(out), case["hidden"]) <= 2e-2, case["name"]
        got = {}
        for r in rec.records():
            got.setdefault((r.batch_id, r.layer), []).append(r)
        for ev in case["events"]:
            recs = sorted(got[(ev["event"], ev["layer"])], key=lambda r: (r.token_id, r.rank))
            T = len(recs) // k
            ids = np.array([r.expert_original for r in recs]).reshape(T, k)
            asg = np.array([r.expert_assigned for r in recs]).reshape(T, k)
            wts = np.array([r.weight for r in recs]).reshape(T, k)
            tag = (case["name"], ev["event"], ev["layer"])
            assert np.array_equal(ids, ev["ids"]), tag
            assert np.array_equal(asg, ev["assigned"]), tag
            assert np.allclose(wts, ev["weights"], atol=1e-2), tag
            ref_t = sorted(ev["trace"], key=lambda r: (r["token_id"], r["rank"]))
            assert [(r["token_id"], r["rank"], r["expert_original"], r["expert_assigned"]) for r in ref_t] == \
                [(r.token_id, r.rank, r.expert_original, r.expert_assigned) for r in recs], tag
        masks = {(m.batch_id, m.layer): m for m in rec.mask_records()}
        for ev in case["events"]:
            m, rm = masks[(ev["event"], ev["layer"])], ev["mask"]
            assert list(m.retained) == list(rm["retained"]) and m.clipped == rm["clipped"], ev
            assert m.num_tokens == rm["num_tokens"] and m.num_important == rm["num_important"], ev


def test_decode_stack_two_kernel_attention():
    """Decode steps normally run the attention as one clustered kernel
    (attn_out_kernel<true>); LYNX_ATTN_CLUSTER=0 keeps attn_qkv + attn_out.
    Rerun the stack's parity tests through the two-kernel path."""
    import os
    import subprocess
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    env = dict(os.environ, LYNX_ATTN_CLUSTER="0")
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider",
                        os.path.join(here, "test_gpu_decode.py"), "-k",
                        "teacher_forced or reference_simulate or graph_replay"],
                       env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, (r.stdout[-3000:], r.stderr[-2000:])
