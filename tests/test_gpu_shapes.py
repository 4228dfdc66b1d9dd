"""GPU parity at the full BASELINE.json shapes the layer is benchmarked on.

C2 (Mixtral-8x7B layer, T=32), C5 (Mixtral-8x22B layer, d=6144, ff=16384)
at T=32 and at T=256 through the CTA-pair K3 kernel, and the C3 decode stack
(d=4096, 32 layers, batch 64) teacher-forced over prefill + 2 decode steps.

Semantics matched: forward_layer (simulator.py:86-113) and the decode loop
(simulator.py:329-357).  The fp32 oracle here does NOT round the SwiGLU
intermediate to bf16 (round_h_bf16=False): the kernel's bf16 H is part of
what is checked.  Tolerances (north star), norm-wise
max|y - y_ref| / max|y_ref|:
  * the f32 expert sum from lynx_moe_forward_partial (no residual, no bf16
    output rounding)                                        <= 1e-2
  * the bf16 layer output (residual included)               <= 1e-2
  * the bf16 layer output minus the input (expert part)     <= 2e-2
Selections are bit-exact against the oracle on the kernel's own logits.
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


def f32(t):
    return t.detach().float().cpu().numpy()


def used_weights(model, layer, experts):
    """fp32 host copies of only the experts a mask uses (w1, w3 [ff, d]; w2 [d, ff])."""
    ff = model.spec.d_ff
    w1, w3, w2 = {}, {}, {}
    for e in experts:
        a, b = L.unpack_w13(model.w13[layer][e:e + 1], ff)
        w1[e], w3[e], w2[e] = f32(a[0]), f32(b[0]), f32(model.w2[layer][e])
    return w1, w3, w2


def oracle_expert_sum(model, layer, hidden_f32, assigned, weights, residual):
    N, S = model.spec.num_experts, model.spec.num_shared_experts
    experts = sorted(set(int(e) for e in assigned.ravel() if e >= 0)) + list(range(N, N + S))
    w1, w3, w2 = used_weights(model, layer, experts)
    return O.forward_swiglu(hidden_f32, w1, w3, w2, assigned.astype(np.int64), weights, round_h_bf16=False,
                            shared=range(N, N + S), residual=residual)


def check_layer(model, T, policy, seed, want_kernel=None):
    g = torch.Generator(device="cuda").manual_seed(seed)
    hidden = torch.randn((T, model.spec.d_model), generator=g, device="cuda").to(torch.bfloat16)
    layer = L.LynxMoELayer(model, 0, T, policy=policy)
    if want_kernel is not None:
        assert layer.ffn_kernel() == want_kernel
    y = layer(hidden)
    torch.cuda.synchronize()
    # selection bit-exact vs the oracle on the kernel's logits
    logits = L.router_logits(model, 0, hidden).cpu().numpy()
    ids, probs, full = O.route(logits, model.spec.top_k)
    opol = O.Policy(mode=policy.mode, drop_count=policy.drop_count, freq_keep_budget=policy.freq_keep_budget)
    m = O.apply(ids, probs, full, opol)
    assert np.array_equal(layer.expert_ids.cpu().numpy(), ids)
    assert np.array_equal(layer.assigned.cpu().numpy(), m.assigned)
    x = f32(hidden)
    # f32 expert sum (lynx_moe_forward_partial): no residual, no output rounding
    part = L.forward_partial(hidden, model, 0, layer.assigned.contiguous(), layer.weights.contiguous())
    ref_sum = oracle_expert_sum(model, 0, x, m.assigned, m.weights, residual=False)
    e_sum = O.norm_rel_err(f32(part), ref_sum)
    ref_y = x + ref_sum
    e_y = O.norm_rel_err(f32(y), ref_y)
    e_delta = O.norm_rel_err(f32(y) - x, ref_sum)
    print(f"T={T} d={model.spec.d_model} ff={model.spec.d_ff} kernel={layer.ffn_kernel()} "
          f"used={layer.used_experts()} err: expert-sum {e_sum:.2e} layer {e_y:.2e} expert-part {e_delta:.2e}")
    assert e_sum <= TOL
    assert e_y <= TOL
    assert e_delta <= 2 * TOL
    return layer


def test_c2_mixtral_layer_unrounded_oracle():
    """C2: Mixtral-8x7B layer, T=32, latency drop 4, vs the un-rounded fp32 oracle."""
    model = L.build_swiglu_model(L.MoEModelSpec(1, 8, 2, 4096, 14336), seed=0)
    check_layer(model, 32, L.PolicyConfig(mode="latency", drop_count=4), seed=0, want_kernel="ffn_kernel")


@pytest.fixture(scope="module")
def c5_model():
    model = L.build_swiglu_model(L.MoEModelSpec(1, 8, 2, 6144, 16384), seed=5)
    yield model
    del model
    torch.cuda.empty_cache()


def test_c5_mixtral_8x22b_layer_T32(c5_model):
    """C5 layer shape (d=6144, ff=16384, N=8, k=2, latency drop 4), T=32."""
    check_layer(c5_model, 32, L.PolicyConfig(mode="latency", drop_count=4), seed=1, want_kernel="ffn_kernel")


def test_c5_mixtral_8x22b_layer_T256_cta_pair(c5_model):
    """C5 at T=256 (the decode-batch-256 config on one GPU): ~128 rows per used
    expert, so K3 runs the CTA-pair kernel (tcgen05 cta_group::2) at its
    production geometry."""
    check_layer(c5_model, 256, L.PolicyConfig(mode="latency", drop_count=4), seed=2,
                want_kernel="ffn_pair_kernel")


def test_c5_no_lynx_T256_cta_pair(c5_model):
    """C5 T=256 with every expert kept (drop 0): 8 used experts, ~64 rows each."""
    check_layer(c5_model, 256, L.PolicyConfig(mode="latency", drop_count=0), seed=3,
                want_kernel="ffn_pair_kernel")


def test_c3_full_stack_teacher_forced():
    """C3: the Mixtral-8x7B 32-layer decode stack (d=4096, ff=14336, batch 64,
    latency drop 4) through prefill + 2 graph-free decode steps, teacher
    forced: every layer's routing is bit-exact vs the oracle on the kernel's
    logits (96 routing events); attention and MoE outputs are checked
    against the oracle on a spread of layers (every event at layers 0, 1,
    15, 31)."""
    nl, B, P, d, ff, dh = 32, 64, 2, 4096, 14336, 16
    spec = L.MoEModelSpec(nl, 8, 2, d, ff)
    moe = L.build_swiglu_model(spec, seed=0)
    attn = L.build_attention(nl, d, dh, seed=1)
    pol = L.PolicyConfig(mode="latency", drop_count=4)
    checked = {0, 1, 15, nl - 1}
    seen = []

    def probe(l, phase, h_in, mid, out, layer):
        full = l in checked
        seen.append(dict(l=l, phase=phase, ids=layer.expert_ids.cpu().numpy(), asg=layer.assigned.cpu().numpy(),
                         w=layer.weights.cpu().numpy(), mid=mid.clone(),
                         # the logits the layer routed on: decode steps take the router fused
                         # into the attention kernel, prefill runs K0
                         logits=(stack.logits if phase is L.Phase.DECODE and stack.fused_router
                                 else L.router_logits(moe, l, mid)).cpu().numpy(),
                         h_in=h_in.clone() if full else None, out=out.clone() if full else None,
                         pos=int(stack.pos.item()),
                         kc=stack.k_cache[l].clone() if full else None, vc=stack.v_cache[l].clone() if full else None))

    stack = L.DecodeStack(moe, attn, B, max_len=8, policy=pol, probe=probe)
    x = np.random.default_rng(2).normal(size=(B, P, d))
    res = stack.simulate(x, 2)
    assert bool(torch.isfinite(res.hidden.float()).all())
    assert len(seen) == nl * 3
    assert stack.fused_router
    for ev in seen:
        decode = ev["phase"] is L.Phase.DECODE
        r_ids, r_probs, r_full = O.route(ev["logits"], 2)
        ref_mask = O.apply(r_ids, r_probs, r_full, O.Policy(mode="latency", drop_count=4), decode=decode)
        assert np.array_equal(ev["ids"], r_ids), (ev["l"], ev["phase"])
        assert np.array_equal(ev["asg"], ref_mask.assigned), (ev["l"], ev["phase"])
        assert np.allclose(ev["w"], ref_mask.weights, rtol=1e-12, atol=1e-15), (ev["l"], ev["phase"])
        if ev["h_in"] is None:
            continue
        l, Tn = ev["l"], 1 if decode else P
        xin = f32(ev["h_in"]).astype(np.float64).reshape(B, Tn, d)
        if decode and l == 0:
            xin = O.rms_norm(xin)
        wqkv = f32(attn.wqkv[l]).astype(np.float64)
        aw = (wqkv[:dh].T, wqkv[dh:2 * dh].T, wqkv[2 * dh:].T, f32(attn.wo[l]).astype(np.float64))
        pos = ev["pos"]
        ref_a, _, _ = O.attention(xin, *aw, f32(ev["kc"][:, :pos]).astype(np.float64),
                                  f32(ev["vc"][:, :pos]).astype(np.float64), pos)
        assert O.norm_rel_err(f32(ev["mid"]).reshape(B, Tn, d), xin + ref_a) <= TOL, (l, ev["phase"])
        mid = f32(ev["mid"])
        ref_sum = oracle_expert_sum(moe, l, mid, ref_mask.assigned, ref_mask.weights, residual=False)
        err = O.norm_rel_err(f32(ev["out"]), mid + ref_sum)
        # the expert sum itself in f32 (lynx_moe_forward_partial on the same input and mask): the
        # depth-damped experts (W2 / sqrt(2L)) add little to the residual, so out - mid would be
        # dominated by the bf16 rounding of the output
        part = L.forward_partial(ev["mid"], moe, l, torch.from_numpy(ev["asg"]).cuda(),
                                 torch.from_numpy(ev["w"]).cuda())
        err_sum = O.norm_rel_err(f32(part), ref_sum)
        print(f"layer {l} {ev['phase'].value}: layer err {err:.2e} expert-sum {err_sum:.2e}")
        assert err <= TOL, (l, ev["phase"])
        assert err_sum <= TOL, (l, ev["phase"])
