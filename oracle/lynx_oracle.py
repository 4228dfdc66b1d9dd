"""CPU oracle for the Lynx MoE decode hot path.  TEST INFRASTRUCTURE ONLY.

This module is the checker, never the product: only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import it.  The shipped package
(``paper_2411_08982_b200``) never imports anything under ``oracle/``; it
fails loudly when its CUDA library is missing.

It restates, in plain numpy + explicit Python loops, the reference
algorithm of ``moetrim`` (``/root/reference/pkg/src/moetrim``):

* routing math          -- router.py:141-192
* retention policies    -- policy.py:116-350
* MoE layer dispatch    -- simulator.py:26-27, 77-113

Parity pin: every function here is checked against golden vectors that
``tests/golden/make_golden.py`` produced by importing the reference
itself (``tests/test_oracle_golden.py``), plus the reference tests'
known-answer cases.  Decisions (ids, retained sets, remaps, important
tokens, permutation order) are bit-exact; float64 probabilities agree to
the last ulp on the machine that made the fixtures and to 1e-12 elsewhere
(numpy's SIMD ``exp`` differs by <=1 ulp between CPUs).

Besides the reference's own ``tanh(x W1) W2`` expert (``expert_mlp``,
simulator.py:77-79, "tanh2" mode) the oracle carries the SwiGLU expert
the north star asks for, ``(silu(x W1^T) * (x W3^T)) W2^T`` in fp32.  The
reference has no SwiGLU, so that expert's numerics are pinned by this
oracle alone; its dispatch/combine semantics are
the reference's forward_layer (simulator.py:86-113).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

RMS_EPS = 1e-12  # simulator.py:23


class OracleError(ValueError):
    """Mirror of moetrim.errors.ValidationError (errors.py:4-5)."""


# --------------------------------------------------------------------------
# numpy's float64 summation order (the reference sums with ndarray.sum)
# --------------------------------------------------------------------------

def pairwise_sum(values) -> float:
    """numpy's pairwise summation of a contiguous float64 run.

    ``e.sum(axis=-1)`` in router.py:154, ``probs.sum(axis=1)`` in
    policy.py:220 and ``slot_p.sum()`` in policy.py:205 all reduce with
    numpy's pairwise scheme: fewer than 8 terms are added left to right
    onto the additive identity; up to 128 terms use eight strided partial
    sums folded as ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) followed by the
    leftover tail; longer runs split at an 8-aligned midpoint.  Verified
    bit-exact against numpy 2.3 for n = 1..513 (tests/test_oracle_golden.py).
    The CUDA selection kernel implements the same recursion.
    """
    a = [float(v) for v in values]
    return _pairwise(a, 0, len(a))


def _pairwise(a, lo, n):
    if n < 8:
        acc = 0.0
        for i in range(lo, lo + n):
            acc = acc + a[i]
        return acc
    if n <= 128:
        part = a[lo:lo + 8]
        body = n - (n % 8)
        for base in range(lo + 8, lo + body, 8):
            for j in range(8):
                part[j] = part[j] + a[base + j]
        acc = ((part[0] + part[1]) + (part[2] + part[3])) + \
              ((part[4] + part[5]) + (part[6] + part[7]))
        for i in range(lo + body, lo + n):
            acc = acc + a[i]
        return acc
    half = n // 2
    half -= half % 8
    return _pairwise(a, lo, half) + _pairwise(a, lo + half, n - half)


# --------------------------------------------------------------------------
# numpy's float64 exp (the reference's np.exp, router.py:153)
# --------------------------------------------------------------------------

# numpy 2.x on x86-64 AVX512_SKX hosts (this build container, which made
# tests/golden/) computes float64 exp with the Intel SVML routine bundled in
# numpy (__svml_exp8_ha, numpy/_core/src/umath/svml).  It is NOT correctly
# rounded, so the device restates it step for step (csrc/npexp.cuh).  The
# constants below are that routine's (read from numpy 2.3.5's
# _multiarray_umath data table __svml_dexp_ha_data_internal_avx512):
# 2^(j/16) = _EXP_HI[j] + _EXP_LO[j], ln2 = _LN2_HI + _LN2_LO, and the
# degree-5 polynomial _EXP_C for (e^r - 1) / r.
_EXP_HI = [float.fromhex(h) for h in (
    "0x1.0000000000000p+0", "0x1.0b5586cf9890fp+0", "0x1.172b83c7d517bp+0", "0x1.2387a6e756238p+0",
    "0x1.306fe0a31b715p+0", "0x1.3dea64c123422p+0", "0x1.4bfdad5362a27p+0", "0x1.5ab07dd485429p+0",
    "0x1.6a09e667f3bcdp+0", "0x1.7a11473eb0187p+0", "0x1.8ace5422aa0dbp+0", "0x1.9c49182a3f090p+0",
    "0x1.ae89f995ad3adp+0", "0x1.c199bdd85529cp+0", "0x1.d5818dcfba487p+0", "0x1.ea4afa2a490dap+0")]
_EXP_LO = [float.fromhex(h) for h in (
    "0x0p+0", "0x1.79aa65d837b6dp-54", "-0x1.01b15eaa59348p-55", "0x1.68efde3a8a894p-54",
    "0x1.34d754db0abb6p-55", "0x1.59f48a72a4c6dp-55", "0x1.690cebb7aafb0p-56", "0x1.063e1e21c5409p-54",
    "-0x1.3b3efbf5e2228p-54", "-0x1.b32dcb94da51dp-56", "0x1.db72fc1f0eab4p-55", "0x1.1affc2b91ce27p-56",
    "0x1.c1a7792cb3387p-55", "0x1.36eae30af0cb3p-56", "0x1.4a385a63d07a7p-56", "-0x1.ff7128fd391f0p-55")]
_LOG2E = float.fromhex("0x1.71547652b82fep+0")
_SHIFT = float.fromhex("0x1.8000000003ff0p+48")
_LN2_HI = float.fromhex("0x1.62e42fefa39efp-1")
_LN2_LO = float.fromhex("0x1.abc9e3b39803fp-56")
_EXP_C = [float.fromhex(h) for h in (  # c0 .. c5
    "0x1.fffffffffff70p-1", "0x1.000000000d008p-1", "0x1.5555553939732p-3",
    "0x1.55557242d68fep-5", "0x1.1101cbbc265c0p-7", "0x1.7411836940c04p-10")]
_EXP_RARE = float.fromhex("0x1.61da04cbafe44p+9")


def _fma(a: float, b: float, c: float, toward_zero: bool = False) -> float:
    """a*b + c with one rounding (exact rational arithmetic), nearest-even or toward zero."""
    from fractions import Fraction
    exact = Fraction(a) * Fraction(b) + Fraction(c)
    f = float(exact)  # correctly rounded to nearest
    if toward_zero and Fraction(f) != exact and abs(Fraction(f)) > abs(exact):
        import math
        f = math.nextafter(f, 0.0)
    return f


def svml_exp_ha(x: float) -> float:
    """np.exp(x) for float64 on AVX512_SKX hosts, restated step for step
    (the same steps as csrc/npexp.cuh np_exp).  |x| >= 707.7 and NaN take
    SVML's scalar fallback, which this restatement does not cover."""
    import math
    x = float(x)
    if not abs(x) < _EXP_RARE:
        raise OracleError("svml_exp_ha: argument outside the vector path")
    t = _fma(x, _LOG2E, _SHIFT, toward_zero=True)
    n = t - _SHIFT
    j = int(np.array(t).view(np.uint64)) & 15
    r = _fma(-n, _LN2_HI, x)
    r = _fma(-_LN2_LO, n, r)
    r2 = r * r
    c0, c1, c2, c3, c4, c5 = _EXP_C
    p = _fma(c5, r, c4)
    q = _fma(c3, r, c2)
    s = _fma(c1, r, c0)
    p = _fma(r2, p, q)
    p = _fma(r2, p, s)
    p = _fma(p, r, _EXP_LO[j])
    p = _fma(_EXP_HI[j], p, _EXP_HI[j])
    return math.ldexp(p, math.floor(n))


def numpy_uses_svml_exp() -> bool:
    """True when this numpy dispatches float64 exp to SVML (AVX512_SKX)."""
    try:
        from numpy._core._multiarray_umath import __cpu_features__ as f
    except ImportError:  # pragma: no cover - numpy < 2
        from numpy.core._multiarray_umath import __cpu_features__ as f
    return bool(f.get("AVX512_SKX"))


# --------------------------------------------------------------------------
# routing (router.py)
# --------------------------------------------------------------------------

def check_logits(logits) -> np.ndarray:
    """RoutingLogits.__post_init__ (router.py:65-73): f64, 2-D, non-empty, finite."""
    z = np.asarray(logits, dtype=np.float64)
    if z.ndim != 2:
        raise OracleError(f"logits must be 2-D, got shape {z.shape}")
    if z.shape[0] < 1 or z.shape[1] < 1:
        raise OracleError(f"logits must be non-empty, got shape {z.shape}")
    if not np.all(np.isfinite(z)):
        raise OracleError("logits contain non-finite values")
    return z


def softmax_rows(z: np.ndarray) -> np.ndarray:
    """softmax_probs (router.py:141-154): exp(z - rowmax) / pairwise row sum."""
    z = check_logits(z)
    e = np.exp(z - z.max(axis=1, keepdims=True))
    out = np.empty_like(e)
    for t in range(e.shape[0]):
        out[t] = e[t] / pairwise_sum(e[t])
    return out


def topk_rows(full: np.ndarray, k: int) -> tuple[np.ndarray, np.ndarray]:
    """route_batch's stable argsort of -p (router.py:181-182).

    Order key: probability descending, expert index ascending.
    """
    T, N = full.shape
    if not (1 <= k <= N):
        raise OracleError(f"k must be in [1, {N}], got {k}")
    ids = np.empty((T, k), dtype=np.int64)
    for t in range(T):
        order = sorted(range(N), key=lambda e: (-full[t, e], e))
        ids[t] = order[:k]
    return ids, np.take_along_axis(full, ids, axis=1)


def route(logits, k: int):
    """route_batch (router.py:174-187) -> (expert_ids, probs, full_probs)."""
    z = check_logits(logits)
    if not (1 <= k <= z.shape[1]):
        raise OracleError(f"k must be in [1, {z.shape[1]}], got {k}")
    full = softmax_rows(z)
    ids, probs = topk_rows(full, k)
    return ids, probs, full


def confidence(full: np.ndarray, metric: str = "top1") -> np.ndarray:
    """ExpertSelection.confidence (router.py:125-138)."""
    if metric == "top1":
        return full.max(axis=1)
    if metric == "margin":
        if full.shape[1] == 1:
            return full[:, 0].copy()
        s = np.sort(full, axis=1)
        return s[:, -1] - s[:, -2]
    raise OracleError(f"unknown confidence metric {metric!r}")


# --------------------------------------------------------------------------
# policies (policy.py)
# --------------------------------------------------------------------------

@dataclass(frozen=True)
class Policy:
    """PolicyConfig (policy.py:26-65) as the oracle needs it."""

    mode: str = "latency"
    drop_count: int = 0
    confidence_threshold: float = 0.5
    sample_threshold: int = 8
    min_experts: int | None = None
    freq_keep_budget: int = 4
    confidence_metric: str = "top1"
    vote_rank_weights: tuple | None = None

    def floor(self, top_k: int) -> int:
        """resolved_min_experts (policy.py:57-65)."""
        if self.min_experts is None:
            return top_k
        if self.min_experts < top_k:
            raise OracleError(
                f"min_experts ({self.min_experts}) must be >= top_k ({top_k})")
        return self.min_experts


def votes(ids: np.ndarray, N: int, rank_weights=None) -> np.ndarray:
    """vote_expert_frequencies (policy.py:116-138).

    bincount walks the flattened [T, k] slots in row-major order; the
    weighted variant adds rank_weights[r] in that same order.
    """
    T, k = ids.shape
    counts = np.zeros(N, dtype=np.float64)
    if rank_weights is not None and len(rank_weights) != k:
        raise OracleError(f"rank_weights must have length top_k={k}")
    for t in range(T):
        for r in range(k):
            counts[ids[t, r]] += 1.0 if rank_weights is None else float(rank_weights[r])
    return counts


def retention_order(counts: np.ndarray) -> list[int]:
    """_retention_order (policy.py:141-148): count desc, expert index asc."""
    return sorted(range(len(counts)), key=lambda e: (-counts[e], e))


def remap(ids: np.ndarray, full: np.ndarray, retained) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
    """remap_tokens (policy.py:151-212) -> (original, assigned, weights)."""
    keep = sorted(set(int(e) for e in np.asarray(retained).ravel()))
    if not keep:
        raise OracleError("retained set must be non-empty")
    N = full.shape[1]
    if keep[0] < 0 or keep[-1] >= N:
        raise OracleError("retained contains out-of-range expert ids")
    keep_set = set(keep)
    T, k = ids.shape
    assigned = np.empty_like(ids)
    weights = np.empty((T, k), dtype=np.float64)
    for t in range(T):
        p = full[t]
        cands = sorted(keep, key=lambda e: (-p[e], e))
        taken = {int(e) for e in ids[t] if int(e) in keep_set}
        for r in range(k):
            e0 = int(ids[t, r])
            if e0 in keep_set:
                assigned[t, r] = e0
                continue
            pick = next((c for c in cands if c not in taken), cands[0])
            assigned[t, r] = pick
            taken.add(pick)
        slot_p = p[assigned[t]]
        total = pairwise_sum(slot_p)
        if total <= 0.0:
            raise OracleError("token has zero probability mass on the assigned experts")
        weights[t] = slot_p / total
    return ids.copy(), assigned, weights


@dataclass
class Mask:
    """ExpertMask (policy.py:83-113) fields."""

    retained: np.ndarray
    original: np.ndarray
    assigned: np.ndarray
    weights: np.ndarray
    clipped: bool
    important: np.ndarray | None
    counts: np.ndarray | None = None


def identity_mask(ids: np.ndarray, probs: np.ndarray, N: int) -> Mask:
    """full_retain_mask (policy.py:215-229)."""
    w = np.empty_like(probs)
    for t in range(probs.shape[0]):
        w[t] = probs[t] / pairwise_sum(probs[t])
    return Mask(np.arange(N, dtype=np.int64), ids.copy(), ids.copy(), w, False, None)


def important_tokens(full: np.ndarray, pol: Policy) -> np.ndarray:
    """select_important_tokens (policy.py:267-284)."""
    conf = confidence(full, pol.confidence_metric)
    q = [t for t in range(len(conf)) if conf[t] >= pol.confidence_threshold]
    if not q:
        best = 0
        for t in range(1, len(conf)):
            if conf[t] > conf[best]:
                best = t
        return np.array([best], dtype=np.int64)
    if len(q) > pol.sample_threshold:
        q = sorted(q, key=lambda t: (-conf[t], t))[: pol.sample_threshold]
    return np.array(sorted(q), dtype=np.int64)


def latency(ids, probs, full, pol: Policy, decode: bool = True) -> Mask:
    """latency_policy (policy.py:232-264)."""
    N = full.shape[1]
    if not decode:
        return identity_mask(ids, probs, N)
    floor = pol.floor(ids.shape[1])
    counts = votes(ids, N, pol.vote_rank_weights)
    eff = min(pol.drop_count, max(0, N - floor))
    order = retention_order(counts)
    keep = np.array(sorted(order[: N - eff]), dtype=np.int64)
    orig, assigned, w = remap(ids, full, keep)
    return Mask(keep, orig, assigned, w, eff != pol.drop_count, None, counts)


def accuracy(ids, probs, full, pol: Policy, decode: bool = True) -> Mask:
    """accuracy_policy (policy.py:287-338)."""
    N = full.shape[1]
    if not decode:
        return identity_mask(ids, probs, N)
    floor = pol.floor(ids.shape[1])
    imp = important_tokens(full, pol)
    counts = votes(ids[imp], N, pol.vote_rank_weights)
    order = retention_order(counts)
    voted = [e for e in order if counts[e] > 0]
    keep = set(voted[: min(pol.freq_keep_budget, N)])
    keep.update(int(e) for e in ids[imp, 0])
    padded = False
    for e in order:
        if len(keep) >= floor:
            break
        if e not in keep:
            keep.add(e)
            padded = True
    keep_arr = np.array(sorted(keep), dtype=np.int64)
    orig, assigned, w = remap(ids, full, keep_arr)
    return Mask(keep_arr, orig, assigned, w, padded, imp, counts)


def apply(ids, probs, full, pol: Policy, decode: bool = True) -> Mask:
    """apply_policy (policy.py:341-350)."""
    if pol.mode == "latency":
        return latency(ids, probs, full, pol, decode)
    if pol.mode == "accuracy":
        return accuracy(ids, probs, full, pol, decode)
    raise OracleError(f"unknown policy mode {pol.mode!r}")


# --------------------------------------------------------------------------
# dispatch / combine (simulator.py:86-113)
# --------------------------------------------------------------------------

@dataclass
class Dispatch:
    """Permutation the layer applies: experts ascending, tokens ascending.

    experts[u]     -- u-th used expert (np.unique(assigned), simulator.py:104)
    rows[u]        -- token rows served by it, ascending (simulator.py:105-106)
    row_weight[u]  -- merged gate weight per row: 0 + sum over that row's
                      slots on the expert, slot order (simulator.py:108-111)
    """

    experts: list
    rows: list
    row_weight: list


def dispatch(assigned: np.ndarray, weights: np.ndarray) -> Dispatch:
    T, k = assigned.shape
    experts = sorted(set(int(e) for e in assigned.ravel()))
    rows, row_w = [], []
    for e in experts:
        toks = [t for t in range(T) if any(int(assigned[t, c]) == e for c in range(k))]
        ws = []
        for t in toks:
            acc = 0.0
            for c in range(k):
                if int(assigned[t, c]) == e:
                    acc += float(weights[t, c])
            ws.append(acc)
        rows.append(np.array(toks, dtype=np.int64))
        row_w.append(np.array(ws, dtype=np.float64))
    return Dispatch(experts, rows, row_w)


def rms_norm(x: np.ndarray) -> np.ndarray:
    """rms_norm (simulator.py:26-27)."""
    return x / np.sqrt(np.mean(np.square(x), axis=-1, keepdims=True) + RMS_EPS)


def router_logits(hidden: np.ndarray, router_w: np.ndarray) -> np.ndarray:
    """router_logits (simulator.py:82-83); router_w is [d, N]."""
    return rms_norm(hidden) @ router_w


def silu(x):
    return x / (1.0 + np.exp(-x))


def forward_swiglu(hidden, w1, w3, w2, assigned, weights, dtype=np.float32,
                   round_h_bf16: bool = False, shared=(), residual: bool = True):
    """forward_layer (simulator.py:86-113) with a SwiGLU expert.

    hidden [T, d]; w1, w3 [E, ff, d]; w2 [E, d, ff] (HF Mixtral / K-major
    layout).  expert(x) = (silu(x w1^T) * (x w3^T)) w2^T.  Residual plus
    merged-weight combine in ascending expert order, like the reference.
    ``round_h_bf16`` rounds the intermediate activation to bf16 the way
    the CUDA kernel stores it (used to tighten tolerances, not required).
    ``shared`` lists always-on experts (indices into w1/w3/w2) applied to
    every token with weight 1 after the routed experts, in the given order
    -- the builder's DeepSeek-MoE extension; the reference has none.
    ``residual=False`` returns the expert sum alone (what
    lynx_moe_forward_partial computes); w1/w3/w2 may be dicts holding only
    the experts the mask uses.
    """
    x = np.asarray(hidden, dtype=dtype)
    if x.shape[0] != assigned.shape[0]:
        raise OracleError(
            f"mask covers {assigned.shape[0]} tokens but hidden has {x.shape[0]}")
    out = x.copy() if residual else np.zeros_like(x)
    disp = dispatch(assigned, weights)

    def expert(e, xr):
        g = xr @ np.asarray(w1[e], dtype=dtype).T
        u = xr @ np.asarray(w3[e], dtype=dtype).T
        h = (silu(g) * u).astype(dtype)
        if round_h_bf16:
            h = bf16_round(h)
        return h @ np.asarray(w2[e], dtype=dtype).T

    for e, rows, rw in zip(disp.experts, disp.rows, disp.row_weight):
        out[rows] += rw.astype(dtype)[:, None] * expert(e, x[rows])
    for e in shared:
        out += expert(e, x)
    return out


def forward_tanh2(hidden, w1, w2, assigned, weights):
    """forward_layer (simulator.py:86-113) with the reference expert
    ``tanh(x @ w1) @ w2`` (simulator.py:77-79); w1 [E, d, ff], w2 [E, ff, d], f64."""
    x = np.asarray(hidden, dtype=np.float64)
    if x.shape[0] != assigned.shape[0]:
        raise OracleError(
            f"mask covers {assigned.shape[0]} tokens but hidden has {x.shape[0]}")
    out = x.copy()
    disp = dispatch(assigned, weights)
    for e, rows, rw in zip(disp.experts, disp.rows, disp.row_weight):
        y = np.tanh(x[rows] @ w1[e]) @ w2[e]
        out[rows] += rw[:, None] * y
    return out


def bf16_round(a: np.ndarray) -> np.ndarray:
    """Round float32 values to the nearest bfloat16 (ties to even), as float32."""
    a = np.ascontiguousarray(a, dtype=np.float32)
    bits = a.view(np.uint32).astype(np.uint64)
    lsb = (bits >> 16) & 1
    bits = (bits + 0x7FFF + lsb) & 0xFFFF0000
    return bits.astype(np.uint32).view(np.float32).reshape(a.shape)


def norm_rel_err(y, y_ref) -> float:
    """max|y - y_ref| / max|y_ref| -- the layer-output tolerance metric."""
    y = np.asarray(y, dtype=np.float64)
    y_ref = np.asarray(y_ref, dtype=np.float64)
    return float(np.max(np.abs(y - y_ref)) / max(np.max(np.abs(y_ref)), 1e-30))


# --------------------------------------------------------------------------
# decode stack around the layer (simulator.py:273-357)
# --------------------------------------------------------------------------

def attention(h, wq, wk, wv, wo, keys, vals, offset):
    """The single-head attention stand-in (simulator.py:308-326) for one layer.

    h [B, Tn, d]; wq/wk/wv [d, dh]; wo [dh, d]; keys/vals [B, S, dh] hold the
    S cached positions.  The chunk sits at positions offset .. offset+Tn-1
    and attends causally.  Returns (attention output [B, Tn, d], keys, vals)
    with the chunk's k/v appended -- the caller adds the residual
    (simulator.py:333).
    """
    h = np.asarray(h, dtype=np.float64)
    xn = rms_norm(h)
    q = xn @ wq
    keys = np.concatenate([keys, xn @ wk], axis=1)
    vals = np.concatenate([vals, xn @ wv], axis=1)
    scores = np.einsum("bth,bsh->bts", q, keys) / np.sqrt(wq.shape[1])
    total, t_new = keys.shape[1], h.shape[1]
    allowed = np.arange(total)[None, :] <= (offset + np.arange(t_new))[:, None]
    scores = np.where(allowed[None], scores, -np.inf)
    a = np.exp(scores - scores.max(axis=-1, keepdims=True))
    a = a / a.sum(axis=-1, keepdims=True)
    return np.einsum("bts,bsh->bth", a, vals) @ wo, keys, vals


def simulate(inputs, decode_steps, num_layers, attn_weights, moe_layer):
    """simulate() (simulator.py:273-357) with a pluggable MoE sublayer.

    attn_weights[l] = (wq, wk, wv, wo); moe_layer(l, phase, flat [T, d]) ->
    flat output ("prefill" / "decode").  Returns hidden [B, P + D, d].
    """
    x = np.asarray(inputs, dtype=np.float64)
    B, P, d = x.shape
    dh = attn_weights[0][0].shape[1]
    keys = [np.zeros((B, 0, dh)) for _ in range(num_layers)]
    vals = [np.zeros((B, 0, dh)) for _ in range(num_layers)]
    out = np.zeros((B, P + decode_steps, d))

    def chunk(h, phase, offset):
        for l in range(num_layers):
            a, keys[l], vals[l] = attention(h, *attn_weights[l], keys[l], vals[l], offset)
            h = h + a
            Bc, Tc, _ = h.shape
            h = moe_layer(l, phase, h.reshape(Bc * Tc, d)).reshape(Bc, Tc, d)
        return h

    h = chunk(x, "prefill", 0)
    out[:, :P] = h
    prev = h[:, -1]
    for s in range(decode_steps):
        h = chunk(rms_norm(prev)[:, None, :], "decode", P + s)
        out[:, P + s] = h[:, 0]
        prev = h[:, 0]
    return out
