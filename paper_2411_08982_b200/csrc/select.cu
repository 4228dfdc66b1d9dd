// select.cu -- K0 router GEMV (+RMSNorm), K1 fused route + retention policy
// + remap + dispatch plan, and the small kernels behind the modular API.
// Decisions are bit-exact with the reference's float64 numpy path (see
// oracle/lynx_oracle.py for the restated algorithm).
//
// Reference:
//   rms_norm / router_logits   simulator.py:26-27, 82-83
//   softmax_probs              router.py:141-154
//   route_batch (stable top-k) router.py:174-187
//   confidence                 router.py:125-138
//   vote_expert_frequencies    policy.py:116-138
//   _retention_order           policy.py:141-148
//   remap_tokens               policy.py:151-212
//   full_retain_mask           policy.py:215-229
//   latency_policy             policy.py:232-264
//   select_important_tokens    policy.py:267-284
//   accuracy_policy            policy.py:287-338
//   dispatch order             simulator.py:104-112
//
// These kernels are latency-bound (a decode batch is a few KB of routing
// state): K1 is one CTA -- a thread per token for N <= 16 (route_select_fast),
// eight lanes per token otherwise (route_select_group) -- with every
// per-token array staged in shared memory when it fits, and rolled loops:
// the kernel runs once per layer from a cold instruction cache.
#include <cooperative_groups.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <stdlib.h>

#include "lynx_internal.cuh"
#include "npexp.cuh"
#include "p2p.cuh"
#include "ptx.cuh"

namespace lynx {

constexpr unsigned kFull = 0xffffffffu;

// Diagnostic library only (-DLYNX_TRACE): phase timestamps of the last K1.
#ifdef LYNX_TRACE
__device__ unsigned long long g_sel_ts[32];
#define SEL_TS(i)                                      \
  do {                                                 \
    __syncthreads();                                   \
    if (threadIdx.x == 0) g_sel_ts[i] = globaltimer(); \
  } while (0)
#define SEL_TS_LOCAL(i) \
  do {                                                 \
    if (threadIdx.x == 0) g_sel_ts[i] = globaltimer(); \
  } while (0)
// K0 (router_route_kernel) phases of block (0, 0), slots 8..12 (free when K1 runs on a given selection)
#define K0_TS(i)                                                                                   \
  do {                                                                                             \
    if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) g_sel_ts[8 + (i)] = globaltimer(); \
  } while (0)
#else
#define SEL_TS(i) (void)0
#define SEL_TS_LOCAL(i) (void)0
#define K0_TS(i) (void)0
#endif

// numpy's pairwise float64 summation (oracle.pairwise_sum): < 8 terms added
// left to right; <= 128 terms with 8 strided partials folded pairwise plus
// the tail; longer runs split at an 8-aligned midpoint.
__device__ __noinline__ double np_pairwise_sum(const double* a, int n) {
  if (n < 8) {
    double acc = 0.0;
    for (int i = 0; i < n; ++i) acc += a[i];
    return acc;
  }
  if (n <= 128) {
    double r[8];
    for (int j = 0; j < 8; ++j) r[j] = a[j];
    const int body = n - (n % 8);
    for (int i = 8; i < body; i += 8)
      for (int j = 0; j < 8; ++j) r[j] += a[i + j];
    double acc = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (int i = body; i < n; ++i) acc += a[i];
    return acc;
  }
  int half = n / 2;
  half -= half % 8;
  return np_pairwise_sum(a, half) + np_pairwise_sum(a + half, n - half);
}

__device__ __forceinline__ uint64_t expert_mask_all(int N) { return N == 64 ? ~0ull : ((1ull << N) - 1); }

// Warp argmax over the experts in `cand` by (value desc, index asc); each
// lane holds experts lane and lane+32.  Returns the index (-1 if none) and
// writes the value to *bv.  All lanes get the result.
__device__ __noinline__ int warp_best(double v0, double v1, uint64_t cand, double* bv) {
  const int lane = threadIdx.x & 31;
  double best = -1.0;
  int bi = -1;
  if ((cand >> lane) & 1ull) {
    best = v0;
    bi = lane;
  }
  if (((cand >> (lane + 32)) & 1ull) && (bi < 0 || v1 > best)) {
    best = v1;
    bi = lane + 32;
  }
  for (int off = 16; off > 0; off >>= 1) {
    const double ov = __shfl_xor_sync(kFull, best, off);
    const int oi = __shfl_xor_sync(kFull, bi, off);
    if (oi >= 0 && (bi < 0 || ov > best || (ov == best && oi < bi))) {
      best = ov;
      bi = oi;
    }
  }
  *bv = best;
  return bi;
}

__device__ __forceinline__ double lane_value(double v0, double v1, int e) {
  const double a = __shfl_sync(kFull, v0, e & 31);
  const double b = __shfl_sync(kFull, v1, e & 31);
  return e < 32 ? a : b;
}

// remap_tokens for one token (policy.py:171-210), one warp.
__device__ __noinline__ void remap_token(const int32_t* ids, const double* p, int k, int N, uint64_t keep,
                                         int32_t* assigned, double* weights, int* flags) {
  const int lane = threadIdx.x & 31;
  const double v0 = lane < N ? p[lane] : 0.0;
  const double v1 = lane + 32 < N ? p[lane + 32] : 0.0;
  uint64_t occupied = 0;
  for (int r = 0; r < k; ++r) {
    const int e = ids[r];
    if ((keep >> e) & 1ull) occupied |= 1ull << e;
  }
  double slot_p[LYNX_MAX_TOPK];
  for (int r = 0; r < k; ++r) {
    int e = ids[r];
    if (!((keep >> e) & 1ull)) {
      double bv;
      int pick = warp_best(v0, v1, keep & ~occupied, &bv);
      if (pick < 0) pick = warp_best(v0, v1, keep, &bv);  // collapse (policy.py:197-200)
      e = pick;
      occupied |= 1ull << e;
    }
    slot_p[r] = lane_value(v0, v1, e);
    if (lane == 0) assigned[r] = e;
  }
  if (lane == 0) {
    const double total = np_pairwise_sum(slot_p, k);
    if (!(total > 0.0)) atomicOr(flags, LYNX_FLAG_ZERO_MASS);
    for (int r = 0; r < k; ++r) weights[r] = slot_p[r] / total;
  }
}

// ------------------------------------------------------------- dispatch plan
// forward_layer's grouping (simulator.py:104-112): used experts ascending,
// each expert's token rows ascending, a token's duplicate slots on one expert
// merged (weights summed in slot order).  Rows of expert e occupy
// [base[e], base[e] + cnt[e]) of the permuted buffer, base 16-aligned;
// segments split an expert at LYNX_SEG_ROWS rows.  Called by every thread
// of one CTA; `asg`/`w` may live in shared or global memory.
__device__ __forceinline__ void plan_dispatch(const int32_t* asg, const double* w, int T, int N, int k,
                                           const PlanOut& o, uint32_t* s_bits, int* s_prefix) {
  // The plan's pointers in registers: through the `o` reference every global
  // store below would force a reload of the fields (possible aliasing).
  int32_t* __restrict__ const o_n_seg = o.n_seg;
  int32_t* __restrict__ const o_n_used = o.n_used;
  int32_t* __restrict__ const o_n_rows = o.n_rows;
  int32_t* __restrict__ const o_max_rows = o.max_rows;
  int32_t* __restrict__ const o_seg_expert = o.seg_expert;
  int32_t* __restrict__ const o_seg_row = o.seg_row;
  int32_t* __restrict__ const o_seg_count = o.seg_count;
  int32_t* __restrict__ const o_seg_order = o.seg_order;
  int32_t* __restrict__ const o_perm_token = o.perm_token;
  float* __restrict__ const o_perm_weight = o.perm_weight;
  int32_t* __restrict__ const o_tok_rows = o.tok_rows;
  float* __restrict__ const o_tok_weight = o.tok_weight;
  int* __restrict__ const o_counters = o.counters;
  __shared__ int s_cnt[LYNX_MAX_EXPERTS];
  __shared__ int s_base[LYNX_MAX_EXPERTS];
  __shared__ int s_shared_base;
  constexpr int kOrderMax = 256;  // segments ranked in shared memory (more: identity order)
  __shared__ int s_segcnt[kOrderMax];
  const int W = (T + 31) >> 5;
  const int S = o.n_shared, kk = k + S, T16 = (T + 15) & ~15;
  const int tid = threadIdx.x, nthr = blockDim.x;
  #pragma unroll 1
  for (int i = tid; i < N * W; i += nthr) s_bits[i] = 0;
  __syncthreads();
  #pragma unroll 1
  for (int i = tid; i < T * k; i += nthr) {
    const int e = asg[i];
    if (e >= 0 && e < N) {
      const int t = i / k;
      atomicOr(&s_bits[e * W + (t >> 5)], 1u << (t & 31));
    }
  }
  __syncthreads();
  #pragma unroll 1
  for (int e = tid; e < N; e += nthr) {
    int run = 0;
    #pragma unroll 1
    for (int q = 0; q < W; ++q) {
      s_prefix[e * W + q] = run;
      run += __popc(s_bits[e * W + q]);
    }
    s_cnt[e] = run;
  }
  #pragma unroll 1
  for (int i = tid; i < o.n_counters; i += nthr) o_counters[i] = 0;
  __syncthreads();
  if (tid < 32) {
    // Expert bases and segment slots: one warp scans the 16-padded row counts
    // and segment counts over experts ascending (lane l: experts l, l + 32).
    const int lane = tid;
    int cnt[2], pad[2], nsg[2], base[2], seg[2];
    #pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int e = lane + 32 * h;
      cnt[h] = e < N ? s_cnt[e] : 0;
      pad[h] = (cnt[h] + 15) & ~15;
      nsg[h] = (cnt[h] + LYNX_SEG_ROWS - 1) / LYNX_SEG_ROWS;
    }
    int row_off = 0, seg_off = 0;
    #pragma unroll
    for (int h = 0; h < 2; ++h) {
      int rs = pad[h], ss = nsg[h];
      #pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int r2 = __shfl_up_sync(kFull, rs, off), s2 = __shfl_up_sync(kFull, ss, off);
        if (lane >= off) {
          rs += r2;
          ss += s2;
        }
      }
      base[h] = row_off + rs - pad[h];
      seg[h] = seg_off + ss - nsg[h];
      row_off += __shfl_sync(kFull, rs, 31);
      seg_off += __shfl_sync(kFull, ss, 31);
    }
    #pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int e = lane + 32 * h;
      if (e < N) s_base[e] = base[h];
      #pragma unroll 1
      for (int c = 0; c < nsg[h]; ++c) {
        const int rows = min(LYNX_SEG_ROWS, cnt[h] - c * LYNX_SEG_ROWS);
        o_seg_expert[seg[h] + c] = e;
        o_seg_row[seg[h] + c] = base[h] + c * LYNX_SEG_ROWS;
        o_seg_count[seg[h] + c] = rows;
        if (seg[h] + c < kOrderMax) s_segcnt[seg[h] + c] = rows;
      }
    }
    const int nused = __popc(__ballot_sync(kFull, cnt[0] > 0)) + __popc(__ballot_sync(kFull, cnt[1] > 0));
    // shared experts: every token, in token order, after the routed experts
    const int seg_per_shared = (T + LYNX_SEG_ROWS - 1) / LYNX_SEG_ROWS;
    #pragma unroll 1
    for (int i = lane; i < S * seg_per_shared; i += 32) {
      const int sx = i / seg_per_shared, c = i - sx * seg_per_shared;
      const int rows = min(LYNX_SEG_ROWS, T - c * LYNX_SEG_ROWS);
      o_seg_expert[seg_off + i] = N + sx;
      o_seg_row[seg_off + i] = row_off + sx * T16 + c * LYNX_SEG_ROWS;
      o_seg_count[seg_off + i] = rows;
      if (seg_off + i < kOrderMax) s_segcnt[seg_off + i] = rows;
    }
    // widest segment (K3 sizes its pipeline stages by it)
    int widest = max(min(cnt[0], LYNX_SEG_ROWS), min(cnt[1], LYNX_SEG_ROWS));
    widest = __reduce_max_sync(kFull, widest);
    if (S > 0) widest = max(widest, min(T, LYNX_SEG_ROWS));
    if (lane == 0) {
      s_shared_base = row_off;
      if (o_max_rows) *o_max_rows = widest;
      *o_n_seg = seg_off + S * seg_per_shared;
      *o_n_used = nused + S;
      *o_n_rows = row_off + S * T16;
    }
  }
  __syncthreads();
  if (o_seg_order) {  // K3 queue order: rows desc, segment index asc (largest first)
    const int nseg = *o_n_seg;  // written by lane 0 above; visible after the barrier
    #pragma unroll 1
    for (int i = tid; i < nseg; i += nthr) {
      if (nseg > kOrderMax) {
        o_seg_order[i] = i;
        continue;
      }
      const int ci = s_segcnt[i];
      int rank = 0;
      #pragma unroll 4
      for (int j = 0; j < nseg; ++j) {
        const int cj = s_segcnt[j];
        rank += (cj > ci || (cj == ci && j < i)) ? 1 : 0;
      }
      o_seg_order[rank] = i;
    }
  }
  // Per token: its distinct experts ascending (bit scan of a 64-bit set), the
  // permuted row of each and the merged weight 0 + sum of its slots on that
  // expert in slot order (simulator.py:108-111).
  #pragma unroll 1
  for (int t = tid; t < T; t += nthr) {
    int a_r[LYNX_MAX_TOPK];
    uint64_t set = 0;
    #pragma unroll
    for (int c = 0; c < LYNX_MAX_TOPK; ++c) {
      a_r[c] = c < k ? asg[t * k + c] : -1;
      if (a_r[c] >= 0 && a_r[c] < N) set |= 1ull << a_r[c];
    }
    int j = 0;
    while (set) {
      const int e = __ffsll(static_cast<long long>(set)) - 1;
      set &= set - 1;
      const uint32_t word = s_bits[e * W + (t >> 5)];
      const int row = s_base[e] + s_prefix[e * W + (t >> 5)] + __popc(word & ((1u << (t & 31)) - 1u));
      double acc = 0.0;
      #pragma unroll
      for (int c = 0; c < LYNX_MAX_TOPK; ++c)
        if (a_r[c] == e) acc += w[t * k + c];
      const float wf = static_cast<float>(acc);
      o_tok_rows[t * kk + j] = row;
      o_tok_weight[t * kk + j] = wf;
      o_perm_token[row] = t;
      o_perm_weight[row] = wf;
      ++j;
    }
    #pragma unroll 1
    for (; j < k; ++j) {
      o_tok_rows[t * kk + j] = -1;
      o_tok_weight[t * kk + j] = 0.f;
    }
    #pragma unroll 1
    for (int sx = 0; sx < S; ++sx) {
      const int row = s_shared_base + sx * T16 + t;
      o_tok_rows[t * kk + k + sx] = row;
      o_tok_weight[t * kk + k + sx] = 1.f;
      o_perm_token[row] = t;
      o_perm_weight[row] = 1.f;
    }
  }
  // zero the 16-row padding of every segment run
  #pragma unroll 1
  for (int e = tid; e < N; e += nthr) {
    const int cnt = s_cnt[e];
    #pragma unroll 1
    for (int r = s_base[e] + cnt; r < s_base[e] + ((cnt + 15) & ~15); ++r) {
      o_perm_token[r] = -1;
      o_perm_weight[r] = 0.f;
    }
  }
  #pragma unroll 1
  for (int i = tid; i < S * (T16 - T); i += nthr) {
    const int row = s_shared_base + (i / (T16 - T)) * T16 + T + i % (T16 - T);
    o_perm_token[row] = -1;
    o_perm_weight[row] = 0.f;
  }
}

// Shared-memory carve-up of K1 (the host computes the same size).
struct SelectSmem {
  size_t p, conf, ids, probs, asg, w, imp, bits, prefix, total;
};

__host__ __device__ inline SelectSmem select_smem(int T, int N, int k, bool stage, bool plan) {
  SelectSmem s{};
  size_t off = 0;
  auto take = [&](size_t b) {
    const size_t o = off;
    off = (off + b + 15) & ~size_t(15);
    return o;
  };
  if (stage) {
    s.p = take(sizeof(double) * T * N);
    s.conf = take(sizeof(double) * T);
    s.ids = take(sizeof(int32_t) * T * k);
    s.probs = take(sizeof(double) * T * k);
    s.asg = take(sizeof(int32_t) * T * k);
    s.w = take(sizeof(double) * T * k);
  }
  s.imp = take(T);
  if (plan) {
    const int W = (T + 31) >> 5;
    s.bits = take(sizeof(uint32_t) * N * W);
    s.prefix = take(sizeof(int) * N * W);
  }
  s.total = off;
  return s;
}

// Batch-level policy: vote, retention order, retained set (policy.py:116-148,
// 232-338).  Writes s_keep / s_counts; returns via s_clipped.
__device__ __forceinline__ void batch_policy(const SelectArgs& a, const int32_t* IDS, const double* CONF, uint8_t* IMP,
                                          int* s_keep, double* s_counts, int* s_icount, int* s_rank, int* s_order,
                                          int* s_nq, int* s_clipped) {
  const int T = a.T, N = a.N, k = a.k, tid = threadIdx.x, nthr = blockDim.x;
  const int lane = tid & 31, warp = tid >> 5, nwarps = nthr >> 5;
  const bool accuracy = a.pol.mode == LYNX_POLICY_ACCURACY;
  const int floor_keep = a.floor_keep, drop = a.pol.drop_count, budget_cfg = a.pol.freq_keep_budget;
  const int n_rank_weights = a.pol.n_rank_weights;
  if (accuracy) {  // select_important_tokens
    const double tau = a.pol.confidence_threshold;
    int local = 0;
    #pragma unroll 1
    for (int t = tid; t < T; t += nthr) {
      const bool q = CONF[t] >= tau;
      IMP[t] = q ? 1 : 0;
      local += q;
    }
    if (local) atomicAdd(s_nq, local);
    __syncthreads();
    SEL_TS_LOCAL(16);
    const int nq = *s_nq;
    const int S = a.pol.sample_threshold;
    if (nq == 0) {
      if (warp == 0) {  // [argmax conf]: first maximum, one warp
        double best = -1.0;
        int bi = -1;
        #pragma unroll 1
        for (int t = lane; t < T; t += 32)
          if (bi < 0 || CONF[t] > best) {
            best = CONF[t];
            bi = t;
          }
        #pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
          const double ob = __shfl_xor_sync(kFull, best, off);
          const int oi = __shfl_xor_sync(kFull, bi, off);
          if (oi >= 0 && (bi < 0 || ob > best || (ob == best && oi < bi))) {
            best = ob;
            bi = oi;
          }
        }
        if (lane == 0) IMP[bi] = 1;
      }
    } else if (nq > S) {
      // keep the S most confident (conf desc, t asc): a warp per candidate,
      // lanes count the better candidates; ranks read CONF only, so marking
      // drops in bit 1 is race-free
      #pragma unroll 1
      for (int t = warp; t < T; t += nwarps) {
        if (!IMP[t]) continue;  // warp-uniform
        const double ct = CONF[t];
        int better = 0;
        #pragma unroll 1
        for (int u = lane; u < T; u += 32) {
          const double cu = CONF[u];
          better += (cu >= tau && (cu > ct || (cu == ct && u < t))) ? 1 : 0;
        }
        better = __reduce_add_sync(kFull, better);
        __syncwarp();  // every lane's read of IMP[t] above precedes lane 0's write
        if (lane == 0 && better >= S) IMP[t] |= 2;
      }
      __syncthreads();
      #pragma unroll 1
      for (int t = tid; t < T; t += nthr) IMP[t] = IMP[t] == 1;
    }
    __syncthreads();
  }
  SEL_TS_LOCAL(17);
  // Unit votes are integers: order-free atomics are exact.  Rank-weighted
  // votes are float sums and keep numpy's slot order (thread per expert).
  if (!n_rank_weights) {
    #pragma unroll 1
    for (int i = tid; i < T * k; i += nthr)
      if (!accuracy || IMP[i / k]) atomicAdd(&s_icount[IDS[i]], 1);
    __syncthreads();
    #pragma unroll 1
    for (int e = tid; e < N; e += nthr) s_counts[e] = static_cast<double>(s_icount[e]);
  } else {
    #pragma unroll 1
    for (int e = tid; e < N; e += nthr) {
      double c = 0.0;
      #pragma unroll 1
      for (int t = 0; t < T; ++t) {
        if (accuracy && !IMP[t]) continue;
        #pragma unroll 1
        for (int r = 0; r < k; ++r)
          if (IDS[t * k + r] == e) c += a.pol.rank_weights[r];
      }
      s_counts[e] = c;
    }
  }
  __syncthreads();
  SEL_TS_LOCAL(18);
  // retention order (count desc, index asc): a thread per expert for small
  // N, else a warp per expert with one ballot per 32 competitors
  if (N <= 32 || nwarps < 4) {
    #pragma unroll 1
    for (int e = tid; e < N; e += nthr) {
      const double ce = s_counts[e];
      int rank = 0;
      #pragma unroll 4
      for (int f = 0; f < N; ++f) {
        const double cf = s_counts[f];
        rank += (cf > ce || (cf == ce && f < e)) ? 1 : 0;
      }
      s_rank[e] = rank;
      s_order[rank] = e;
    }
  } else {
  #pragma unroll 1
  for (int e = warp; e < N; e += nwarps) {
    const double ce = s_counts[e];
    int rank = 0;
    #pragma unroll 1
    for (int f0 = 0; f0 < N; f0 += 32) {
      const int f = f0 + lane;
      const double cf = f < N ? s_counts[f] : 0.0;
      rank += __popc(__ballot_sync(kFull, f < N && (cf > ce || (cf == ce && f < e))));
    }
    if (lane == 0) {
      s_rank[e] = rank;
      s_order[rank] = e;
    }
  }
  }
  __syncthreads();
  SEL_TS_LOCAL(19);
  if (!accuracy) {  // latency_policy
    const int room = N - floor_keep > 0 ? N - floor_keep : 0;
    const int eff = drop < room ? drop : room;
    #pragma unroll 1
    for (int e = tid; e < N; e += nthr) s_keep[e] = s_rank[e] < N - eff;
    if (tid == 0) *s_clipped = eff != drop;
  } else {  // accuracy_policy
    const int budget = budget_cfg < N ? budget_cfg : N;
    #pragma unroll 1
    for (int e = tid; e < N; e += nthr) s_keep[e] = (s_counts[e] > 0.0 && s_rank[e] < budget) ? 1 : 0;
    __syncthreads();
    #pragma unroll 1
    for (int t = tid; t < T; t += nthr)
      if (IMP[t]) s_keep[IDS[t * k]] = 1;
    __syncthreads();
    if (warp == 0) {
      // pad from the retention order up to the floor: the first (floor - kept)
      // unkept experts by rank, found with two ballots (N <= 64)
      const bool k0 = lane < N && s_keep[lane], k1 = lane + 32 < N && s_keep[lane + 32];
      const int kept = __popc(__ballot_sync(kFull, k0)) + __popc(__ballot_sync(kFull, k1));
      const int need = floor_keep - kept;
      if (need > 0) {
        const int e0 = lane < N ? s_order[lane] : -1, e1 = lane + 32 < N ? s_order[lane + 32] : -1;
        const bool u0 = e0 >= 0 && !s_keep[e0], u1 = e1 >= 0 && !s_keep[e1];
        const unsigned b0 = __ballot_sync(kFull, u0), b1 = __ballot_sync(kFull, u1);
        const unsigned below = (1u << lane) - 1u;
        if (u0 && __popc(b0 & below) < need) s_keep[e0] = 1;
        if (u1 && __popc(b0) + __popc(b1 & below) < need) s_keep[e1] = 1;
      }
      if (lane == 0) *s_clipped = need > 0;
    }
  }
}

// ------------------------------------------------- K1 fast path (N <= 16)
// One thread per token with its whole probability row in registers: the N
// exps are independent (they interleave), numpy's pairwise sum and the
// stable top-k run on registers, and the same thread keeps its row from
// routing through the remap.  Probabilities are np_exp(z - max) / sum --
// numpy's exp bits, numpy's summation order and a true IEEE division -- so
// full_probs equal the reference's bit for bit and float64 near-ties order
// as they do there.
template <int NT>
__device__ __forceinline__ double reg_pairwise_sum(const double (&e)[NT], int n) {
  if (n < 8) {
    double acc = 0.0;
#pragma unroll
    for (int i = 0; i < (NT < 8 ? NT : 8); ++i)
      if (i < n) acc += e[i];
    return acc;
  }
  double r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = e[j];
  const int body = n - (n % 8);
#pragma unroll
  for (int i = 8; i < NT; ++i)
    if (i < body) r[i % 8] += e[i];
  double acc = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
#pragma unroll
  for (int i = 8; i < NT; ++i)
    if (i >= body && i < n) acc += e[i];
  return acc;
}

// best index in `cand` by (value desc, index asc) over a register row
template <int NT>
__device__ __forceinline__ int reg_best(const double (&p)[NT], uint64_t cand) {
  int best = -1;
  double bv = 0.0;
#pragma unroll
  for (int i = 0; i < NT; ++i)
    if (((cand >> i) & 1ull) && (best < 0 || p[i] > bv)) {
      best = i;
      bv = p[i];
    }
  return best;
}

template <int NT>
__device__ __forceinline__ double reg_at(const double (&p)[NT], int e) {
  double v = 0.0;
#pragma unroll
  for (int i = 0; i < NT; ++i)
    if (i == e) v = p[i];
  return v;
}

template <int NT>
__global__ void __launch_bounds__(kSelectThreads) route_select_fast(const __grid_constant__ SelectArgs a) {
  __shared__ double s_counts[LYNX_MAX_EXPERTS];
  __shared__ int s_icount[LYNX_MAX_EXPERTS];
  __shared__ int s_rank[LYNX_MAX_EXPERTS];
  __shared__ int s_order[LYNX_MAX_EXPERTS];
  __shared__ int s_keep[LYNX_MAX_EXPERTS];
  __shared__ int s_flags, s_nq, s_clipped;
  __shared__ unsigned long long s_keepmask;
  __shared__ double s_exp[32];
  extern __shared__ __align__(16) uint8_t s_dyn[];

  griddep_launch_dependents();
  const int T = a.T, N = a.N, k = a.k;
  const int t = threadIdx.x;
  if (a.logits) np_exp_stage(s_exp);
  const bool active = t < T;
  const SelectSmem L = select_smem(T, N, k, true, a.plan.enabled);
  double* CONF = reinterpret_cast<double*>(s_dyn + L.conf);
  int32_t* IDS = reinterpret_cast<int32_t*>(s_dyn + L.ids);
  int32_t* ASG = reinterpret_cast<int32_t*>(s_dyn + L.asg);
  double* WT = reinterpret_cast<double*>(s_dyn + L.w);
  uint8_t* IMP = s_dyn + L.imp;
  if (t == 0) {
    s_flags = 0;
    s_nq = 0;
    s_clipped = 0;
  }
  if (t < N) s_icount[t] = 0;
  warm_params(a);
  __syncthreads();  // s_exp
  SEL_TS(0);
  griddep_wait();  // logits come from K0 (programmatic dependent launch)
  if (a.ep.enabled) {  // peer-memory EP: every rank's logits rows have landed
    if (threadIdx.x == 0) wait_peers(a.ep.P, a.ep.kind, *a.ep.P.epoch + 1);
    __syncthreads();
  }
  SEL_TS(1);

  // 1) softmax + stable top-k + confidence, thread per token
  double p[NT];
  int ids[LYNX_MAX_TOPK];
  double probs[LYNX_MAX_TOPK];
  if (active) {
    if (a.logits) {
      const double* z = a.logits + static_cast<size_t>(t) * N;
#pragma unroll
      for (int i = 0; i < NT; ++i) p[i] = i < N ? z[i] : 0.0;
      bool finite = true;
      double m = p[0];
#pragma unroll
      for (int i = 0; i < NT; ++i)
        if (i < N) {
          finite &= isfinite(p[i]);
          m = p[i] > m ? p[i] : m;
        }
      if (!finite) atomicOr(&s_flags, LYNX_FLAG_NONFINITE);
#pragma unroll
      for (int i = 0; i < NT; ++i) p[i] = i < N ? np_exp(p[i] - m, s_exp) : 0.0;
      const double sum = reg_pairwise_sum<NT>(p, N);
#pragma unroll
      for (int i = 0; i < NT; ++i) p[i] = p[i] / sum;  // e / s, as numpy divides (router.py:154)
      uint64_t taken = ~expert_mask_all(N);
#pragma unroll 1
      for (int r = 0; r < k; ++r) {
          const int b = reg_best<NT>(p, ~taken);
          taken |= 1ull << b;
          ids[r] = b;
          probs[r] = reg_at<NT>(p, b);
          a.ids[t * k + r] = b;
          a.probs[t * k + r] = probs[r];
        }
#pragma unroll
      for (int i = 0; i < NT; ++i)
        if (i < N) a.full[static_cast<size_t>(t) * N + i] = p[i];
    } else {
      const double* row = a.full + static_cast<size_t>(t) * N;
#pragma unroll
      for (int i = 0; i < NT; ++i) p[i] = i < N ? row[i] : 0.0;
#pragma unroll 1
      for (int r = 0; r < k; ++r) {
          ids[r] = a.ids[t * k + r];
          probs[r] = a.probs[t * k + r];
        }
    }
    const int first = reg_best<NT>(p, expert_mask_all(N));
    const double top1 = reg_at<NT>(p, first);
    double c = top1;
    if (a.pol.confidence_metric == LYNX_CONF_MARGIN)
      c = N == 1 ? p[0] : top1 - reg_at<NT>(p, reg_best<NT>(p, expert_mask_all(N) & ~(1ull << first)));
    CONF[t] = c;
#pragma unroll 1
    for (int r = 0; r < k; ++r) IDS[t * k + r] = ids[r];
  }
  __syncthreads();
  SEL_TS(2);

  const bool run_policy = a.decode && a.pol.mode != LYNX_POLICY_NONE;
  const bool accuracy = run_policy && a.pol.mode == LYNX_POLICY_ACCURACY;
  if (!run_policy) {
    if (t < N) {
      s_keep[t] = 1;
      s_counts[t] = 0.0;
    }
    if (active) IMP[t] = 0;
  } else {
    batch_policy(a, IDS, CONF, IMP, s_keep, s_counts, s_icount, s_rank, s_order, &s_nq, &s_clipped);
  }
  __syncthreads();
  if (t == 0) {
    unsigned long long mk = 0;
    for (int e = 0; e < N; ++e)
      if (s_keep[e]) mk |= 1ull << e;
    s_keepmask = mk;
  }
  __syncthreads();
  SEL_TS(3);

  // 2) remap (policy.py:171-210) or identity (policy.py:215-229), same thread
  if (active) {
    double slot_p[LYNX_MAX_TOPK];
    int asg[LYNX_MAX_TOPK];
    // slot loops unrolled over LYNX_MAX_TOPK: the per-slot arrays stay in
    // registers (a rolled loop with a run-time slot index puts them on the stack)
    if (run_policy) {
      const uint64_t keep = s_keepmask;
      uint64_t occupied = 0;
#pragma unroll
      for (int r = 0; r < LYNX_MAX_TOPK; ++r)
        if (r < k && ((keep >> ids[r]) & 1ull)) occupied |= 1ull << ids[r];
#pragma unroll
      for (int r = 0; r < LYNX_MAX_TOPK; ++r) {
        if (r >= k) break;
        int e = ids[r];
        if (!((keep >> e) & 1ull)) {
          int pick = reg_best<NT>(p, keep & ~occupied);
          if (pick < 0) pick = reg_best<NT>(p, keep);  // collapse (policy.py:197-200)
          e = pick;
          occupied |= 1ull << e;
        }
        asg[r] = e;
        slot_p[r] = reg_at<NT>(p, e);
      }
    } else {
#pragma unroll
      for (int r = 0; r < LYNX_MAX_TOPK; ++r) {
        asg[r] = r < k ? ids[r] : 0;
        slot_p[r] = r < k ? probs[r] : 0.0;
      }
    }
    const double total = reg_pairwise_sum<LYNX_MAX_TOPK>(slot_p, k);
    if (run_policy && !(total > 0.0)) atomicOr(&s_flags, LYNX_FLAG_ZERO_MASS);
#pragma unroll
    for (int r = 0; r < LYNX_MAX_TOPK; ++r) {
      if (r >= k) break;
      const double w = slot_p[r] / total;  // policy.py:208, 220
      ASG[t * k + r] = asg[r];
      WT[t * k + r] = w;
      a.assigned[t * k + r] = asg[r];
      a.weights[t * k + r] = w;
    }
    a.conf[t] = CONF[t];
    if (a.important) a.important[t] = accuracy ? IMP[t] : 0;
  }
  if (t < N) {
    if (a.retained) a.retained[t] = static_cast<uint8_t>(s_keep[t]);
    if (a.counts) a.counts[t] = s_counts[t];
  }
  __syncthreads();
  if (t == 0) a.flags[0] = s_flags | (s_clipped ? LYNX_FLAG_CLIPPED : 0);
  SEL_TS(4);
  SEL_TS(5);
  if (a.plan.enabled)
    plan_dispatch(ASG, WT, T, N, k, a.plan, reinterpret_cast<uint32_t*>(s_dyn + L.bits),
                  reinterpret_cast<int*>(s_dyn + L.prefix));
  SEL_TS(6);
}

// --------------------------------------- K1 group path (16 < N <= 64)
// Eight lanes per token, four tokens per warp, 128 tokens per pass of the
// CTA.  Lane j of a group holds experts j, j+8, j+16, ... (EPL of them), so
// numpy's pairwise row sum maps exactly onto the group: lane j runs numpy's
// j-th strided partial in register, and three xor-shuffles fold
// ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) -- IEEE addition is commutative, so
// every lane's fold is the same bits as numpy's.  Arg-max rounds (top-k,
// remap picks) are an in-lane scan plus three shuffles.
constexpr int kGroup = 8;

// value of element e (lane e%8, slot e/8) of a group row, on every lane
template <int EPL>
__device__ __forceinline__ double grp_at(const double (&v)[EPL], int e, int gbase) {
  double mine = 0.0;
#pragma unroll
  for (int m = 0; m < EPL; ++m)
    if (m == (e >> 3)) mine = v[m];
  return __shfl_sync(kFull, mine, gbase + (e & 7));
}

// numpy pairwise sum of the first n (<= 128) elements of a group row
template <int EPL>
__device__ __forceinline__ double grp_pairwise(const double (&v)[EPL], int n, int j, int gbase) {
  if (n < 8) {
    double acc = 0.0;
#pragma unroll 1
    for (int i = 0; i < n; ++i) acc += __shfl_sync(kFull, v[0], gbase + i);
    return acc;
  }
  const int body = n - (n & 7);
  double r = v[0];
#pragma unroll
  for (int m = 1; m < EPL; ++m)
    if (8 * m < body) r += v[m];
  r += __shfl_xor_sync(kFull, r, 1);
  r += __shfl_xor_sync(kFull, r, 2);
  r += __shfl_xor_sync(kFull, r, 4);
#pragma unroll 1
  for (int i = body; i < n; ++i) r += grp_at<EPL>(v, i, gbase);
  (void)j;
  return r;
}

// Lane-local candidate masks: bit m of lane j's mask <-> expert j + 8m.
template <int EPL>
__device__ __forceinline__ uint32_t lane_bits(uint64_t mask, int j) {
  // the low bit of every byte of mask >> j, packed by one multiply
  const uint64_t x = (mask >> j) & 0x0101010101010101ull;
  return static_cast<uint32_t>((x * 0x0102040810204080ull) >> 56) & ((1u << EPL) - 1u);
}

__device__ __forceinline__ void lane_mark(uint32_t& l, int e, int j) {
  if ((e & 7) == j) l |= 1u << (e >> 3);
}

// best expert among the lane-local candidates by (value desc, index asc); -1
// if none.  In-lane: a depth-log2(EPL) tree over adjacent ranges (the lower
// slot of a pair covers the lower ids, so strict > keeps ties on the smaller
// id); across the group:
// three xor-shuffles.  "None" is (-1.0, 64): probabilities are >= 0.
template <int EPL>
__device__ __forceinline__ int grp_best(const double (&v)[EPL], uint32_t cand, int j, double* bv) {
  double bvv[EPL];
  int bm[EPL];
#pragma unroll
  for (int m = 0; m < EPL; ++m) {
    const bool c = (cand >> m) & 1u;
    bvv[m] = c ? v[m] : -1.0;
    bm[m] = c ? j + 8 * m : 64;
  }
#pragma unroll
  for (int st = 1; st < EPL; st <<= 1)  // adjacent ranges: slot m always holds the lower ids
#pragma unroll
    for (int m = 0; m + st < EPL; m += 2 * st)
      if (bvv[m + st] > bvv[m]) {
        bvv[m] = bvv[m + st];
        bm[m] = bm[m + st];
      }
  double best = bvv[0];
  int bi = bm[0];
#pragma unroll
  for (int off = 1; off < kGroup; off <<= 1) {
    const double ov = __shfl_xor_sync(kFull, best, off);
    const int oi = __shfl_xor_sync(kFull, bi, off);
    if (ov > best || (ov == best && oi < bi)) {
      best = ov;
      bi = oi;
    }
  }
  *bv = best;
  return bi == 64 ? -1 : bi;
}

// remap_tokens for one token row (policy.py:171-210) on the group layout,
// over the COMPACT retained list: candidate c (lane c % 8, slot c / 8) is
// the c-th retained expert ascending, so (p desc, c asc) is the reference's
// (p desc, expert asc) and the arg-max scans EPR = ceil(|R| / 8) values per
// lane instead of one per expert.  Displaced slots take the best retained,
// unoccupied expert, else collapse onto the best retained one.  Writes the
// assignment and the slot probability (renormalised by the caller).
template <int EPR>
__device__ __forceinline__ void remap_row(const double* prow, bool live, int t, int k, int j, uint64_t keep, int nR,
                                          const int* rlist, const int32_t* IDS, int32_t* ASG, double* WT) {
  double v[EPR];
#pragma unroll
  for (int q = 0; q < EPR; ++q) {
    const int c = j + 8 * q;
    v[q] = (live && c < nR) ? prow[rlist[c]] : 0.0;
  }
  const uint32_t all_c = lane_bits<EPR>(nR >= 64 ? ~0ull : ((1ull << nR) - 1ull), j);
  // Retained originals keep their slot and are occupied up front; the
  // displaced slots, in slot order, take the best unoccupied retained experts
  // in (p desc, c asc) order -- so one arg-max round per displaced slot of
  // the warp's neediest token, not one per slot -- or collapse onto the best
  // retained expert when none is left.
  // slot r's original expert and full_probs[t, e] (policy.py:206-208) on
  // lane r: the row's k loads from `full` (global when K0 routed) issue in
  // one round instead of one dependent round trip per slot
  if (live)
    for (int r = j; r < k; r += 8) {
      const int e = IDS[t * k + r];
      ASG[t * k + r] = e;
      WT[t * k + r] = prow[e];
    }
  SEL_TS_LOCAL(21);
  uint32_t occ = 0, dmask = 0;  // occ: lane-local compact bits; dmask: displaced slots
#pragma unroll 1
  for (int r = 0; r < k; ++r) {
    const int e = live ? IDS[t * k + r] : 0;
    if ((keep >> e) & 1ull)
      lane_mark(occ, __popcll(keep & ((1ull << e) - 1ull)), j);
    else
      dmask |= 1u << r;
  }
  __syncwarp();  // the displaced slots' picks below overwrite lane r's stores
  SEL_TS_LOCAL(24);
  const int d = live ? __popc(dmask) : 0;
  const int rounds = __reduce_max_sync(kFull, static_cast<unsigned>(d));  // warp-uniform: shuffles stay converged
  SEL_TS_LOCAL(25);
#pragma unroll 1
  for (int i = 0; i < rounds; ++i) {
    double bv;
    int pick = grp_best<EPR>(v, all_c & ~occ, j, &bv);
    if (__any_sync(kFull, pick < 0)) {
      double bv_any;
      const int any = grp_best<EPR>(v, all_c, j, &bv_any);  // collapse (policy.py:197-200)
      if (pick < 0) {
        pick = any;
        bv = bv_any;
      }
    }
    if (i < d) {
      if (pick >= 0) lane_mark(occ, pick, j);
      const int r = __ffs(dmask) - 1;
      dmask &= dmask - 1;
      if (j == 0) {
        ASG[t * k + r] = pick >= 0 ? rlist[pick] : -1;
        WT[t * k + r] = bv;
      }
    }
  }
}

// kGiven: the selection (ids/probs/full) is an input (a.logits == null; the
// N > 16 layer path, routed in K0): the softmax / top-k code is compiled
// out, so the cold kernel's instruction stream runs straight through.
template <int EPL, bool kGiven>
__global__ void __launch_bounds__(kSelectThreads) route_select_group(const __grid_constant__ SelectArgs a) {
  __shared__ double s_counts[LYNX_MAX_EXPERTS];
  __shared__ int s_icount[LYNX_MAX_EXPERTS];
  __shared__ int s_rank[LYNX_MAX_EXPERTS];
  __shared__ int s_order[LYNX_MAX_EXPERTS];
  __shared__ int s_keep[LYNX_MAX_EXPERTS];
  __shared__ int s_flags, s_nq, s_clipped;
  __shared__ unsigned long long s_keepmask;
  __shared__ int s_rlist[LYNX_MAX_EXPERTS];  // retained experts ascending
  __shared__ double s_exp[32];
  extern __shared__ __align__(16) uint8_t s_dyn[];

  griddep_launch_dependents();
  if (!kGiven) np_exp_stage(s_exp);
  const int T = a.T, N = a.N, k = a.k;
  const int tid = threadIdx.x, nthr = blockDim.x;
  const int j = tid & 7, gbase = tid & 24, grp = tid >> 3, ngrp = nthr >> 3;
  const SelectSmem L = select_smem(T, N, k, a.stage, a.plan.enabled);
  double* P = a.stage ? reinterpret_cast<double*>(s_dyn + L.p) : a.full;
  double* CONF = a.stage ? reinterpret_cast<double*>(s_dyn + L.conf) : a.conf;
  int32_t* IDS = a.stage ? reinterpret_cast<int32_t*>(s_dyn + L.ids) : a.ids;
  double* PROBS = a.stage ? reinterpret_cast<double*>(s_dyn + L.probs) : a.probs;
  int32_t* ASG = a.stage ? reinterpret_cast<int32_t*>(s_dyn + L.asg) : a.assigned;
  double* WT = a.stage ? reinterpret_cast<double*>(s_dyn + L.w) : a.weights;
  uint8_t* IMP = s_dyn + L.imp;
  const uint32_t all_l = lane_bits<EPL>(expert_mask_all(N), j);
  if (tid == 0) {
    s_flags = 0;
    s_nq = 0;
    s_clipped = 0;
  }
  if (tid < N) s_icount[tid] = 0;
  warm_params(a);
  __syncthreads();  // s_exp
  SEL_TS(0);
  griddep_wait();  // logits come from K0 (programmatic dependent launch)
  if (a.ep.enabled) {  // peer-memory EP: every rank's logits rows have landed
    if (threadIdx.x == 0) wait_peers(a.ep.P, a.ep.kind, *a.ep.P.epoch + 1);
    __syncthreads();
  }
  SEL_TS(1);

  // 1) softmax + stable top-k + confidence, eight lanes per token.  Passes
  // run whole warps (T rounded up to 4 tokens per warp) so shuffles converge.
  const int Tw = (T + 3) & ~3;
#pragma unroll 1
  for (int t = grp; t < Tw; t += ngrp) {
    const bool live = t < T;
    double v[EPL];
    if (!kGiven) {
      const double* z = a.logits + static_cast<size_t>(t) * N;
      bool bad = false;
      double m = -INFINITY;
#pragma unroll
      for (int q = 0; q < EPL; ++q) {
        const int e = j + 8 * q;
        v[q] = e < N ? (live ? z[e] : 0.0) : -INFINITY;  // padding tokens route zeros
        if (live && e < N) bad |= !isfinite(v[q]);
        m = v[q] > m ? v[q] : m;
      }
      m = fmax(m, __shfl_xor_sync(kFull, m, 1));
      m = fmax(m, __shfl_xor_sync(kFull, m, 2));
      m = fmax(m, __shfl_xor_sync(kFull, m, 4));
      SEL_TS_LOCAL(8);
      if (bad) atomicOr(&s_flags, LYNX_FLAG_NONFINITE);
#pragma unroll
      for (int q = 0; q < EPL; ++q) v[q] = (j + 8 * q < N) ? np_exp(v[q] - m, s_exp) : 0.0;
      SEL_TS_LOCAL(9);
      const double sum = grp_pairwise<EPL>(v, N, j, gbase);
      SEL_TS_LOCAL(10);
#pragma unroll
      for (int q = 0; q < EPL; ++q) v[q] = v[q] / sum;  // e / s, as numpy divides
      SEL_TS_LOCAL(11);
      if (live) {
#pragma unroll
        for (int q = 0; q < EPL; ++q)
          if (j + 8 * q < N) {
            P[static_cast<size_t>(t) * N + j + 8 * q] = v[q];
            if (a.stage) a.full[static_cast<size_t>(t) * N + j + 8 * q] = v[q];
          }
      }
      SEL_TS_LOCAL(12);
      uint32_t taken = ~all_l;
#pragma unroll 1
      for (int r = 0; r < k; ++r) {
        double bv;
        const int b = grp_best<EPL>(v, ~taken, j, &bv);
        lane_mark(taken, b, j);
        if (live && j == 0) {
          IDS[t * k + r] = b;
          PROBS[t * k + r] = bv;
          if (a.stage) {
            a.ids[t * k + r] = b;
            a.probs[t * k + r] = bv;
          }
        }
      }
    } else {  // apply_policy on a given selection
      if (live && j < k) {
        IDS[t * k + j] = a.ids[t * k + j];
        PROBS[t * k + j] = a.probs[t * k + j];
      }
      // A selection K0 routed itself (a.routed_top) has probs[:, 0] = the row
      // max and probs[:, 1] = the second largest, bit for bit, so the
      // confidence (router.py:125-138) follows from it: top1 = the first
      // pick, margin = first - second pick.  The probability row is then never
      // staged: the remap reads its retained entries straight from `full`.
      // A row routed from non-finite logits arrives with NaN probabilities.
      // Any other given selection (lynx_apply_policy: e.g. a deny-rank
      // intervention, simulator.py:183-213) scores the full row below.
      if (a.routed_top && (a.pol.confidence_metric != LYNX_CONF_MARGIN || k >= 2)) {
        if (live && j == 0) {
          const double p0 = a.probs[t * k], p1 = k > 1 ? a.probs[t * k + 1] : 0.0;
          if (isnan(p0)) atomicOr(&s_flags, LYNX_FLAG_NONFINITE);
          CONF[t] = a.pol.confidence_metric == LYNX_CONF_MARGIN ? p0 - p1 : p0;
        }
        continue;
      }
#pragma unroll
      for (int q = 0; q < EPL; ++q) {
        const int e = j + 8 * q;
        v[q] = (live && e < N) ? a.full[static_cast<size_t>(t) * N + e] : 0.0;
        if (live && e < N) P[static_cast<size_t>(t) * N + e] = v[q];
        // a row routed from non-finite logits arrives as NaN (router_route_kernel)
        if (live && e < N && isnan(v[q])) atomicOr(&s_flags, LYNX_FLAG_NONFINITE);
      }
    }
    SEL_TS_LOCAL(13);
    double top1;
    const int first = grp_best<EPL>(v, all_l, j, &top1);
    double c = top1;
    if (a.pol.confidence_metric == LYNX_CONF_MARGIN) {
      if (N == 1) {
        c = grp_at<EPL>(v, 0, gbase);
      } else {
        double second;
        uint32_t rest = all_l;
        if ((first & 7) == j) rest &= ~(1u << (first >> 3));
        grp_best<EPL>(v, rest, j, &second);
        c = top1 - second;
      }
    }
    if (live && j == 0) CONF[t] = c;
  }
  __syncthreads();
  SEL_TS(2);

  const bool run_policy = a.decode && a.pol.mode != LYNX_POLICY_NONE;
  const bool accuracy = run_policy && a.pol.mode == LYNX_POLICY_ACCURACY;
  if (!run_policy) {
    for (int e = tid; e < N; e += nthr) {
      s_keep[e] = 1;
      s_counts[e] = 0.0;
    }
    for (int t = tid; t < T; t += nthr) IMP[t] = 0;
  } else {
    batch_policy(a, IDS, CONF, IMP, s_keep, s_counts, s_icount, s_rank, s_order, &s_nq, &s_clipped);
  }
  __syncthreads();
  if (tid < 32) {  // retained bitmask: one ballot per 32 experts
    const unsigned lo = __ballot_sync(kFull, tid < N && s_keep[tid]);
    const unsigned hi = __ballot_sync(kFull, tid + 32 < N && s_keep[tid + 32]);
    const unsigned long long km = (static_cast<unsigned long long>(hi) << 32) | lo;
    if (tid == 0) s_keepmask = km;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int e = tid + 32 * h;
      if ((km >> e) & 1ull) s_rlist[__popcll(km & ((1ull << e) - 1ull))] = e;
    }
  }
  __syncthreads();
  SEL_TS(3);

  // 2) remap onto the retained set (policy.py:171-210), or the identity
  // mask with weights = probs / row sum (policy.py:215-229)
  const uint64_t keep = s_keepmask;
  const int nR = __popcll(keep);
  SEL_TS_LOCAL(20);
#pragma unroll 1
  for (int t = grp; t < Tw; t += ngrp) {
    const bool live = t < T;
    if (run_policy) {
      // rolled slot loop (one inlined arg-max): the kernel runs from a cold
      // instruction cache once per layer, so code size is latency.  Slot
      // probabilities park in WT until the row's renormalisation.
      const double* prow = (kGiven ? a.full : P) + static_cast<size_t>(t) * N;
      if (EPL > 4 && nR <= 32)
        remap_row<(EPL > 4 ? 4 : EPL)>(prow, live, t, k, j, keep, nR, s_rlist, IDS, ASG, WT);
      else
        remap_row<EPL>(prow, live, t, k, j, keep, nR, s_rlist, IDS, ASG, WT);
      SEL_TS_LOCAL(22);
    } else if (live && j == 0) {
#pragma unroll 1
      for (int r = 0; r < k; ++r) {
        ASG[t * k + r] = IDS[t * k + r];
        WT[t * k + r] = PROBS[t * k + r];
      }
    }
    __syncwarp();
    SEL_TS_LOCAL(23);
    // row sum on lane 0 (numpy's pairwise order), then lane r divides slot r
    double total = 0.0;
    if (live && j == 0) {
      double slot[LYNX_MAX_TOPK];
#pragma unroll
      for (int r = 0; r < LYNX_MAX_TOPK; ++r) slot[r] = r < k ? WT[t * k + r] : 0.0;
      total = reg_pairwise_sum<LYNX_MAX_TOPK>(slot, k);
      if (run_policy && !(total > 0.0)) atomicOr(&s_flags, LYNX_FLAG_ZERO_MASS);
    }
    total = __shfl_sync(kFull, total, gbase);
    if (live && j < k) WT[t * k + j] = WT[t * k + j] / total;
  }
  __syncthreads();
  SEL_TS(4);

  // 3) outputs
  if (a.stage) {
    for (int t = tid; t < T; t += nthr) a.conf[t] = CONF[t];
    for (int i = tid; i < T * k; i += nthr) {
      a.assigned[i] = ASG[i];
      a.weights[i] = WT[i];
    }
  }
  for (int e = tid; e < N; e += nthr) {
    if (a.retained) a.retained[e] = static_cast<uint8_t>(s_keep[e]);
    if (a.counts) a.counts[e] = s_counts[e];
  }
  if (a.important)
    for (int t = tid; t < T; t += nthr) a.important[t] = accuracy ? IMP[t] : 0;
  if (tid == 0) a.flags[0] = s_flags | (s_clipped ? LYNX_FLAG_CLIPPED : 0);
  SEL_TS(5);
  if (a.plan.enabled)
    plan_dispatch(ASG, WT, T, N, k, a.plan, reinterpret_cast<uint32_t*>(s_dyn + L.bits),
                  reinterpret_cast<int*>(s_dyn + L.prefix));
  SEL_TS(6);
}

// Dispatch plan from an assigned/weights mask in global memory (forward_layer path).
__global__ void __launch_bounds__(kSelectThreads) plan_kernel(const int32_t* asg, const double* w, int T, int N,
                                                              int k, const __grid_constant__ PlanOut o) {
  extern __shared__ __align__(16) uint8_t s_dyn[];
  griddep_launch_dependents();
  griddep_wait();
  const int W = (T + 31) >> 5;
  plan_dispatch(asg, w, T, N, k, o, reinterpret_cast<uint32_t*>(s_dyn),
                reinterpret_cast<int*>(s_dyn + sizeof(uint32_t) * N * W));
}

// remap_tokens on a caller-supplied retained mask; one warp per token.
__global__ void remap_kernel(const int32_t* ids, const double* full, int T, int N, int k, const uint8_t* retained,
                             int32_t* assigned, double* weights, int32_t* flags) {
  __shared__ unsigned long long s_keep;
  __shared__ int s_flags;
  if (threadIdx.x == 0) {
    unsigned long long m = 0;
    for (int e = 0; e < N; ++e)
      if (retained[e]) m |= 1ull << e;
    s_keep = m;
    s_flags = 0;
  }
  __syncthreads();
  const int warps = blockDim.x >> 5;
  for (int t = blockIdx.x * warps + (threadIdx.x >> 5); t < T; t += gridDim.x * warps)
    remap_token(ids + t * k, full + static_cast<size_t>(t) * N, k, N, s_keep, assigned + t * k, weights + t * k,
                &s_flags);
  __syncthreads();
  if (threadIdx.x == 0 && s_flags) atomicOr(flags, s_flags);
}

// top_k_select (router.py:157-171) over float64 rows: (value desc, index asc).
__global__ void topk_kernel(const double* vals, int T, int N, int k, int32_t* ids, double* out) {
  const int warps = blockDim.x >> 5, lane = threadIdx.x & 31;
  for (int t = blockIdx.x * warps + (threadIdx.x >> 5); t < T; t += gridDim.x * warps) {
    const double* p = vals + static_cast<size_t>(t) * N;
    const double v0 = lane < N ? p[lane] : 0.0, v1 = lane + 32 < N ? p[lane + 32] : 0.0;
    uint64_t taken = 0;
    for (int r = 0; r < k; ++r) {
      double bv;
      const int b = warp_best(v0, v1, expert_mask_all(N) & ~taken, &bv);
      taken |= 1ull << b;
      if (lane == 0) {
        ids[t * k + r] = b;
        out[t * k + r] = bv;
      }
    }
  }
}

// vote_expert_frequencies (policy.py:116-138): slots in row-major order.
__global__ void vote_kernel(const int32_t* ids, int T, int k, int N, lynx_policy_t w, double* counts) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= N) return;
  double c = 0.0;
  for (int t = 0; t < T; ++t)
    for (int r = 0; r < k; ++r)
      if (ids[t * k + r] == e) c += w.n_rank_weights ? w.rank_weights[r] : 1.0;
  counts[e] = c;
}

// ------------------------------------------------------------------- K0
// logits[t, n] = (h_t . Wr_n) / sqrt(mean(h_t^2) + 1e-12).  One CTA per
// (token, group of 8 experts); every thread issues its 1 + 8 independent
// 16-byte loads before any math, so an iteration costs one memory latency.
// The 8 logits of experts n0..n0+7 for token row h (RMSNorm fused: dots and
// the row's sum of squares in one pass, f64 result dot / sqrt(ss / d + eps)).
// 256 threads; result valid in threads 0..7 (z), all threads return.
__device__ __forceinline__ double router_dots8(const uint16_t* __restrict__ hidden, const uint16_t* __restrict__ wt,
                                               int t, int d, int N, int n0) {
  const __nv_bfloat16* h = reinterpret_cast<const __nv_bfloat16*>(hidden) + static_cast<size_t>(t) * d;
  const __nv_bfloat16* w = reinterpret_cast<const __nv_bfloat16*>(wt);
  float acc[8];
#pragma unroll
  for (int n = 0; n < 8; ++n) acc[n] = 0.f;
  float ss = 0.f;
  for (int c = threadIdx.x * 8; c < d; c += blockDim.x * 8) {
    uint4 wv[8];
    const uint4 hv = *reinterpret_cast<const uint4*>(h + c);
#pragma unroll
    for (int n = 0; n < 8; ++n) {
      const int e = min(n0 + n, N - 1);
      wv[n] = __ldg(reinterpret_cast<const uint4*>(w + static_cast<size_t>(e) * d + c));
    }
    const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&hv);
    float hf[8];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float2 f = __bfloat1622float2(h2[j]);
      hf[2 * j] = f.x;
      hf[2 * j + 1] = f.y;
      ss += f.x * f.x + f.y * f.y;
    }
#pragma unroll
    for (int n = 0; n < 8; ++n) {
      const __nv_bfloat162* w2 = reinterpret_cast<const __nv_bfloat162*>(&wv[n]);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 f = __bfloat1622float2(w2[j]);
        acc[n] += hf[2 * j] * f.x + hf[2 * j + 1] * f.y;
      }
    }
  }
  __shared__ float s_red[8][9];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int n = 0; n < 9; ++n) {
    float v = n < 8 ? acc[n] : ss;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
    if (lane == 0) s_red[warp][n] = v;
  }
  __syncthreads();
  if (threadIdx.x < 9) {
    float v = 0.f;
    for (int i = 0; i < 8; ++i) v += s_red[i][threadIdx.x];
    s_red[0][threadIdx.x] = v;
  }
  __syncthreads();
  double z = 0.0;
  if (threadIdx.x < 8) {
    const double inv = 1.0 / sqrt(static_cast<double>(s_red[0][8]) / d + 1e-12);
    z = static_cast<double>(s_red[0][threadIdx.x]) * inv;
  }
  return z;
}

__global__ void __launch_bounds__(256) router_logits_kernel(const uint16_t* __restrict__ hidden,
                                                            const uint16_t* __restrict__ wt, int d, int N,
                                                            double* __restrict__ logits,
                                                            const __grid_constant__ EpLink put) {
  griddep_launch_dependents();
  const int t = blockIdx.x;
  const int n0 = blockIdx.y * 8;
  griddep_wait();  // hidden may be produced by the previous kernel
  const double z = router_dots8(hidden, wt, t, d, N, n0);
  if (threadIdx.x < 8 && n0 + threadIdx.x < N) {
    if (put.enabled) {  // peer-memory EP: this rank's rows straight into every rank's logits buffer
      const size_t o = (static_cast<size_t>(put.P.rank) * put.P.tokens_per_rank + t) * N + n0 + threadIdx.x;
      for (int p = 0; p < put.P.world_size; ++p) put.P.logits[p][o] = z;
    } else {
      logits[static_cast<size_t>(t) * N + n0 + threadIdx.x] = z;
    }
  }
  if (put.enabled && last_cta(put.P.counters + 3)) {
    if (threadIdx.x == 0) signal_peers(put.P, kSigLogits, *put.P.epoch + 1);
  }
}

// router_dots8 for TPC tokens at once (rows t0 .. t0+TPC-1, clamped): every
// weight vector loaded is reused for all TPC tokens, so the CTAs of a routing
// cluster re-read the router TPC times less.  Per token the arithmetic is
// router_dots8's (same per-thread column walk, same reduction order): the
// same bits.  Threads 0..7 return z[q] for expert n0 + tid of token t0 + q.
template <int TPC>
__device__ __forceinline__ void router_dots8_multi(const uint16_t* __restrict__ hidden,
                                                   const uint16_t* __restrict__ wt, int t0, int T, int d, int N,
                                                   int n0, double (&z)[TPC]) {
  const __nv_bfloat16* w = reinterpret_cast<const __nv_bfloat16*>(wt);
  float acc[TPC][8];
  float ss[TPC];
#pragma unroll
  for (int q = 0; q < TPC; ++q) {
    ss[q] = 0.f;
#pragma unroll
    for (int n = 0; n < 8; ++n) acc[q][n] = 0.f;
  }
  for (int c = threadIdx.x * 8; c < d; c += blockDim.x * 8) {
    uint4 wv[8];
    uint4 hv[TPC];
#pragma unroll
    for (int q = 0; q < TPC; ++q) {
      const int t = min(t0 + q, T - 1);
      hv[q] = *reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(hidden) +
                                              static_cast<size_t>(t) * d + c);
    }
#pragma unroll
    for (int n = 0; n < 8; ++n) {
      const int e = min(n0 + n, N - 1);
      wv[n] = __ldg(reinterpret_cast<const uint4*>(w + static_cast<size_t>(e) * d + c));
    }
#pragma unroll
    for (int q = 0; q < TPC; ++q) {
      const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&hv[q]);
      float hf[8];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 f = __bfloat1622float2(h2[j]);
        hf[2 * j] = f.x;
        hf[2 * j + 1] = f.y;
        ss[q] += f.x * f.x + f.y * f.y;
      }
#pragma unroll
      for (int n = 0; n < 8; ++n) {
        const __nv_bfloat162* w2 = reinterpret_cast<const __nv_bfloat162*>(&wv[n]);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float2 f = __bfloat1622float2(w2[j]);
          acc[q][n] += hf[2 * j] * f.x + hf[2 * j + 1] * f.y;
        }
      }
    }
  }
  __shared__ float s_red[8][TPC][9];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < TPC; ++q)
#pragma unroll
    for (int n = 0; n < 9; ++n) {
      float v = n < 8 ? acc[q][n] : ss[q];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
      if (lane == 0) s_red[warp][q][n] = v;
    }
  __syncthreads();
  if (threadIdx.x < 9 * TPC) {
    const int q = threadIdx.x / 9, n = threadIdx.x % 9;
    float v = 0.f;
    for (int i = 0; i < 8; ++i) v += s_red[i][q][n];
    s_red[0][q][n] = v;
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < TPC; ++q) {
    z[q] = 0.0;
    if (threadIdx.x < 8) {
      const double inv = 1.0 / sqrt(static_cast<double>(s_red[0][q][8]) / d + 1e-12);
      z[q] = static_cast<double>(s_red[0][q][threadIdx.x]) * inv;
    }
  }
}

// K0 with the routing folded in (router.py:141-187), for 16 < N <= 64.  A
// cluster of ceil(N/8) CTAs per group of TPC tokens computes their logits
// (8 experts per CTA, router_dots8_multi) into the cluster leader's shared
// memory (DSMEM); after one cluster barrier the leader's warp 0 routes the
// tokens, eight lanes each (the group path's softmax with numpy's pairwise
// sum + stable top-k), four tokens per warp.  The softmax over 64 experts of
// 128 tokens then spreads over many SMs instead of K1's one, and K1 runs on
// the given selection.  Rows with non-finite logits are written as NaN so K1
// raises LYNX_FLAG_NONFINITE.
template <int TPC>
__global__ void __launch_bounds__(256) router_route_kernel(const uint16_t* __restrict__ hidden,
                                                           const uint16_t* __restrict__ wt, int T, int d, int N,
                                                           int k, double* logits, double* full, int32_t* ids,
                                                           double* probs) {
  namespace cg = cooperative_groups;
  static_assert(TPC <= 4, "four tokens per routing warp");
  __shared__ double zs[TPC][LYNX_MAX_EXPERTS];
  __shared__ double s_exp[32];
  cg::cluster_group cluster = cg::this_cluster();
  griddep_launch_dependents();
  // DSMEM rule: the leader must have started before its shared memory is
  // written.  Arrive now, wait just before the remote store, so the
  // barrier's latency hides behind the dot products.
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
  const int t0 = blockIdx.y * TPC, c = static_cast<int>(cluster.block_rank());
  const int n0 = c * 8;
  if (c == 0) np_exp_stage(s_exp);  // read by warp 0 after cluster.sync()
  K0_TS(0);
  griddep_wait();  // hidden may be produced by the previous kernel
  K0_TS(1);
  double z[TPC];
  router_dots8_multi<TPC>(hidden, wt, t0, T, d, N, n0, z);
  K0_TS(2);
  asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
  if (threadIdx.x < 8 && n0 + threadIdx.x < N) {
#pragma unroll
    for (int q = 0; q < TPC; ++q) {
      double* zl = cluster.map_shared_rank(&zs[q][0], 0);
      zl[n0 + threadIdx.x] = z[q];
      if (logits && t0 + q < T) logits[static_cast<size_t>(t0 + q) * N + n0 + threadIdx.x] = z[q];
    }
  }
  cluster.sync();
  K0_TS(3);
  if (c != 0 || threadIdx.x >= 32) return;
  // warp 0 of the leader: group g = lanes 8g..8g+7 routes token t0 + g; the
  // groups past TPC (or past T) shadow on zeros (shuffles stay warp-converged)
  const int j = threadIdx.x & 7, gbase = threadIdx.x & 24, g = threadIdx.x >> 3;
  const int t = t0 + g;
  const bool live = g < TPC && t < T;
  constexpr int EPL = 8;
  double v[EPL];
  bool bad = false;
  double m = -INFINITY;
#pragma unroll
  for (int q = 0; q < EPL; ++q) {
    const int e = j + 8 * q;
    v[q] = e < N ? (live ? zs[g < TPC ? g : 0][e] : 0.0) : -INFINITY;
    if (e < N) bad |= !isfinite(v[q]);
    m = v[q] > m ? v[q] : m;
  }
  m = fmax(m, __shfl_xor_sync(kFull, m, 1));
  m = fmax(m, __shfl_xor_sync(kFull, m, 2));
  m = fmax(m, __shfl_xor_sync(kFull, m, 4));
  const unsigned badg = __ballot_sync(kFull, live && bad);
  bad = (badg >> gbase) & 0xffu;  // any lane of this token's group
#pragma unroll
  for (int q = 0; q < EPL; ++q) v[q] = (j + 8 * q < N) ? np_exp(v[q] - m, s_exp) : 0.0;
  const double sum = grp_pairwise<EPL>(v, N, j, gbase);
#pragma unroll
  for (int q = 0; q < EPL; ++q) v[q] = v[q] / sum;  // e / s, as numpy divides
  if (live) {
#pragma unroll
    for (int q = 0; q < EPL; ++q)
      if (j + 8 * q < N) full[static_cast<size_t>(t) * N + j + 8 * q] = bad ? NAN : v[q];
  }
  const uint32_t all_l = lane_bits<EPL>(expert_mask_all(N), j);
  uint32_t taken = ~all_l;
#pragma unroll 1
  for (int r = 0; r < k; ++r) {
    double bv;
    const int b = grp_best<EPL>(v, ~taken, j, &bv);
    lane_mark(taken, b, j);
    if (live && j == 0) {
      ids[t * k + r] = b;
      probs[t * k + r] = bad ? NAN : bv;
    }
  }
  K0_TS(4);
}

// ------------------------------------------- fused front (N <= 8, T <= 256)
// K0 + K1 + K2 of the layer in ONE launch of T CTAs, one token each, with one
// grid-wide barrier.  The chain it replaces is a run of latency-bound steps
// on the critical path before the expert stream can start (router GEMV ->
// single-CTA selection -> gather); here the per-token steps run on T SMs at
// once and only the batch-level decisions are global:
//
//   A  router logits of token t (RMSNorm fused, router_dots8)
//   B  softmax (np_exp, numpy's pairwise sum, e / s) + stable top-k +
//      confidence of token t on warp 0 (lane j = expert j)
//   -- grid barrier (every CTA resident: K3 may now launch beside us) --
//   C  the batch policy, computed by every CTA from all tokens' selections
//      (identical everywhere: integer votes and ranks, the same compares)
//   D  the remap of every token (thread per token), so each CTA holds the
//      whole batch's assignment without a second barrier
//   E  dispatch plan: token t's permuted rows and merged weights, the gather
//      of its hidden row into them; CTA 0 writes the segment tables.
//
// Results are identical to router_logits_kernel + route_select_fast +
// plan_dispatch + gather_kernel (same arithmetic, same order).  The barrier
// words (f.sync) must be zero before the first launch; every launch leaves
// them ready for the next one (grid_barrier).  Co-residency: the T CTAs only
// wait for each other (the next kernel's programmatic launch is released
// after the barrier), and T <= 256 small CTAs always fit the 148 SMs.
struct FrontArgs {
  SelectArgs s;               // selection outputs + plan (s.logits unused)
  const uint16_t* hidden;     // [T, d] bf16
  const uint16_t* router_wt;  // [N, d] bf16
  int d;
  uint16_t* x_perm;           // [rows_cap, d] gathered rows
  int* sync;                  // [4]: arrival counters (even / odd launches), non-finite flag accumulator,
                              //   generation (all zero before the first launch)
  const double* logits_in;    // [T, N] given logits (the decode stack's fused router), or null: phase A
};

#ifdef LYNX_TRACE
__device__ unsigned long long g_front_cta[4 * 256];  // per CTA: entry, after wait, at the barrier, after it
#define FRONT_CTA_TS(i)                                                                       \
  do {                                                                                        \
    if (threadIdx.x == 0 && blockIdx.x < 256) g_front_cta[4 * blockIdx.x + (i)] = globaltimer(); \
  } while (0)
#define FRONT_TS(i)                                                                \
  do {                                                                             \
    if (blockIdx.x == 0 && threadIdx.x == 0) g_sel_ts[24 + (i)] = globaltimer(); \
  } while (0)
#else
#define FRONT_TS(i) (void)0
#define FRONT_CTA_TS(i) (void)0
#endif

// Grid-wide barrier of the fused front (all CTAs resident, see above), on
// two arrival counters used alternately by launch parity (f.sync[0], [1]):
// each CTA arrives with one release reduction -- no returned value to wait
// for -- and polls its counter until every CTA has arrived, so the barrier
// completes one L2 round trip after the last arrival (the last arriver no
// longer resets a count and publishes a generation first: that cost
// 1.6-2.2 us from the last arrival to the first exit).  The launch's
// parity comes from the generation word f.sync[3], read at kernel start
// (the launch that last wrote it has completed); after its wait CTA 0
// zeroes the OTHER counter, which only the previous launch used, and
// after the barrier it advances the generation for the next launch.
__device__ __forceinline__ void red_release_gpu_add_int(int* p, int v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void grid_barrier(int* counter, int nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    red_release_gpu_add_int(counter, 1);
    Watchdog wd;
    while (ld_acquire_gpu(counter) < nblocks) wd.tick(9);
  }
  __syncthreads();
}

template <int NT>
__global__ void __launch_bounds__(256) front_kernel(const __grid_constant__ FrontArgs f) {
  const SelectArgs& a = f.s;
  __shared__ double s_exp[32];
  __shared__ double s_counts[LYNX_MAX_EXPERTS];
  __shared__ int s_icount[LYNX_MAX_EXPERTS];
  __shared__ int s_rank[LYNX_MAX_EXPERTS];
  __shared__ int s_order[LYNX_MAX_EXPERTS];
  __shared__ int s_keep[LYNX_MAX_EXPERTS];
  __shared__ int s_cnt[NT], s_base[NT];
  __shared__ int s_nq, s_clipped;
  __shared__ int s_flags;
  __shared__ uint32_t s_keepmask;
  __shared__ int s_rows[LYNX_MAX_TOPK];
  __shared__ int s_nrows;
  extern __shared__ __align__(16) uint8_t s_dyn[];
  FRONT_CTA_TS(0);
  const int T = a.T, N = a.N, k = a.k, t = blockIdx.x, tid = threadIdx.x;
  const int W = (T + 31) >> 5;
  double* WT = reinterpret_cast<double*>(s_dyn);                            // [T*k] remap weights
  double* CONF = WT + T * k;                                                  // [T]
  int32_t* IDS = reinterpret_cast<int32_t*>(CONF + T);                        // [T*k] top-k ids
  int32_t* ASG = IDS + T * k;                                                 // [T*k] assignments
  uint32_t* BITS = reinterpret_cast<uint32_t*>(ASG + T * k);                  // [N*W]
  uint8_t* IMP = reinterpret_cast<uint8_t*>(BITS + N * W);                    // [T]
  np_exp_stage(s_exp);
  if (tid < LYNX_MAX_EXPERTS) s_icount[tid] = 0;
  if (tid == 0) {
    s_nq = 0;
    s_clipped = 0;
    s_flags = 0;
  }
  warm_params(f);
  // the barrier generation: last written by the previous front on this
  // workspace, which completed before this launch's predecessor started
  __shared__ int s_gen;
  if (tid == 0) s_gen = *reinterpret_cast<volatile int*>(f.sync + 3);
  griddep_wait();  // hidden comes from the previous kernel
  if (t == 0 && tid == 0) f.sync[1 - (s_gen & 1)] = 0;  // the previous launch's counter, for the next one
  FRONT_TS(0);
  FRONT_CTA_TS(1);

  // token t's hidden row -> shared memory (cp.async), for the gather in E
  const int nvec = f.d >> 3;
  uint4* s_row = reinterpret_cast<uint4*>((reinterpret_cast<uintptr_t>(IMP + T) + 15) & ~uintptr_t(15));
  {
    const uint4* src = reinterpret_cast<const uint4*>(f.hidden) + static_cast<size_t>(t) * nvec;
    for (int v4 = tid; v4 < nvec; v4 += blockDim.x)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(s_row + v4)), "l"(src + v4) : "memory");
    asm volatile("cp.async.commit_group;" ::: "memory");
  }

  // A) logits of token t: threads 0..N-1 hold them
  const double z = f.logits_in ? (tid < N ? f.logits_in[static_cast<size_t>(t) * N + tid] : 0.0)
                               : router_dots8(f.hidden, f.router_wt, t, f.d, N, 0);
  FRONT_TS(1);

  // B) softmax + stable top-k + confidence on warp 0, lane j = expert j (the
  // group layout with one expert per lane: numpy's pairwise sum folds the 8
  // lanes as ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)); fewer than 8 add in order)
  const int j = tid & 7, gbase = tid & 24;
  double v = 0.0;
  int ids[LYNX_MAX_TOPK];
  if (tid < 32) {
    const bool mine = tid < 8 && j < N;
    v = mine ? z : (tid < 8 ? -INFINITY : 0.0);  // lanes 8..31 shadow on finite zeros
    const bool bad = __any_sync(kFull, mine && !isfinite(v));
    double m = v;
    m = fmax(m, __shfl_xor_sync(kFull, m, 1));
    m = fmax(m, __shfl_xor_sync(kFull, m, 2));
    m = fmax(m, __shfl_xor_sync(kFull, m, 4));
    double e1[1] = {j < N ? np_exp(v - m, s_exp) : 0.0};
    const double sum = grp_pairwise<1>(e1, N, j, gbase);
    v = e1[0] / sum;  // e / s, as numpy divides (router.py:154)
    if (tid < 8 && j < N) a.full[static_cast<size_t>(t) * N + j] = v;
    const uint32_t all_l = j < N ? 1u : 0u;
    uint32_t taken = ~all_l;
#pragma unroll
    for (int r = 0; r < LYNX_MAX_TOPK; ++r) {
      if (r >= k) break;
      double bv;
      uint32_t cand[1] = {~taken & 1u};
      double vv[1] = {v};
      const int b = __shfl_sync(kFull, grp_best<1>(vv, cand[0], j, &bv), 0);  // group 0's pick on every lane
      if (b == j) taken |= 1u;
      ids[r] = b;  // warp-uniform: the remap below branches on it around shuffles
      if (tid == 0) {
        a.ids[t * k + r] = b;
        a.probs[t * k + r] = bv;
      }
    }
    double vv[1] = {v}, top1, second;
    grp_best<1>(vv, all_l, j, &top1);
    double c = top1;
    if (a.pol.confidence_metric == LYNX_CONF_MARGIN) {
      if (N == 1) {
        c = __shfl_sync(kFull, v, gbase);
      } else {
        const int first = grp_best<1>(vv, all_l, j, &top1);
        grp_best<1>(vv, first == j ? 0u : all_l, j, &second);
        c = top1 - second;
      }
    }
    if (tid == 0) {
      a.conf[t] = c;
      if (bad) atomicOr(f.sync + 2, LYNX_FLAG_NONFINITE);
    }
  }
  FRONT_TS(2);
  FRONT_CTA_TS(2);
  grid_barrier(f.sync + (s_gen & 1), T);  // (s_gen: written before the first __syncthreads of the barrier)
  FRONT_CTA_TS(3);
  griddep_launch_dependents();  // every CTA is resident: the expert FFN may launch now
  FRONT_TS(3);

  if (t == 0 && tid == 0) {
    s_flags = f.sync[2];  // every CTA's non-finite report precedes barrier 1
    f.sync[2] = 0;
    f.sync[3] = s_gen + 1;  // the next launch's parity
  }

  // the probability rows of this thread's tokens (remap, D), issued before
  // the policy so the loads overlap it (T <= 256 = blockDim: one per thread)
  double pr[NT];
#pragma unroll
  for (int i = 0; i < NT; ++i) pr[i] = (tid < T && i < N) ? a.full[static_cast<size_t>(tid) * N + i] : 0.0;

  // C) batch policy (every CTA, identical)
  const bool run_policy = a.decode && a.pol.mode != LYNX_POLICY_NONE;
  const bool accuracy = run_policy && a.pol.mode == LYNX_POLICY_ACCURACY;
  if (run_policy && !accuracy && a.pol.n_rank_weights == 0) {
    // latency_policy with unit votes on warp 0 (policy.py:116-148, 232-264):
    // the ids are staged by the whole CTA in one load round and counted --
    // by ballots on warp 0 for up to 256 slots, by shared-memory atomics of
    // the whole CTA beyond -- then lane e ranks expert e by (count desc,
    // index asc) against the others, the first N - eff are kept.  Integer
    // arithmetic: the same decisions as batch_policy.
    const bool by_atomics = T * k > 256;
    for (int i = tid; i < T * k; i += blockDim.x) {
      const int id = a.ids[i];
      IDS[i] = id;
      if (by_atomics && id >= 0 && id < N) atomicAdd(&s_icount[id], 1);
    }
    __syncthreads();
    if (tid < 32) {
      int cnt = by_atomics && tid < N ? s_icount[tid] : 0;
      for (int i0 = 0; i0 < (by_atomics ? 0 : T * k); i0 += 32) {
        const int i = i0 + tid;
        const int id = i < T * k ? IDS[i] : -1;
        for (int e = 0; e < N; ++e) {
          const unsigned m = __ballot_sync(kFull, id == e);
          if (tid == e) cnt += __popc(m);
        }
      }
      int rank = 0;
      for (int f = 0; f < N; ++f) {
        const int cf = __shfl_sync(kFull, cnt, f);
        rank += (cf > cnt || (cf == cnt && f < tid)) ? 1 : 0;
      }
      const int room = N - a.floor_keep > 0 ? N - a.floor_keep : 0;
      const int eff = a.pol.drop_count < room ? a.pol.drop_count : room;
      const bool kept = tid < N && rank < N - eff;
      const unsigned km = __ballot_sync(kFull, kept);
      if (tid < N) {
        s_keep[tid] = kept ? 1 : 0;
        s_counts[tid] = static_cast<double>(cnt);
      }
      if (tid == 0) {
        s_keepmask = km;
        s_clipped = eff != a.pol.drop_count;
      }
    }
    __syncthreads();
  } else {
    for (int i = tid; i < T * k; i += blockDim.x) IDS[i] = a.ids[i];
    if (accuracy)
      for (int i = tid; i < T; i += blockDim.x) CONF[i] = a.conf[i];
    __syncthreads();
    if (run_policy) {
      batch_policy(a, IDS, CONF, IMP, s_keep, s_counts, s_icount, s_rank, s_order, &s_nq, &s_clipped);
    } else if (tid < N) {
      s_keep[tid] = 1;
      s_counts[tid] = 0.0;
    }
    __syncthreads();
    if (tid == 0) {
      uint32_t keep = 0;
      for (int e = 0; e < N; ++e)
        if (s_keep[e]) keep |= 1u << e;
      s_keepmask = keep;
    }
    __syncthreads();
  }

  // D) remap of EVERY token (policy.py:171-210), or the identity mask
  // (policy.py:215-229), thread per token with its probability row in
  // registers: each CTA then plans the dispatch on its own, with no second
  // barrier.  The same arithmetic as route_select_fast.
  const uint32_t keep = s_keepmask;
  if (tid < T) {
    const int u = tid;
    double slot_p[LYNX_MAX_TOPK];
    int asg[LYNX_MAX_TOPK];
    uint64_t occupied = 0;
#pragma unroll
    for (int r = 0; r < LYNX_MAX_TOPK; ++r)
      if (r < k && ((keep >> IDS[u * k + r]) & 1u)) occupied |= 1ull << IDS[u * k + r];
#pragma unroll
    for (int r = 0; r < LYNX_MAX_TOPK; ++r) {
      if (r >= k) break;
      int e = IDS[u * k + r];
      if (run_policy && !((keep >> e) & 1u)) {
        int pick = reg_best<NT>(pr, keep & ~occupied);
        if (pick < 0) pick = reg_best<NT>(pr, keep);  // collapse (policy.py:197-200)
        e = pick;
        occupied |= 1ull << e;
      }
      asg[r] = e;
      slot_p[r] = reg_at<NT>(pr, e);  // full_probs[u, e] (= probs for the identity mask)
    }
    const double total = reg_pairwise_sum<LYNX_MAX_TOPK>(slot_p, k);
    if (run_policy && !(total > 0.0)) atomicOr(&s_flags, LYNX_FLAG_ZERO_MASS);  // CTA 0's copy is written
#pragma unroll
    for (int r = 0; r < LYNX_MAX_TOPK; ++r) {
      if (r >= k) break;
      ASG[u * k + r] = asg[r];
      WT[u * k + r] = slot_p[r] / total;  // policy.py:208, 220
    }
  }
  __syncthreads();
  if (tid < k) {
    a.assigned[t * k + tid] = ASG[t * k + tid];
    a.weights[t * k + tid] = WT[t * k + tid];
  }
  if (tid == 0 && a.important) a.important[t] = accuracy ? IMP[t] : 0;
  if (t == 0) {
    if (tid < N) {
      if (a.retained) a.retained[tid] = static_cast<uint8_t>(s_keep[tid]);
      if (a.counts) a.counts[tid] = s_counts[tid];
    }
    if (tid == 0) a.flags[0] = s_flags | (s_clipped ? LYNX_FLAG_CLIPPED : 0);
  }
  FRONT_TS(4);

  // E) dispatch plan (simulator.py:104-112 order) + gather of token t's row
  const PlanOut& o = a.plan;
  if (T <= 32) {
    // one warp, lane u = token u: per expert a ballot of the tokens using it
    // gives its count and every token's rank among them; the 16-padded bases
    // accumulate over the experts in order.  No shared bitmap, no barrier.
    if (tid < 32) {
      const int u = tid;
      uint32_t set = 0;
      if (u < T)
        for (int r = 0; r < k; ++r) set |= 1u << ASG[u * k + r];
      int base = 0;
      for (int e = 0; e < N; ++e) {
        const bool uses = (set >> e) & 1u;
        const unsigned m = __ballot_sync(kFull, uses);
        const int cnt = __popc(m);
        if (tid == e) {
          s_cnt[e] = cnt;
          s_base[e] = base;
        }
        if (u == t && uses) {
          const int slot = __popc(set & ((1u << e) - 1u));
          double acc = 0.0;  // merged weight: token t's slots on e in slot order (simulator.py:108-111)
          for (int r = 0; r < k; ++r)
            if (ASG[t * k + r] == e) acc += WT[t * k + r];
          const float wf = static_cast<float>(acc);
          const int r0 = base + __popc(m & ((1u << u) - 1u));
          o.tok_rows[t * k + slot] = r0;
          o.tok_weight[t * k + slot] = wf;
          o.perm_token[r0] = t;
          o.perm_weight[r0] = wf;
          s_rows[slot] = r0;
        }
        base += (cnt + 15) & ~15;
      }
      if (u == t) {
        const int nj = __popc(set);
        s_nrows = nj;
        for (int q = nj; q < k; ++q) {
          o.tok_rows[t * k + q] = -1;
          o.tok_weight[t * k + q] = 0.f;
        }
      }
    }
  } else {
  for (int i = tid; i < N * W; i += blockDim.x) BITS[i] = 0;
  __syncthreads();
  for (int i = tid; i < T * k; i += blockDim.x) {
    const int e = ASG[i];
    if (e >= 0 && e < N) atomicOr(&BITS[e * W + ((i / k) >> 5)], 1u << ((i / k) & 31));
  }
  __syncthreads();
  if (tid < 32) {
    // lane e: expert e's row count, 16-padded base (exclusive scan) and the
    // number of its tokens before t
    int cnt = 0, below = 0;
    if (tid < N) {
      for (int q = 0; q < W; ++q) {
        const uint32_t word = BITS[tid * W + q];
        cnt += __popc(word);
        if (q < (t >> 5)) below += __popc(word);
        else if (q == (t >> 5)) below += __popc(word & ((1u << (t & 31)) - 1u));
      }
    }
    const int pad = (cnt + 15) & ~15;
    int incl = pad;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int y = __shfl_up_sync(kFull, incl, off);
      if (tid >= off) incl += y;
    }
    const int base = incl - pad;
    if (tid < N) {
      s_cnt[tid] = cnt;
      s_base[tid] = base;
    }
    // token t's distinct experts ascending; lane e writes the row of expert e
    // if t uses it, with the merged weight 0 + its slots on e in slot order
    // (simulator.py:108-111)
    uint32_t set = 0;
    for (int r = 0; r < k; ++r) set |= 1u << ASG[t * k + r];
    const bool uses = tid < N && ((set >> tid) & 1u);
    const int slot = __popc(set & ((1u << tid) - 1u));  // position among t's experts
    if (uses) {
      double acc = 0.0;
      for (int r = 0; r < k; ++r)
        if (ASG[t * k + r] == tid) acc += WT[t * k + r];
      const float wf = static_cast<float>(acc);
      const int r0 = base + below;
      o.tok_rows[t * k + slot] = r0;
      o.tok_weight[t * k + slot] = wf;
      o.perm_token[r0] = t;
      o.perm_weight[r0] = wf;
      s_rows[slot] = r0;
    }
    const int nj = __popc(set);
    if (tid == 0) s_nrows = nj;
    if (tid >= nj && tid < k) {
      o.tok_rows[t * k + tid] = -1;
      o.tok_weight[t * k + tid] = 0.f;
    }
  }
  }
  __syncthreads();
  // gather token t's hidden row (staged in shared memory by cp.async at the
  // start) into each of its permuted rows -- K2's work; padding rows are left
  // as they are: K3 masks every store of a padding token
  FRONT_TS(5);
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
  const int nrows = s_nrows;
  for (int vv = tid; vv < nvec; vv += blockDim.x) {
    const uint4 x = s_row[vv];
    for (int q = 0; q < nrows; ++q)
      reinterpret_cast<uint4*>(f.x_perm)[static_cast<size_t>(s_rows[q]) * nvec + vv] = x;
  }
  // experts t, t + T, ...: mark their 16-row padding (perm_token = -1)
  for (int e = t; e < N; e += T) {
    const int c = s_cnt[e];
    for (int r = s_base[e] + c + tid; r < s_base[e] + ((c + 15) & ~15); r += blockDim.x) {
      o.perm_token[r] = -1;
      o.perm_weight[r] = 0.f;
    }
  }
  if (t == 0) {
    // segment tables: one segment per used expert (T <= LYNX_SEG_ROWS), queue
    // order by rows desc then index asc (LPT), scheduler words zeroed
    for (int i = tid; i < o.n_counters; i += blockDim.x) o.counters[i] = 0;
    if (tid < 32) {
      const int c = tid < N ? s_cnt[tid] : 0;
      const unsigned used = __ballot_sync(kFull, c > 0);
      const int seg = __popc(used & ((1u << tid) - 1u));  // segment index of expert tid
      const int nseg = __popc(used);
      if (c > 0) {
        o.seg_expert[seg] = tid;
        o.seg_row[seg] = s_base[tid];
        o.seg_count[seg] = c;
        int rank = 0;  // rows desc, segment index asc
        for (int e2 = 0; e2 < N; ++e2) {
          const int c2 = s_cnt[e2];
          const int seg2 = __popc(used & ((1u << e2) - 1u));
          rank += (c2 > 0 && (c2 > c || (c2 == c && seg2 < seg))) ? 1 : 0;
        }
        if (o.seg_order) o.seg_order[rank] = seg;
      }
      const int widest = __reduce_max_sync(kFull, static_cast<unsigned>(c));
      const int nrows = __reduce_add_sync(kFull, static_cast<unsigned>((c + 15) & ~15));
      if (tid == 0) {
        if (o.max_rows) *o.max_rows = widest;
        *o.n_seg = nseg;
        *o.n_used = nseg;
        *o.n_rows = nrows;
      }
    }
  }
  __syncthreads();
  FRONT_TS(6);
}

size_t front_smem_bytes(int T, int N, int k, int d) {
  const int W = (T + 31) >> 5;
  return sizeof(double) * (static_cast<size_t>(T) * k + T) + 8ull * T * k + 4ull * N * W + T + 16 + 2ull * d + 16;
}

cudaError_t launch_front(const SelectArgs& a, const uint16_t* hidden, const uint16_t* router_wt, int d,
                         uint16_t* x_perm, int* sync, const double* logits_in, cudaStream_t s) {
  FrontArgs f{};
  f.s = a;
  f.hidden = hidden;
  f.router_wt = router_wt;
  f.d = d;
  f.x_perm = x_perm;
  f.sync = sync;
  f.logits_in = logits_in;
  const size_t smem = front_smem_bytes(a.T, a.N, a.k, d);
  if (smem > 48 * 1024) return cudaErrorInvalidValue;
  static int configured = -1;  // static + dynamic shared memory may pass 48 KB: opt in once per device
  int dev = 0;
  cudaGetDevice(&dev);
  if (configured != dev) {
    const cudaError_t e = cudaFuncSetAttribute(reinterpret_cast<const void*>(front_kernel<8>),
                                               cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    if (e != cudaSuccess) return e;
    configured = dev;
  }
  return launch_pdl(front_kernel<8>, dim3(a.T), dim3(256), smem, s, f);
}

// ------------------------------------------------------------- launchers
cudaError_t launch_router_logits(const uint16_t* hidden, const uint16_t* wt, int T, int d, int N, double* logits,
                                 cudaStream_t s, const EpLink* put) {
  EpLink none{};
  return launch_pdl(router_logits_kernel, dim3(T, (N + 7) / 8), dim3(256), 0, s, hidden, wt, d, N, logits,
                    put ? *put : none);
}

cudaError_t launch_router_route(const uint16_t* hidden, const uint16_t* wt, int T, int d, int N, int k,
                                double* logits, double* full, int32_t* ids, double* probs, cudaStream_t s) {
  const int cl = (N + 7) / 8;
  // tokens per cluster: 4 once there are enough tokens to keep the SMs busy
  const int tpc = T >= 64 ? 4 : 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cl, (T + tpc - 1) / tpc);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = cl;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  if (tpc == 4) return cudaLaunchKernelEx(&cfg, router_route_kernel<4>, hidden, wt, T, d, N, k, logits, full, ids, probs);
  return cudaLaunchKernelEx(&cfg, router_route_kernel<1>, hidden, wt, T, d, N, k, logits, full, ids, probs);
}

size_t select_smem_bytes(int T, int N, int k, bool stage, bool plan) {
  return select_smem(T, N, k, stage, plan).total;
}

bool select_can_stage(int T, int N, int k, bool plan) {
  return select_smem(T, N, k, true, plan).total <= kSelectMaxSmem;
}

static cudaError_t allow_big_smem(const void* fn, int& configured_device) {
  int dev = 0;
  cudaGetDevice(&dev);
  if (configured_device == dev) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(kSelectMaxSmem));
  if (e == cudaSuccess) configured_device = dev;
  return e;
}

cudaError_t launch_route_select(const SelectArgs& a, cudaStream_t s) {
  const size_t smem = select_smem_bytes(a.T, a.N, a.k, a.stage, a.plan.enabled);
  if (smem > kSelectMaxSmem) return cudaErrorInvalidValue;
  // Fast path: N <= 16 and one thread per token (the decode case).
  if (a.N <= 16 && a.T <= kSelectThreads && a.stage) {
    const int threads = ((a.T > a.N ? a.T : a.N) + 31) / 32 * 32;
    static int configured8 = -1, configured16 = -1;
    if (a.N <= 8) {
      {  // static + dynamic shared memory may pass 48 KB: opt in (once per device)
        cudaError_t e = allow_big_smem(reinterpret_cast<const void*>(route_select_fast<8>), configured8);
        if (e != cudaSuccess) return e;
      }
      return launch_pdl(route_select_fast<8>, dim3(1), dim3(threads), smem, s, a);
    }
    {
      cudaError_t e = allow_big_smem(reinterpret_cast<const void*>(route_select_fast<16>), configured16);
      if (e != cudaSuccess) return e;
    }
    return launch_pdl(route_select_fast<16>, dim3(1), dim3(threads), smem, s, a);
  }
  // Group path: every other shape (N <= 64, or rows too large to stage),
  // eight lanes per token.
  const bool given = a.logits == nullptr;
  const void* fn;
  static int configured[4] = {-1, -1, -1, -1};
  int* conf;
  if (a.N <= 32) {
    fn = given ? reinterpret_cast<const void*>(route_select_group<4, true>)
               : reinterpret_cast<const void*>(route_select_group<4, false>);
    conf = &configured[given ? 1 : 0];
  } else {
    fn = given ? reinterpret_cast<const void*>(route_select_group<8, true>)
               : reinterpret_cast<const void*>(route_select_group<8, false>);
    conf = &configured[given ? 3 : 2];
  }
  {  // the kernel's static shared memory (policy / plan tables) adds to `smem`
    cudaError_t e = allow_big_smem(fn, *conf);
    if (e != cudaSuccess) return e;
  }
  if (a.N <= 32)
    return given ? launch_pdl(route_select_group<4, true>, dim3(1), dim3(kSelectThreads), smem, s, a)
                 : launch_pdl(route_select_group<4, false>, dim3(1), dim3(kSelectThreads), smem, s, a);
  return given ? launch_pdl(route_select_group<8, true>, dim3(1), dim3(kSelectThreads), smem, s, a)
               : launch_pdl(route_select_group<8, false>, dim3(1), dim3(kSelectThreads), smem, s, a);
}

cudaError_t launch_plan(const int32_t* asg, const double* w, int T, int N, int k, const PlanOut& o, cudaStream_t s) {
  const int W = (T + 31) / 32;
  const size_t smem = static_cast<size_t>(N) * W * 8;
  if (smem > kSelectMaxSmem) return cudaErrorInvalidValue;
  static int configured = -1;
  {
    cudaError_t e = allow_big_smem(reinterpret_cast<const void*>(plan_kernel), configured);
    if (e != cudaSuccess) return e;
  }
  return launch_pdl(plan_kernel, dim3(1), dim3(kSelectThreads), smem, s, asg, w, T, N, k, o);
}

cudaError_t launch_remap(const int32_t* ids, const double* full, int T, int N, int k, const uint8_t* retained,
                         int32_t* assigned, double* weights, int32_t* flags, cudaStream_t s) {
  const int blocks = (T + 7) / 8;
  remap_kernel<<<blocks, 256, 0, s>>>(ids, full, T, N, k, retained, assigned, weights, flags);
  return cudaGetLastError();
}

cudaError_t launch_topk(const double* vals, int T, int N, int k, int32_t* ids, double* out, cudaStream_t s) {
  topk_kernel<<<(T + 7) / 8, 256, 0, s>>>(vals, T, N, k, ids, out);
  return cudaGetLastError();
}

cudaError_t launch_vote(const int32_t* ids, int T, int k, int N, const lynx_policy_t& w, double* counts,
                        cudaStream_t s) {
  vote_kernel<<<1, 64, 0, s>>>(ids, T, k, N, w, counts);
  return cudaGetLastError();
}

}  // namespace lynx

#ifdef LYNX_TRACE
extern "C" int lynx_debug_select_ts(unsigned long long* host) {
  return cudaMemcpyFromSymbol(host, lynx::g_sel_ts, sizeof(lynx::g_sel_ts)) == cudaSuccess ? 32 : -1;
}
extern "C" int lynx_debug_front_cta_ts(unsigned long long* host) {
  return cudaMemcpyFromSymbol(host, lynx::g_front_cta, sizeof(lynx::g_front_cta)) == cudaSuccess ? 1024 : -1;
}
#endif
