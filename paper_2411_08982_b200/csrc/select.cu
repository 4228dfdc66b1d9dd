// select.cu -- K0 router GEMV (+RMSNorm) and K1 fused route + retention
// policy + remap.  Decisions are bit-exact with the reference's float64
// numpy path (see oracle/lynx_oracle.py for the restated algorithm).
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
#include <cuda_bf16.h>
#include <stdint.h>

#include "lynx_internal.cuh"

namespace lynx {

// numpy's pairwise float64 summation (oracle.pairwise_sum): < 8 terms added
// left to right; <= 128 terms with 8 strided partials folded pairwise plus
// the tail; longer runs split at an 8-aligned midpoint.
__device__ double np_pairwise_sum(const double* a, int n) {
  if (n < 8) {
    double acc = 0.0;
    for (int i = 0; i < n; ++i) acc += a[i];
    return acc;
  }
  if (n <= 128) {
    double r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = a[j];
    const int body = n - (n % 8);
    for (int i = 8; i < body; i += 8) {
#pragma unroll
      for (int j = 0; j < 8; ++j) r[j] += a[i + j];
    }
    double acc = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (int i = body; i < n; ++i) acc += a[i];
    return acc;
  }
  int half = n / 2;
  half -= half % 8;
  return np_pairwise_sum(a, half) + np_pairwise_sum(a + half, n - half);
}

// Best expert in `cand` by (probability desc, index asc); -1 if none.
__device__ __forceinline__ int best_of(const double* p, uint64_t cand, int N) {
  int best = -1;
  double bp = 0.0;
  for (int e = 0; e < N; ++e) {
    if ((cand >> e) & 1ull) {
      const double v = p[e];
      if (best < 0 || v > bp) {
        best = e;
        bp = v;
      }
    }
  }
  return best;
}

// remap_tokens for one token (policy.py:171-210).
__device__ __forceinline__ void remap_one(const int32_t* ids, const double* p, int k, int N, uint64_t keep,
                                          int32_t* assigned, double* weights, int* flags) {
  uint64_t occupied = 0;
  for (int r = 0; r < k; ++r) {
    const int e = ids[r];
    if ((keep >> e) & 1ull) occupied |= 1ull << e;
  }
  double slot_p[LYNX_MAX_TOPK];
  for (int r = 0; r < k; ++r) {
    int e = ids[r];
    if (!((keep >> e) & 1ull)) {
      int pick = best_of(p, keep & ~occupied, N);
      if (pick < 0) pick = best_of(p, keep, N);  // collapse (policy.py:197-200)
      e = pick;
      occupied |= 1ull << e;
    }
    assigned[r] = e;
    slot_p[r] = p[e];
  }
  const double total = np_pairwise_sum(slot_p, k);
  if (!(total > 0.0)) atomicOr(flags, LYNX_FLAG_ZERO_MASS);
  for (int r = 0; r < k; ++r) weights[r] = slot_p[r] / total;
}

// ------------------------------------------------------------------- K1
__global__ void __launch_bounds__(kSelectThreads) route_select_kernel(SelectArgs a) {
  __shared__ double s_counts[LYNX_MAX_EXPERTS];
  __shared__ int s_rank[LYNX_MAX_EXPERTS];
  __shared__ int s_order[LYNX_MAX_EXPERTS];
  __shared__ int s_keep[LYNX_MAX_EXPERTS];
  __shared__ int s_flags, s_nq, s_clipped;
  __shared__ unsigned long long s_keepmask;
  extern __shared__ uint8_t s_imp[];  // [T]

  const int T = a.T, N = a.N, k = a.k;
  const int tid = threadIdx.x;
  if (tid == 0) {
    s_flags = 0;
    s_nq = 0;
    s_clipped = 0;
  }
  __syncthreads();

  // 1) softmax + top-k (when routing from logits) + confidence, one thread
  //    per token.  With logits == null the selection (ids/probs/full) is an
  //    input: apply_policy on an existing ExpertSelection.
  for (int t = tid; t < T; t += blockDim.x) {
    double* p = a.full + static_cast<size_t>(t) * N;
    if (a.logits) {
      const double* z = a.logits + static_cast<size_t>(t) * N;
      double m = z[0];
      bool finite = true;
      for (int i = 0; i < N; ++i) {
        const double v = z[i];
        finite &= isfinite(v);
        m = v > m ? v : m;
      }
      if (!finite) atomicOr(&s_flags, LYNX_FLAG_NONFINITE);
      for (int i = 0; i < N; ++i) p[i] = exp(z[i] - m);
      const double s = np_pairwise_sum(p, N);
      for (int i = 0; i < N; ++i) p[i] = p[i] / s;
      uint64_t taken = 0;
      for (int r = 0; r < k; ++r) {
        const int b = best_of(p, ~taken & (N == 64 ? ~0ull : ((1ull << N) - 1)), N);
        taken |= 1ull << b;
        a.ids[t * k + r] = b;
        a.probs[t * k + r] = p[b];
      }
    }
    double top1 = p[0];
    for (int i = 1; i < N; ++i) top1 = p[i] > top1 ? p[i] : top1;
    double c = top1;
    if (a.pol.confidence_metric == LYNX_CONF_MARGIN) {
      if (N == 1) {
        c = p[0];
      } else {
        // np.sort(full)[-1] - np.sort(full)[-2]: the two largest values
        int first = 0;
        for (int i = 1; i < N; ++i)
          if (p[i] > p[first]) first = i;
        double second = -1.0;
        for (int i = 0; i < N; ++i)
          if (i != first && p[i] > second) second = p[i];
        c = top1 - second;
      }
    }
    a.conf[t] = c;
  }
  __syncthreads();

  const bool run_policy = a.decode && a.pol.mode != LYNX_POLICY_NONE;
  if (!run_policy) {
    // full_retain_mask: identity, weights = probs / row sum.
    for (int t = tid; t < T; t += blockDim.x) {
      const double s = np_pairwise_sum(a.probs + t * k, k);
      for (int r = 0; r < k; ++r) {
        a.assigned[t * k + r] = a.ids[t * k + r];
        a.weights[t * k + r] = a.probs[t * k + r] / s;
      }
    }
    for (int e = tid; e < N; e += blockDim.x) {
      if (a.retained) a.retained[e] = 1;
      if (a.counts) a.counts[e] = 0.0;
    }
    for (int t = tid; t < T; t += blockDim.x)
      if (a.important) a.important[t] = 0;
    __syncthreads();
    if (tid == 0) a.flags[0] = s_flags;
    return;
  }

  const bool accuracy = a.pol.mode == LYNX_POLICY_ACCURACY;
  // 2a) important tokens (accuracy) -- select_important_tokens.
  if (accuracy) {
    const double tau = a.pol.confidence_threshold;
    int local = 0;
    for (int t = tid; t < T; t += blockDim.x) {
      const bool q = a.conf[t] >= tau;
      s_imp[t] = q ? 1 : 0;
      local += q;
    }
    if (local) atomicAdd(&s_nq, local);
    __syncthreads();
    const int nq = s_nq;
    const int S = a.pol.sample_threshold;
    if (nq == 0) {
      if (tid == 0) {
        int best = 0;
        for (int t = 1; t < T; ++t)
          if (a.conf[t] > a.conf[best]) best = t;
        s_imp[best] = 1;
      }
    } else if (nq > S) {
      // keep the S most confident qualifying tokens (conf desc, t asc);
      // ranks come from conf alone, so marking drops in bit 1 is race-free.
      for (int t = tid; t < T; t += blockDim.x) {
        if (!s_imp[t]) continue;
        const double ct = a.conf[t];
        int rank = 0;
        for (int u = 0; u < T; ++u) {
          const double cu = a.conf[u];
          if (cu >= tau && (cu > ct || (cu == ct && u < t))) ++rank;
        }
        if (rank >= S) s_imp[t] |= 2;
      }
      __syncthreads();
      for (int t = tid; t < T; t += blockDim.x) s_imp[t] = s_imp[t] == 1;
    }
    __syncthreads();
  }

  // 2b) vote tally (over all tokens, or the important ones), slot order.
  for (int e = tid; e < N; e += blockDim.x) {
    double c = 0.0;
    for (int t = 0; t < T; ++t) {
      if (accuracy && !s_imp[t]) continue;
      for (int r = 0; r < k; ++r)
        if (a.ids[t * k + r] == e) c += a.pol.n_rank_weights ? a.pol.rank_weights[r] : 1.0;
    }
    s_counts[e] = c;
  }
  __syncthreads();
  // 2c) retention order: count desc, index asc.
  for (int e = tid; e < N; e += blockDim.x) {
    const double ce = s_counts[e];
    int rank = 0;
    for (int f = 0; f < N; ++f) {
      const double cf = s_counts[f];
      if (cf > ce || (cf == ce && f < e)) ++rank;
    }
    s_rank[e] = rank;
    s_order[rank] = e;
  }
  __syncthreads();

  const int floor_keep = a.floor_keep;
  if (!accuracy) {
    // latency_policy: drop the `eff` least-voted experts.
    int eff = a.pol.drop_count;
    const int room = N - floor_keep > 0 ? N - floor_keep : 0;
    if (eff > room) eff = room;
    for (int e = tid; e < N; e += blockDim.x) s_keep[e] = s_rank[e] < N - eff;
    if (tid == 0) s_clipped = eff != a.pol.drop_count;
  } else {
    int budget = a.pol.freq_keep_budget < N ? a.pol.freq_keep_budget : N;
    for (int e = tid; e < N; e += blockDim.x) s_keep[e] = (s_counts[e] > 0.0 && s_rank[e] < budget) ? 1 : 0;
    __syncthreads();
    for (int t = tid; t < T; t += blockDim.x)
      if (s_imp[t]) s_keep[a.ids[t * k]] = 1;
    __syncthreads();
    if (tid == 0) {
      int cnt = 0;
      for (int e = 0; e < N; ++e) cnt += s_keep[e];
      int padded = 0;
      for (int pos = 0; pos < N && cnt < floor_keep; ++pos) {
        const int e = s_order[pos];
        if (!s_keep[e]) {
          s_keep[e] = 1;
          ++cnt;
          padded = 1;
        }
      }
      s_clipped = padded;
    }
  }
  __syncthreads();
  if (tid == 0) {
    unsigned long long m = 0;
    for (int e = 0; e < N; ++e)
      if (s_keep[e]) m |= 1ull << e;
    s_keepmask = m;
  }
  __syncthreads();

  // 3) remap every token onto the retained set.
  const uint64_t keep = s_keepmask;
  for (int t = tid; t < T; t += blockDim.x)
    remap_one(a.ids + t * k, a.full + static_cast<size_t>(t) * N, k, N, keep, a.assigned + t * k,
              a.weights + t * k, &s_flags);

  for (int e = tid; e < N; e += blockDim.x) {
    if (a.retained) a.retained[e] = static_cast<uint8_t>(s_keep[e]);
    if (a.counts) a.counts[e] = s_counts[e];
  }
  for (int t = tid; t < T; t += blockDim.x)
    if (a.important) a.important[t] = accuracy ? s_imp[t] : 0;
  __syncthreads();
  if (tid == 0) a.flags[0] = s_flags | (s_clipped ? LYNX_FLAG_CLIPPED : 0);
}

// remap_tokens on a caller-supplied retained mask.
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
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < T; t += gridDim.x * blockDim.x)
    remap_one(ids + t * k, full + static_cast<size_t>(t) * N, k, N, s_keep, assigned + t * k, weights + t * k,
              &s_flags);
  __syncthreads();
  if (threadIdx.x == 0 && s_flags) atomicOr(flags, s_flags);
}

// ------------------------------------------------------------------- K0
// logits[t, n] = (h_t . Wr_n) / sqrt(mean(h_t^2) + 1e-12); one CTA per token,
// 16-byte vector loads of the bf16 row and the [N, d] router weights.
template <int NT>
__global__ void __launch_bounds__(256) router_logits_kernel(const uint16_t* __restrict__ hidden,
                                                            const uint16_t* __restrict__ wt, int d, int N,
                                                            double* __restrict__ logits) {
  const int t = blockIdx.x;
  const __nv_bfloat16* h = reinterpret_cast<const __nv_bfloat16*>(hidden) + static_cast<size_t>(t) * d;
  const __nv_bfloat16* w = reinterpret_cast<const __nv_bfloat16*>(wt);
  float acc[NT];
#pragma unroll
  for (int n = 0; n < NT; ++n) acc[n] = 0.f;
  float ss = 0.f;
  for (int c = threadIdx.x * 8; c < d; c += blockDim.x * 8) {
    const uint4 hv = *reinterpret_cast<const uint4*>(h + c);
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
    for (int n = 0; n < NT; ++n) {
      if (n < N) {
        const uint4 wv = *reinterpret_cast<const uint4*>(w + static_cast<size_t>(n) * d + c);
        const __nv_bfloat162* w2 = reinterpret_cast<const __nv_bfloat162*>(&wv);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float2 f = __bfloat1622float2(w2[j]);
          acc[n] += hf[2 * j] * f.x + hf[2 * j + 1] * f.y;
        }
      }
    }
  }
  __shared__ float s_red[8][NT + 1];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int n = 0; n <= NT; ++n) {
    float v = n < NT ? acc[n] : ss;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) s_red[warp][n] = v;
  }
  __syncthreads();
  if (threadIdx.x <= NT) {
    float v = 0.f;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) v += s_red[i][threadIdx.x];
    s_red[0][threadIdx.x] = v;
  }
  __syncthreads();
  if (threadIdx.x < N) {
    const double inv = 1.0 / sqrt(static_cast<double>(s_red[0][NT]) / d + 1e-12);
    logits[static_cast<size_t>(t) * N + threadIdx.x] = static_cast<double>(s_red[0][threadIdx.x]) * inv;
  }
}

cudaError_t launch_router_logits(const uint16_t* hidden, const uint16_t* wt, int T, int d, int N, double* logits,
                                 cudaStream_t s) {
  if (N <= 8)
    router_logits_kernel<8><<<T, 256, 0, s>>>(hidden, wt, d, N, logits);
  else if (N <= 16)
    router_logits_kernel<16><<<T, 256, 0, s>>>(hidden, wt, d, N, logits);
  else if (N <= 32)
    router_logits_kernel<32><<<T, 256, 0, s>>>(hidden, wt, d, N, logits);
  else
    router_logits_kernel<64><<<T, 256, 0, s>>>(hidden, wt, d, N, logits);
  return cudaGetLastError();
}

cudaError_t launch_route_select(const SelectArgs& a, cudaStream_t s) {
  const size_t smem = static_cast<size_t>(a.T);
  route_select_kernel<<<1, kSelectThreads, smem, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_remap(const int32_t* ids, const double* full, int T, int N, int k, const uint8_t* retained,
                         int32_t* assigned, double* weights, int32_t* flags, cudaStream_t s) {
  const int blocks = (T + 255) / 256;
  remap_kernel<<<blocks, 256, 0, s>>>(ids, full, T, N, k, retained, assigned, weights, flags);
  return cudaGetLastError();
}

}  // namespace lynx

namespace lynx {

// top_k_select (router.py:157-171) over arbitrary float64 rows:
// k largest by (value desc, index asc).
__global__ void topk_kernel(const double* vals, int T, int N, int k, int32_t* ids, double* out) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T) return;
  const double* p = vals + static_cast<size_t>(t) * N;
  uint64_t taken = 0;
  const uint64_t all = N == 64 ? ~0ull : ((1ull << N) - 1);
  for (int r = 0; r < k; ++r) {
    const int b = best_of(p, all & ~taken, N);
    taken |= 1ull << b;
    ids[t * k + r] = b;
    out[t * k + r] = p[b];
  }
}

// vote_expert_frequencies (policy.py:116-138): per expert, slots in
// row-major order; optional per-rank weights.
__global__ void vote_kernel(const int32_t* ids, int T, int k, int N, lynx_policy_t w, double* counts) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= N) return;
  double c = 0.0;
  for (int t = 0; t < T; ++t)
    for (int r = 0; r < k; ++r)
      if (ids[t * k + r] == e) c += w.n_rank_weights ? w.rank_weights[r] : 1.0;
  counts[e] = c;
}

cudaError_t launch_topk(const double* vals, int T, int N, int k, int32_t* ids, double* out, cudaStream_t s) {
  topk_kernel<<<(T + 127) / 128, 128, 0, s>>>(vals, T, N, k, ids, out);
  return cudaGetLastError();
}

cudaError_t launch_vote(const int32_t* ids, int T, int k, int N, const lynx_policy_t& w, double* counts,
                        cudaStream_t s) {
  vote_kernel<<<1, 64, 0, s>>>(ids, T, k, N, w, counts);
  return cudaGetLastError();
}

}  // namespace lynx
