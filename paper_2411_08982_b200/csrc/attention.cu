// attention.cu -- the reference model's single-head attention stand-in with
// its residual, for the decode stack around the MoE layer:
//
//   h_out = h + attention(layer, h)                     simulator.py:333
//   attention: xn = rms_norm(h); q, k, v = xn Wq, xn Wk, xn Wv; append k, v
//   to the layer's cache; causal softmax(q K^T / sqrt(dh)) V; ctx Wo
//                                                       simulator.py:308-326
//
// The cost is tiny next to the expert stream (3*dh + dh rows of d weights
// per layer), so the kernels are latency-shaped: one CTA per token row.
//   A  attn_qkv:  RMSNorm + the 3*dh projections (a warp per token row and
//                 projection) -> q scratch, k/v appended to the cache.
//   B  attn_out:  scores over the visible cache (online softmax over chunks),
//                 ctx, ctx Wo + the residual -> h_out (bf16).
// A chunk of Tn new tokens per sequence (prefill: Tn = P; decode: Tn = 1)
// sits at cache positions pos .. pos+Tn-1; `pos` is read from device memory
// so one captured decode step can be replayed step after step
// (lynx_advance_position bumps it inside the graph).
#include <cooperative_groups.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <stdlib.h>

#include "lynx_internal.cuh"
#include "ptx.cuh"

namespace lynx {

constexpr int kAttnThreads = 256;

// Diagnostic library only (-DLYNX_TRACE): phase timestamps of the decode
// attention kernel (CTA (0, 0)), read back by lynx_debug_attn_ts().
#ifdef LYNX_TRACE
__device__ unsigned long long g_attn_ts[16];
#define ATT_TS(i)                                                                             \
  do {                                                                                        \
    if (kCluster && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) g_attn_ts[i] = globaltimer(); \
  } while (0)
#else
#define ATT_TS(i) (void)0
#endif
constexpr unsigned kAll = 0xffffffffu;

__device__ __forceinline__ float block_sum(float v, float* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kAll, v, o);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  float t = 0.f;
  for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += red[i];
  return t;
}

__device__ __forceinline__ float block_max(float v, float* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(kAll, v, o));
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  float t = -INFINITY;
  for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t = fmaxf(t, red[i]);
  return t;
}

// Latency shaping.  Both kernels are a handful of dependent L2 round trips;
// every load a thread will need is issued before the first use.
//   qkv: a warp per (token row, projection): the lane streams its 1/32 of
//        the row and of the weight row together (16-byte loads, unrolled),
//        so the RMSNorm statistic and the dot product come out of ONE pass
//        with no block barrier: rms_norm(h) . w = (h . w) / rms(h).
//   out: a CTA per (token row, 1024 output columns): the residual columns,
//        the head's Wo columns, q and a chunk of cached K/V are all loaded
//        up front; causal softmax is online over chunks of cached positions
//        (so the cache length is not bounded by shared memory).
constexpr int kQkvPerCta = kAttnThreads / 32;
constexpr int kOutCols = kAttnThreads * 4;
constexpr int kChunkFloats = 4096;  // K (or V) floats per chunk: chunk = 4096 / dh positions
constexpr int kWoPrefetch = 16;     // Wo head rows held in registers from the start
constexpr int kMaxAttnCluster = 8;  // decode kernel: CTAs (1024-column chunks) per row cluster, d <= 8192

// sum of squares of the whole row (the decode step's input normalisation)
__device__ __forceinline__ float row_sumsq(const uint16_t* row, int d, float* red) {
  float ss = 0.f;
  for (int c = threadIdx.x * 8; c < d; c += blockDim.x * 8) {
    const uint4 u = __ldg(reinterpret_cast<const uint4*>(row + c));
    const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float2 f = __bfloat1622float2(h2[j]);
      ss += f.x * f.x + f.y * f.y;
    }
  }
  return block_sum(ss, red);
}

// Output o of the 3*dh q/k/v projections for token row `row`, one warp:
// the lane streams its 1/32 of the row and of the weight row together, so
// the RMSNorm statistic and the dot come out of one pass.  Every lane
// returns the value.
// hs (optional): the row staged in shared memory by the caller, so the warp's
// loads in flight are its weight row's only (same arithmetic, same bits).
__device__ __forceinline__ float qkv_dot(const AttnArgs& a, int row, int o, int lane, const uint4* hs = nullptr) {
  const int nvec = a.d >> 3;
  const uint4* hr = reinterpret_cast<const uint4*>(a.h_in + static_cast<size_t>(row) * a.d);
  const uint4* wr = reinterpret_cast<const uint4*>(a.wqkv + static_cast<size_t>(o) * a.d);
  float ss = 0.f, acc = 0.f;
#pragma unroll 16
  for (int v = lane; v < nvec; v += 32) {
    const uint4 hu = hs ? hs[v] : __ldg(hr + v), wu = __ldg(wr + v);
    const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&hu);
    const __nv_bfloat162* w2 = reinterpret_cast<const __nv_bfloat162*>(&wu);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float2 h = __bfloat1622float2(h2[j]), w = __bfloat1622float2(w2[j]);
      ss += h.x * h.x + h.y * h.y;
      acc += h.x * w.x + h.y * w.y;
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    ss += __shfl_xor_sync(kAll, ss, off);
    acc += __shfl_xor_sync(kAll, acc, off);
  }
  // x = h * s1 (s1 = 1 unless the input is the step's rms_norm(prev));
  // the attention's own rms_norm of x has mean square s1^2 * ss / d
  const float s1 = a.norm_input ? 1.f / sqrtf(ss / a.d + 1e-12f) : 1.f;
  const float s2 = 1.f / sqrtf(s1 * s1 * ss / a.d + 1e-12f);
  return acc * s1 * s2;
}

__global__ void __launch_bounds__(kAttnThreads) attn_qkv_kernel(const __grid_constant__ AttnArgs a) {
  griddep_launch_dependents();
  warm_params(a);
  griddep_wait();
  const int row = blockIdx.x;  // b * Tn + i
  const int b = row / a.Tn, i = row - b * a.Tn;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nout = 3 * a.dh;
  const int o = blockIdx.y * kQkvPerCta + warp;
  if (o >= nout) return;
  const float val = qkv_dot(a, row, o, lane);
  if (lane == 0) {
    const int which = o / a.dh, c = o - which * a.dh;
    if (which == 0) {
      a.q[static_cast<size_t>(row) * a.dh + c] = val;
    } else {
      float* cache = which == 1 ? a.kcache : a.vcache;
      cache[(static_cast<size_t>(b) * a.max_len + *a.pos + i) * a.dh + c] = val;
    }
  }
}

// Fused router: rms_norm(h_out) . W_r (simulator.py:26-27,
// 82-83) for the row this CTA writes part of.  Each CTA reduces its 1024
// columns' partial dots and sum of squares; the row's last CTA sums the
// chunks in chunk order (deterministic) and writes the f64 logits the way
// K0 does: dot * 1 / sqrt(ss / d + 1e-12).
// kCluster (the decode kernel, one cluster per row): the chunk partials go
// to the leader CTA's shared memory over DSMEM and the leader finishes, with
// the same chunk-order sums -- no global partials and no arrival counter.
template <bool kCluster>
__device__ __forceinline__ void fused_router(const AttnArgs& a, int row, int chunk, int chunks, const float (&x)[4],
                                             const uint2 (&rw)[LYNX_MAX_FUSED_ROUTER]) {
  __shared__ float red2[kAttnThreads / 32][LYNX_MAX_FUSED_ROUTER + 1];
  __shared__ float s_chunks[kMaxAttnCluster][LYNX_MAX_FUSED_ROUTER + 1];  // leader: every chunk's partials
  __shared__ int s_last;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int N = a.N;
  const bool live = chunk * kOutCols + threadIdx.x * 4 < a.d;
  float v = x[0] * x[0] + x[1] * x[1] + x[2] * x[2] + x[3] * x[3];
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(kAll, v, off);
  if (lane == 0) red2[warp][N] = v;
#pragma unroll
  for (int e = 0; e < LYNX_MAX_FUSED_ROUTER; ++e) {
    if (e >= N) break;
    float dot = 0.f;
    if (live) {
      const float2 w0 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&rw[e].x));
      const float2 w1 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&rw[e].y));
      dot = x[0] * w0.x + x[1] * w0.y + x[2] * w1.x + x[3] * w1.y;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) dot += __shfl_xor_sync(kAll, dot, off);
    if (lane == 0) red2[warp][e] = dot;
  }
  __syncthreads();
  if (kCluster) {
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    if (threadIdx.x <= N) {
      float t = 0.f;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red2[w][threadIdx.x];
      cluster.map_shared_rank(&s_chunks[0][0], 0)[chunk * (LYNX_MAX_FUSED_ROUTER + 1) + threadIdx.x] = t;
    }
    cluster.sync();
    if (chunk == 0 && threadIdx.x < N) {
      float dot = 0.f, ss = 0.f;
      for (int c = 0; c < chunks; ++c) {
        dot += s_chunks[c][threadIdx.x];
        ss += s_chunks[c][N];
      }
      const double inv = 1.0 / sqrt(static_cast<double>(ss) / a.d + 1e-12);
      a.logits[static_cast<size_t>(row) * N + threadIdx.x] = static_cast<double>(dot) * inv;
    }
    return;
  }
  float* part = a.rpart + (static_cast<size_t>(row) * chunks + chunk) * (N + 1);
  if (threadIdx.x <= N) {
    float t = 0.f;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red2[w][threadIdx.x];
    part[threadIdx.x] = t;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const int t = atomicAdd(&a.row_arrivals[row], 1);
    s_last = t == chunks - 1;
    if (s_last) a.row_arrivals[row] = 0;  // re-armed for the next launch
  }
  __syncthreads();
  if (s_last && threadIdx.x < N) {
    __threadfence();
    const float* rp = a.rpart + static_cast<size_t>(row) * chunks * (N + 1);
    float dot = 0.f, ss = 0.f;
    for (int c = 0; c < chunks; ++c) {
      dot += __ldcg(rp + c * (N + 1) + threadIdx.x);
      ss += __ldcg(rp + c * (N + 1) + N);
    }
    const double inv = 1.0 / sqrt(static_cast<double>(ss) / a.d + 1e-12);
    a.logits[static_cast<size_t>(row) * N + threadIdx.x] = static_cast<double>(dot) * inv;
  }
}

// kCluster = false: attn_out, grid (rows, column chunks), after attn_qkv.
// kCluster = true: the decode step (Tn = 1) in ONE kernel, grid (column
// chunks, rows) with one thread-block cluster per row: the cluster's CTAs
// first split the row's 3*dh q/k/v projections (qkv_dot, as attn_qkv), send q
// to every CTA's shared memory over DSMEM and write k/v to the cache; after
// a cluster barrier (release/acquire: the new cache entries are visible to
// the cluster) each CTA runs attn_out's attention and its 1024 output
// columns, and the fused router finishes in the leader over DSMEM.  The
// same arithmetic as attn_qkv + attn_out, so the same bits; it saves a
// launch boundary and the router's global partials / arrival counter.
template <bool kCluster>
__global__ void __launch_bounds__(kAttnThreads) attn_out_kernel(const __grid_constant__ AttnArgs a) {
  extern __shared__ float sm[];  // K chunk | V chunk | scores chunk | ctx partials
  __shared__ float red[32];
  __shared__ float qs[LYNX_MAX_DHEAD];
  __shared__ float ctx[LYNX_MAX_DHEAD];
  griddep_launch_dependents();
  warm_params(a);
  // DSMEM rule: peers may store into this CTA's qs only once it runs
  if (kCluster) asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
  ATT_TS(0);
  griddep_wait();
  ATT_TS(1);
  const int row = kCluster ? blockIdx.y : blockIdx.x;
  const int ochunk = kCluster ? blockIdx.x : blockIdx.y, nochunk = kCluster ? gridDim.x : gridDim.y;
  const int b = row / a.Tn, i = row - b * a.Tn;
  const int dh = a.dh, chunk = kChunkFloats / dh;
  float* Ks = sm;
  float* Vs = sm + kChunkFloats;
  float* sc = Vs + kChunkFloats;
  float* part = sc + chunk;  // [blockDim/dh][dh]
  // ---- everything this CTA reads, issued up front
  const int col = ochunk * kOutCols + threadIdx.x * 4;
  const bool live = col < a.d;
  const uint16_t* hrow = a.h_in + static_cast<size_t>(row) * a.d;
  uint2 hres = make_uint2(0, 0);
  uint2 wo[kWoPrefetch];  // the first kWoPrefetch head rows of Wo (all of them at the reference's dh = 16)
  uint2 rw[LYNX_MAX_FUSED_ROUTER];  // fused router: this thread's 4 columns of every expert's router row
  auto prefetch = [&]() {
    if (live) {
      hres = __ldg(reinterpret_cast<const uint2*>(hrow + col));
#pragma unroll
      for (int c = 0; c < kWoPrefetch; ++c)
        if (c < dh) wo[c] = __ldg(reinterpret_cast<const uint2*>(a.wo + static_cast<size_t>(c) * a.d + col));
      if (a.router_wt) {
#pragma unroll
        for (int e = 0; e < LYNX_MAX_FUSED_ROUTER; ++e)
          if (e < a.N) rw[e] = __ldg(reinterpret_cast<const uint2*>(a.router_wt + static_cast<size_t>(e) * a.d + col));
      }
    }
  };
  // decode kernel: the projections' loads go first, the output-side
  // prefetch after them (it has the attention's duration to land)
  if (!kCluster) prefetch();
  if (kCluster) {
    // q / k / v: output o = ochunk + nochunk * (warp + 8 r) on this CTA; the
    // row is staged in shared memory once, so each warp's loads in flight
    // are only its weight row's (one round trip per projection)
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    __shared__ uint4 s_row[8192 / 8];  // d <= 8192 (kMaxAttnCluster chunks of 1024)
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int v = threadIdx.x; v < (a.d >> 3); v += blockDim.x) s_row[v] = __ldg(reinterpret_cast<const uint4*>(hrow) + v);
    const int pos = *a.pos;  // loaded once: a store address must not stall the next projection's loads
    __syncthreads();
    ATT_TS(10);
    asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
    ATT_TS(11);
    for (int o = ochunk + nochunk * warp; o < 3 * dh; o += nochunk * (kAttnThreads / 32)) {
      const float val = qkv_dot(a, row, o, lane, s_row);
      const int which = o / dh, c = o - which * dh;
      if (which == 0) {
        if (lane < nochunk) cluster.map_shared_rank(&qs[0], lane)[c] = val;
      } else if (lane == 0) {
        float* cache = which == 1 ? a.kcache : a.vcache;
        cache[(static_cast<size_t>(b) * a.max_len + pos + i) * dh + c] = val;
      }
      if (o == ochunk) ATT_TS(9);  // warp 0's first projection done
    }
    prefetch();
    ATT_TS(2);
    cluster.sync();  // q in every CTA, the new k / v entries visible to the cluster
    ATT_TS(3);
  } else if (threadIdx.x < dh) {
    qs[threadIdx.x] = a.q[static_cast<size_t>(row) * dh + threadIdx.x];
  }
  const int total = *a.pos + i + 1;  // causal: cache positions 0 .. pos+i
  const float* K = a.kcache + static_cast<size_t>(b) * a.max_len * dh;
  const float* V = a.vcache + static_cast<size_t>(b) * a.max_len * dh;
  const float s1 = a.norm_input ? 1.f / sqrtf(row_sumsq(hrow, a.d, red) / a.d + 1e-12f) : 1.f;
  ATT_TS(4);
  const float inv_sqrt = 1.f / sqrtf(static_cast<float>(dh));
  const int per = blockDim.x / dh;
  float m_run = -INFINITY, l_run = 0.f, c_run = 0.f;  // c_run: this thread's (c, slice) ctx partial
  for (int j0 = 0; j0 < total; j0 += chunk) {
    const int n = min(chunk, total - j0);
    // K/V chunk -> shared (float4, coalesced)
    const float4* K4 = reinterpret_cast<const float4*>(K + static_cast<size_t>(j0) * dh);
    const float4* V4 = reinterpret_cast<const float4*>(V + static_cast<size_t>(j0) * dh);
    for (int t = threadIdx.x; t < n * dh / 4; t += blockDim.x) {
      reinterpret_cast<float4*>(Ks)[t] = K4[t];
      reinterpret_cast<float4*>(Vs)[t] = V4[t];
    }
    __syncthreads();
    float m = -INFINITY;
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
      float sj = 0.f;
      for (int c = 0; c < dh; ++c) sj += qs[c] * Ks[j * dh + c];
      sj *= inv_sqrt;
      sc[j] = sj;
      m = fmaxf(m, sj);
    }
    m = block_max(m, red);
    const float m_new = fmaxf(m_run, m);
    float l = 0.f;
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
      const float e = __expf(sc[j] - m_new);
      sc[j] = e;
      l += e;
    }
    l = block_sum(l, red);  // also a barrier: sc[] complete
    const float rescale = __expf(m_run - m_new);
    l_run = l_run * rescale + l;
    m_run = m_new;
    if (threadIdx.x < per * dh) {
      const int c = threadIdx.x % dh, s0 = threadIdx.x / dh;
      float acc = 0.f;
      for (int j = s0; j < n; j += per) acc += sc[j] * Vs[j * dh + c];
      c_run = c_run * rescale + acc;
    }
    __syncthreads();  // Ks/Vs/sc reused by the next chunk
  }
  ATT_TS(5);
  if (threadIdx.x < per * dh) part[(threadIdx.x / dh) * dh + threadIdx.x % dh] = c_run;
  __syncthreads();
  if (threadIdx.x < dh) {
    float acc = 0.f;
    for (int s0 = 0; s0 < per; ++s0) acc += part[s0 * dh + threadIdx.x];
    ctx[threadIdx.x] = acc / l_run;
  }
  __syncthreads();
  ATT_TS(6);
  float rout[4] = {0.f, 0.f, 0.f, 0.f};
  if (live) {
    float o[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int c = 0; c < kWoPrefetch; ++c)
      if (c < dh) {
        const float2 w0 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&wo[c].x));
        const float2 w1 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&wo[c].y));
        o[0] += ctx[c] * w0.x;
        o[1] += ctx[c] * w0.y;
        o[2] += ctx[c] * w1.x;
        o[3] += ctx[c] * w1.y;
      }
#pragma unroll 8
    for (int c = kWoPrefetch; c < dh; ++c) {
      const uint2 u = __ldg(reinterpret_cast<const uint2*>(a.wo + static_cast<size_t>(c) * a.d + col));
      const float2 w0 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.x));
      const float2 w1 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.y));
      o[0] += ctx[c] * w0.x;
      o[1] += ctx[c] * w0.y;
      o[2] += ctx[c] * w1.x;
      o[3] += ctx[c] * w1.y;
    }
    const float2 h0 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&hres.x));
    const float2 h1 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&hres.y));
    uint2 out;
    *reinterpret_cast<__nv_bfloat162*>(&out.x) = __floats2bfloat162_rn(h0.x * s1 + o[0], h0.y * s1 + o[1]);
    *reinterpret_cast<__nv_bfloat162*>(&out.y) = __floats2bfloat162_rn(h1.x * s1 + o[2], h1.y * s1 + o[3]);
    *reinterpret_cast<uint2*>(a.h_out + static_cast<size_t>(row) * a.d + col) = out;
    if (a.router_wt) {
      // the next layer's router on the values as stored (bf16), like K0
      const float2 y0 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&out.x));
      const float2 y1 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&out.y));
      rout[0] = y0.x;
      rout[1] = y0.y;
      rout[2] = y1.x;
      rout[3] = y1.y;
    }
  }
  ATT_TS(7);
  if (a.router_wt) fused_router<kCluster>(a, row, ochunk, nochunk, rout, rw);
  ATT_TS(8);
}

__global__ void advance_position_kernel(int32_t* pos, int by) {
  griddep_wait();
  if (threadIdx.x == 0) *pos += by;
}

size_t attn_out_smem(int d, int dh, int max_len) {
  (void)d;
  (void)max_len;
  return sizeof(float) * (2 * kChunkFloats + kChunkFloats / dh + (kAttnThreads / dh) * dh);
}

// LYNX_ATTN_CLUSTER=0 keeps the two-kernel decode attention (A/B switch).
static bool decode_cluster_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("LYNX_ATTN_CLUSTER");
    v = (e && e[0] == '0' && !e[1]) ? 0 : 1;
  }
  return v == 1;
}

cudaError_t launch_attention(const AttnArgs& a, cudaStream_t s) {
  const size_t smem_a = 0;
  const size_t smem_b = attn_out_smem(a.d, a.dh, a.max_len);
  static int configured = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (configured != dev) {
    cudaError_t e = cudaFuncSetAttribute(attn_out_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(attn_out_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(attn_qkv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (e != cudaSuccess) return e;
    configured = dev;
  }
  const int rows = a.B * a.Tn, chunks = (a.d + kOutCols - 1) / kOutCols;
  if (a.Tn == 1 && chunks <= kMaxAttnCluster && decode_cluster_enabled()) {
    // decode: one kernel, a cluster of `chunks` CTAs per row
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(chunks, rows);
    cfg.blockDim = dim3(kAttnThreads);
    cfg.dynamicSmemBytes = smem_b;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = chunks;
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    return cudaLaunchKernelEx(&cfg, attn_out_kernel<true>, a);
  }
  cudaError_t e = launch_pdl(attn_qkv_kernel, dim3(rows, (3 * a.dh + kQkvPerCta - 1) / kQkvPerCta),
                             dim3(kAttnThreads), smem_a, s, a);
  if (e != cudaSuccess) return e;
  return launch_pdl(attn_out_kernel<false>, dim3(rows, chunks), dim3(kAttnThreads), smem_b, s, a);
}

#ifdef LYNX_TRACE
extern "C" int lynx_debug_attn_ts(unsigned long long* host) {
  return cudaMemcpyFromSymbol(host, g_attn_ts, sizeof(g_attn_ts)) == cudaSuccess ? 16 : -1;
}
#endif

cudaError_t launch_advance_position(int32_t* pos, int by, cudaStream_t s) {
  return launch_pdl(advance_position_kernel, dim3(1), dim3(32), 0, s, pos, by);
}

}  // namespace lynx
