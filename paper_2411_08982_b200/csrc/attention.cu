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
//   A  attn_qkv:  RMSNorm + the 3*dh projections (warp per output row, 16-byte
//                 weight loads) -> q scratch, k/v appended to the cache.
//   B  attn_out:  scores over the visible cache, softmax, ctx, ctx Wo + the
//                 residual -> h_out (bf16).
// A chunk of Tn new tokens per sequence (prefill: Tn = P; decode: Tn = 1)
// sits at cache positions pos .. pos+Tn-1; `pos` is read from device memory
// so one captured decode step can be replayed step after step
// (lynx_advance_position bumps it inside the graph).
#include <cuda_bf16.h>
#include <stdint.h>

#include "lynx_internal.cuh"

namespace lynx {

constexpr int kAttnThreads = 256;
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

// x (shared, f32) <- row of h_in, optionally rms-normalised (the decode
// step's input is rms_norm(prev), simulator.py:353); returns rms_norm scale
// of the resulting x (the attention's own rms_norm, simulator.py:310).
__device__ __forceinline__ float load_row(const AttnArgs& a, int row, float* x, float* red) {
  const uint16_t* src = a.h_in + static_cast<size_t>(row) * a.d;
  float ss = 0.f;
  for (int c = threadIdx.x * 2; c < a.d; c += blockDim.x * 2) {
    const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(src + c));
    x[c] = f.x;
    x[c + 1] = f.y;
    ss += f.x * f.x + f.y * f.y;
  }
  ss = block_sum(ss, red);
  float scale = 1.f / sqrtf(ss / a.d + 1e-12f);
  if (a.norm_input) {
    for (int c = threadIdx.x; c < a.d; c += blockDim.x) x[c] *= scale;
    // rms of the normalised row is 1 up to rounding; recompute exactly
    float s2 = 0.f;
    for (int c = threadIdx.x; c < a.d; c += blockDim.x) s2 += x[c] * x[c];
    s2 = block_sum(s2, red);
    scale = 1.f / sqrtf(s2 / a.d + 1e-12f);
  }
  __syncthreads();
  return scale;
}

// Latency shaping: the grid spreads a token's work over several CTAs
// (blockIdx.y) so every lane issues all of its 16-byte weight loads at once
// and a kernel costs a couple of L2 round trips.  qkv: one projection per
// warp, 8 per CTA.  out: 1024 output columns per CTA (4 per thread).
constexpr int kQkvPerCta = kAttnThreads / 32;
constexpr int kOutCols = kAttnThreads * 4;

__global__ void __launch_bounds__(kAttnThreads) attn_qkv_kernel(const __grid_constant__ AttnArgs a) {
  extern __shared__ float x[];  // [d]
  __shared__ float red[32];
  griddep_launch_dependents();
  griddep_wait();
  const int row = blockIdx.x;  // b * Tn + i
  const int b = row / a.Tn, i = row - b * a.Tn;
  const float scale = load_row(a, row, x, red);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nout = 3 * a.dh, nvec = a.d >> 3;
  const int o = blockIdx.y * kQkvPerCta + warp;
  if (o >= nout) return;
  const uint4* wr = reinterpret_cast<const uint4*>(a.wqkv + static_cast<size_t>(o) * a.d);
  float acc = 0.f;
#pragma unroll 16
  for (int v = lane; v < nvec; v += 32) {
    const uint4 u = __ldg(wr + v);
    const float4 x0 = *reinterpret_cast<const float4*>(x + 8 * v);
    const float4 x1 = *reinterpret_cast<const float4*>(x + 8 * v + 4);
    const __nv_bfloat162* w2 = reinterpret_cast<const __nv_bfloat162*>(&u);
    float2 f = __bfloat1622float2(w2[0]);
    acc += x0.x * f.x + x0.y * f.y;
    f = __bfloat1622float2(w2[1]);
    acc += x0.z * f.x + x0.w * f.y;
    f = __bfloat1622float2(w2[2]);
    acc += x1.x * f.x + x1.y * f.y;
    f = __bfloat1622float2(w2[3]);
    acc += x1.z * f.x + x1.w * f.y;
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(kAll, acc, off);
  if (lane == 0) {
    acc *= scale;  // (x * s) . w == s * (x . w)
    const int which = o / a.dh, c = o - which * a.dh;
    if (which == 0) {
      a.q[static_cast<size_t>(row) * a.dh + c] = acc;
    } else {
      float* cache = which == 1 ? a.kcache : a.vcache;
      cache[(static_cast<size_t>(b) * a.max_len + *a.pos + i) * a.dh + c] = acc;
    }
  }
}

__global__ void __launch_bounds__(kAttnThreads) attn_out_kernel(const __grid_constant__ AttnArgs a) {
  extern __shared__ float sm[];  // x[d] | scores[max_len] | ctx partials
  __shared__ float red[32];
  __shared__ float qs[LYNX_MAX_DHEAD];
  __shared__ float ctx[LYNX_MAX_DHEAD];
  griddep_launch_dependents();
  griddep_wait();
  const int row = blockIdx.x;
  const int b = row / a.Tn, i = row - b * a.Tn;
  float* x = sm;
  float* sc = sm + a.d;
  const int dh = a.dh;
  if (threadIdx.x < dh) qs[threadIdx.x] = a.q[static_cast<size_t>(row) * dh + threadIdx.x];
  load_row(a, row, x, red);  // ends with a barrier: qs visible
  const int total = *a.pos + i + 1;  // causal: cache positions 0 .. pos+i
  const float* K = a.kcache + static_cast<size_t>(b) * a.max_len * dh;
  const float* V = a.vcache + static_cast<size_t>(b) * a.max_len * dh;
  const float inv_sqrt = 1.f / sqrtf(static_cast<float>(dh));
  // scores: half a warp per cached position, lanes over the head dimension
  const int lane = threadIdx.x & 31, half = lane >> 4, hl = lane & 15;
  const int hw = (threadIdx.x >> 5) * 2 + half, nhw = (blockDim.x >> 5) * 2;
  float m = -INFINITY;
  for (int jb = hw - half; jb < total; jb += nhw) {  // warp-uniform trip count
    const int j = jb + half;
    float s = 0.f;
    if (j < total) {
#pragma unroll
      for (int c0 = 0; c0 < LYNX_MAX_DHEAD; c0 += 16)
        if (c0 + hl < dh) s += qs[c0 + hl] * K[static_cast<size_t>(j) * dh + c0 + hl];
    }
#pragma unroll
    for (int off = 8; off > 0; off >>= 1) s += __shfl_xor_sync(kAll, s, off);
    s *= inv_sqrt;
    if (j < total) {
      if (hl == 0) sc[j] = s;
      m = fmaxf(m, s);
    }
  }
  m = block_max(m, red);
  float l = 0.f;
  for (int j = threadIdx.x; j < total; j += blockDim.x) {
    const float e = __expf(sc[j] - m);
    sc[j] = e;
    l += e;
  }
  l = block_sum(l, red);  // also a barrier: sc[] complete
  // ctx[c] = sum_j p_j V[j][c]: thread (c, slice of j)
  float* part = sc + a.max_len;  // [blockDim/dh][dh]
  const int per = blockDim.x / dh;
  if (threadIdx.x < per * dh) {
    const int c = threadIdx.x % dh, s0 = threadIdx.x / dh;
    float acc = 0.f;
#pragma unroll 4
    for (int j = s0; j < total; j += per) acc += sc[j] * V[static_cast<size_t>(j) * dh + c];
    part[s0 * dh + c] = acc;
  }
  __syncthreads();
  if (threadIdx.x < dh) {
    float acc = 0.f;
    for (int s0 = 0; s0 < per; ++s0) acc += part[s0 * dh + threadIdx.x];
    ctx[threadIdx.x] = acc / l;
  }
  __syncthreads();
  // h_out = x + ctx Wo for this CTA's 1024 columns (Wo stored [dh, d]:
  // coalesced over the columns; every head row's load is in flight at once)
  uint16_t* dst = a.h_out + static_cast<size_t>(row) * a.d;
  const int col = blockIdx.y * kOutCols + threadIdx.x * 4;
  if (col < a.d) {
    float o[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll 16
    for (int c = 0; c < dh; ++c) {
      const uint2 u = __ldg(reinterpret_cast<const uint2*>(a.wo + static_cast<size_t>(c) * a.d + col));
      const float2 w0 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.x));
      const float2 w1 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.y));
      o[0] += ctx[c] * w0.x;
      o[1] += ctx[c] * w0.y;
      o[2] += ctx[c] * w1.x;
      o[3] += ctx[c] * w1.y;
    }
    uint2 out;
    *reinterpret_cast<__nv_bfloat162*>(&out.x) = __floats2bfloat162_rn(x[col] + o[0], x[col + 1] + o[1]);
    *reinterpret_cast<__nv_bfloat162*>(&out.y) = __floats2bfloat162_rn(x[col + 2] + o[2], x[col + 3] + o[3]);
    *reinterpret_cast<uint2*>(dst + col) = out;
  }
}

__global__ void advance_position_kernel(int32_t* pos, int by) {
  griddep_wait();
  if (threadIdx.x == 0) *pos += by;
}

size_t attn_out_smem(int d, int dh, int max_len) {
  return sizeof(float) * (static_cast<size_t>(d) + max_len + (kAttnThreads / dh) * dh);
}

cudaError_t launch_attention(const AttnArgs& a, cudaStream_t s) {
  const size_t smem_a = sizeof(float) * a.d;
  const size_t smem_b = attn_out_smem(a.d, a.dh, a.max_len);
  static int configured = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (configured != dev) {
    cudaError_t e = cudaFuncSetAttribute(attn_out_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(attn_qkv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (e != cudaSuccess) return e;
    configured = dev;
  }
  const int rows = a.B * a.Tn;
  cudaError_t e = launch_pdl(attn_qkv_kernel, dim3(rows, (3 * a.dh + kQkvPerCta - 1) / kQkvPerCta),
                             dim3(kAttnThreads), smem_a, s, a);
  if (e != cudaSuccess) return e;
  return launch_pdl(attn_out_kernel, dim3(rows, (a.d + kOutCols - 1) / kOutCols), dim3(kAttnThreads), smem_b, s,
                    a);
}

cudaError_t launch_advance_position(int32_t* pos, int by, cudaStream_t s) {
  return launch_pdl(advance_position_kernel, dim3(1), dim3(32), 0, s, pos, by);
}

}  // namespace lynx
