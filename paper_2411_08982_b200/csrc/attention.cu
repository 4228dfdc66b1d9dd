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

__global__ void __launch_bounds__(kAttnThreads) attn_qkv_kernel(const __grid_constant__ AttnArgs a) {
  extern __shared__ float x[];  // [d]
  __shared__ float red[32];
  griddep_launch_dependents();
  griddep_wait();
  const int row = blockIdx.x;  // b * Tn + i
  const int b = row / a.Tn, i = row - b * a.Tn;
  const float scale = load_row(a, row, x, red);
  const int pos = *a.pos + i;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int nout = 3 * a.dh;
  for (int o = warp; o < nout; o += nw) {
    const uint4* wr = reinterpret_cast<const uint4*>(a.wqkv + static_cast<size_t>(o) * a.d);
    float acc = 0.f;
    for (int v = lane; v < (a.d >> 3); v += 32) {
      const uint4 u = wr[v];
      const __nv_bfloat162* w2 = reinterpret_cast<const __nv_bfloat162*>(&u);
      const float* xs = x + 8 * v;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 f = __bfloat1622float2(w2[j]);
        acc += xs[2 * j] * f.x + xs[2 * j + 1] * f.y;
      }
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
        cache[(static_cast<size_t>(b) * a.max_len + pos) * a.dh + c] = acc;
      }
    }
  }
}

__global__ void __launch_bounds__(kAttnThreads) attn_out_kernel(const __grid_constant__ AttnArgs a) {
  extern __shared__ float sm[];  // x[d] | scores[max_len] | ctx partials
  __shared__ float red[32];
  __shared__ float ctx[LYNX_MAX_DHEAD];
  griddep_launch_dependents();
  griddep_wait();
  const int row = blockIdx.x;
  const int b = row / a.Tn, i = row - b * a.Tn;
  float* x = sm;
  float* sc = sm + a.d;
  load_row(a, row, x, red);
  const int total = *a.pos + i + 1;  // causal: cache positions 0 .. pos+i
  const float* q = a.q + static_cast<size_t>(row) * a.dh;
  const float* K = a.kcache + static_cast<size_t>(b) * a.max_len * a.dh;
  const float* V = a.vcache + static_cast<size_t>(b) * a.max_len * a.dh;
  const float inv_sqrt = 1.f / sqrtf(static_cast<float>(a.dh));
  float m = -INFINITY;
  for (int j = threadIdx.x; j < total; j += blockDim.x) {
    float s = 0.f;
    for (int c = 0; c < a.dh; ++c) s += q[c] * K[static_cast<size_t>(j) * a.dh + c];
    s *= inv_sqrt;
    sc[j] = s;
    m = fmaxf(m, s);
  }
  m = block_max(m, red);
  float l = 0.f;
  for (int j = threadIdx.x; j < total; j += blockDim.x) {
    const float e = __expf(sc[j] - m);
    sc[j] = e;
    l += e;
  }
  l = block_sum(l, red);  // also a barrier: sc[] complete
  // ctx[c] = sum_j p_j V[j][c]: thread (c, lane-slice of j)
  float* part = sc + a.max_len;  // [blockDim/dh][dh]
  const int per = blockDim.x / a.dh;
  if (threadIdx.x < per * a.dh) {
    const int c = threadIdx.x % a.dh, s0 = threadIdx.x / a.dh;
    float acc = 0.f;
    for (int j = s0; j < total; j += per) acc += sc[j] * V[static_cast<size_t>(j) * a.dh + c];
    part[s0 * a.dh + c] = acc;
  }
  __syncthreads();
  if (threadIdx.x < a.dh) {
    float acc = 0.f;
    for (int s0 = 0; s0 < per; ++s0) acc += part[s0 * a.dh + threadIdx.x];
    ctx[threadIdx.x] = acc / l;
  }
  __syncthreads();
  // h_out = x + ctx Wo   (Wo stored [dh, d]: coalesced over the columns)
  uint16_t* dst = a.h_out + static_cast<size_t>(row) * a.d;
  for (int col = threadIdx.x * 2; col < a.d; col += blockDim.x * 2) {
    float o0 = 0.f, o1 = 0.f;
    for (int c = 0; c < a.dh; ++c) {
      const float2 w = __bfloat1622float2(
          *reinterpret_cast<const __nv_bfloat162*>(a.wo + static_cast<size_t>(c) * a.d + col));
      o0 += ctx[c] * w.x;
      o1 += ctx[c] * w.y;
    }
    *reinterpret_cast<__nv_bfloat162*>(dst + col) = __floats2bfloat162_rn(x[col] + o0, x[col + 1] + o1);
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
  const dim3 grid(a.B * a.Tn);
  cudaError_t e = launch_pdl(attn_qkv_kernel, grid, dim3(kAttnThreads), smem_a, s, a);
  if (e != cudaSuccess) return e;
  return launch_pdl(attn_out_kernel, grid, dim3(kAttnThreads), smem_b, s, a);
}

cudaError_t launch_advance_position(int32_t* pos, int by, cudaStream_t s) {
  return launch_pdl(advance_position_kernel, dim3(1), dim3(32), 0, s, pos, by);
}

}  // namespace lynx
