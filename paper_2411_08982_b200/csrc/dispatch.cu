// dispatch.cu -- K2 histogram/scan permutation + gather, K4 weighted
// combine, gate/up weight packing and the expert-parallel pack/combine
// helpers.
//
// Reference order (simulator.py:101-113): out = hidden.copy(); for each
// used expert e ascending (np.unique(assigned)), rows = the tokens with a
// slot on e, ascending; the row's gate weight is the sum of its slot
// weights on e in slot order; out[rows] += w * expert(hidden[rows]).
#include <cuda_bf16.h>
#include <stdint.h>

#include "lynx_internal.cuh"

namespace lynx {

constexpr int kPermThreads = 512;

__device__ __forceinline__ int round16(int v) { return (v + 15) & ~15; }

// Every CTA rebuilds the (tiny) expert x token bitmap in shared memory, so
// no grid-wide barrier is needed; CTAs then split the tokens for the
// gather and the per-token bookkeeping.
__global__ void __launch_bounds__(kPermThreads) permute_kernel(PermuteArgs a) {
  extern __shared__ uint32_t s_bits[];  // [N][W] bitmap, then [N][W] prefix counts
  __shared__ int s_cnt[LYNX_MAX_EXPERTS];
  __shared__ int s_base[LYNX_MAX_EXPERTS];
  __shared__ int s_list_row[LYNX_MAX_TOPK];
  __shared__ float s_list_w[LYNX_MAX_TOPK];
  __shared__ int s_nl;

  const int T = a.T, N = a.N, k = a.k, d = a.d;
  const int W = (T + 31) >> 5;
  int* s_prefix = reinterpret_cast<int*>(s_bits + N * W);
  const int tid = threadIdx.x;

  for (int i = tid; i < N * W; i += blockDim.x) s_bits[i] = 0;
  __syncthreads();
  for (int i = tid; i < T * k; i += blockDim.x) {
    const int e = a.assigned[i];
    if (e >= 0 && e < N) {
      const int t = i / k;
      atomicOr(&s_bits[e * W + (t >> 5)], 1u << (t & 31));
    }
  }
  __syncthreads();
  for (int e = tid; e < N; e += blockDim.x) {
    int run = 0;
    for (int w = 0; w < W; ++w) {
      s_prefix[e * W + w] = run;
      run += __popc(s_bits[e * W + w]);
    }
    s_cnt[e] = run;
  }
  __syncthreads();
  if (tid == 0) {
    int base = 0, nseg = 0, nused = 0;
    for (int e = 0; e < N; ++e) {
      const int cnt = s_cnt[e];
      if (cnt == 0) {
        s_base[e] = -1;
        continue;
      }
      s_base[e] = base;
      ++nused;
      for (int c0 = 0; c0 < cnt; c0 += LYNX_SEG_ROWS) {
        if (blockIdx.x == 0) {
          a.out.seg_expert[nseg] = e;
          a.out.seg_row[nseg] = base + c0;
          a.out.seg_count[nseg] = cnt - c0 < LYNX_SEG_ROWS ? cnt - c0 : LYNX_SEG_ROWS;
        }
        ++nseg;
      }
      base += round16(cnt);
    }
    if (blockIdx.x == 0) {
      *a.out.n_seg = nseg;
      *a.out.n_used = nused;
    }
  }
  if (blockIdx.x == 0)
    for (int i = tid; i < a.n_counters; i += blockDim.x) a.counters[i] = 0;
  __syncthreads();

  const int nvec = d >> 3;  // 16-byte vectors per row
  for (int t = blockIdx.x; t < T; t += gridDim.x) {
    if (tid == 0) {
      int ids[LYNX_MAX_TOPK];
      int n = 0;
      for (int c = 0; c < k; ++c) {
        const int e = a.assigned[t * k + c];
        if (e < 0 || e >= N) continue;
        bool dup = false;
        for (int j = 0; j < n; ++j) dup |= ids[j] == e;
        if (dup) continue;
        int j = n++;
        while (j > 0 && ids[j - 1] > e) {
          ids[j] = ids[j - 1];
          --j;
        }
        ids[j] = e;
      }
      for (int j = 0; j < n; ++j) {
        const int e = ids[j];
        const uint32_t word = s_bits[e * W + (t >> 5)];
        const int pos = s_prefix[e * W + (t >> 5)] + __popc(word & ((1u << (t & 31)) - 1u));
        const int row = s_base[e] + pos;
        double w = 0.0;
        for (int c = 0; c < k; ++c)
          if (a.assigned[t * k + c] == e) w += a.weights[t * k + c];
        s_list_row[j] = row;
        s_list_w[j] = static_cast<float>(w);
        a.out.tok_rows[t * k + j] = row;
        a.out.tok_weight[t * k + j] = static_cast<float>(w);
        a.out.perm_token[row] = t;
        a.out.perm_weight[row] = static_cast<float>(w);
      }
      for (int j = n; j < k; ++j) {
        a.out.tok_rows[t * k + j] = -1;
        a.out.tok_weight[t * k + j] = 0.f;
      }
      s_nl = n;
    }
    __syncthreads();
    const uint4* src = reinterpret_cast<const uint4*>(a.hidden + static_cast<size_t>(t) * d);
    for (int j = 0; j < s_nl; ++j) {
      uint4* dst = reinterpret_cast<uint4*>(a.out.x_perm + static_cast<size_t>(s_list_row[j]) * d);
      for (int v = tid; v < nvec; v += blockDim.x) dst[v] = src[v];
    }
    __syncthreads();
  }
  // Padding rows of each used expert: zero input, no token.
  for (int e = blockIdx.x; e < N; e += gridDim.x) {
    const int cnt = s_cnt[e];
    if (cnt == 0) continue;
    const int r0 = s_base[e] + cnt, r1 = s_base[e] + round16(cnt);
    for (int r = r0; r < r1; ++r) {
      uint4* dst = reinterpret_cast<uint4*>(a.out.x_perm + static_cast<size_t>(r) * d);
      for (int v = tid; v < nvec; v += blockDim.x) dst[v] = make_uint4(0, 0, 0, 0);
      if (tid == 0) {
        a.out.perm_token[r] = -1;
        a.out.perm_weight[r] = 0.f;
      }
    }
  }
}

cudaError_t launch_permute(const PermuteArgs& a, int sm_count, cudaStream_t s) {
  const int W = (a.T + 31) / 32;
  const size_t smem = static_cast<size_t>(a.N) * W * 8;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(permute_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
  }
  int grid = a.T < sm_count ? a.T : sm_count;
  if (grid < 1) grid = 1;
  permute_kernel<<<grid, kPermThreads, smem, s>>>(a);
  return cudaGetLastError();
}

// ------------------------------------------------------------------- K4
// y[t] = hidden[t] + sum_j w_j * (sum_s partial[s][row_j]), j over the
// token's experts ascending -- the reference's accumulation order.
__global__ void __launch_bounds__(256) combine_kernel(CombineArgs a) {
  const int t = blockIdx.x;
  const int c = (blockIdx.y * blockDim.x + threadIdx.x) * 4;
  if (c >= a.d) return;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  if (a.hidden) {
    const __nv_bfloat162* h =
        reinterpret_cast<const __nv_bfloat162*>(a.hidden + static_cast<size_t>(t) * a.d + c);
    const float2 h0 = __bfloat1622float2(h[0]), h1 = __bfloat1622float2(h[1]);
    acc = make_float4(h0.x, h0.y, h1.x, h1.y);
  }
  for (int j = 0; j < a.k; ++j) {
    const int row = a.tok_rows[t * a.k + j];
    if (row < 0) break;
    const float w = a.tok_weight[t * a.k + j];
    float4 y = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int sp = 0; sp < a.split2; ++sp) {
      const float4 v = *reinterpret_cast<const float4*>(
          a.partial + (static_cast<size_t>(sp) * a.rows_cap + row) * a.d + c);
      y.x += v.x;
      y.y += v.y;
      y.z += v.z;
      y.w += v.w;
    }
    acc.x += w * y.x;
    acc.y += w * y.y;
    acc.z += w * y.z;
    acc.w += w * y.w;
  }
  const size_t o = static_cast<size_t>(t) * a.d + c;
  if (a.out_f32) {
    *reinterpret_cast<float4*>(a.out_f32 + o) = acc;
  } else {
    __nv_bfloat162* out = reinterpret_cast<__nv_bfloat162*>(a.out_bf16 + o);
    out[0] = __floats2bfloat162_rn(acc.x, acc.y);
    out[1] = __floats2bfloat162_rn(acc.z, acc.w);
  }
}

cudaError_t launch_combine(const CombineArgs& a, cudaStream_t s) {
  dim3 grid(a.T, (a.d + 1023) / 1024);
  combine_kernel<<<grid, 256, 0, s>>>(a);
  return cudaGetLastError();
}

// --------------------------------------------------------------- packing
// w13 row r of expert e: tile = r/128, q = (r%128)/32, half = (r%32)/16,
// i = r%16 -> feature f = 64*tile + 16*q + i of w1 (half 0) or w3 (half 1).
// Gate and up of a feature sit 16 TMEM lanes apart in the same warp
// quarter, so the epilogue pairs them with one shuffle.
__global__ void pack_w13_kernel(const uint16_t* w1, const uint16_t* w3, int ff, int d, int rows, uint16_t* w13) {
  const int e = blockIdx.y;
  const int r = blockIdx.x;
  const int tile = r >> 7, q = (r & 127) >> 5, half = (r & 31) >> 4, i = r & 15;
  const int f = tile * 64 + q * 16 + i;
  uint16_t* dst = w13 + (static_cast<size_t>(e) * rows + r) * d;
  if (f < ff) {
    const uint16_t* src = (half ? w3 : w1) + (static_cast<size_t>(e) * ff + f) * d;
    for (int c = threadIdx.x; c < d; c += blockDim.x) dst[c] = src[c];
  } else {
    for (int c = threadIdx.x; c < d; c += blockDim.x) dst[c] = 0;
  }
}

cudaError_t launch_pack_w13(const uint16_t* w1, const uint16_t* w3, int N, int ff, int d, uint16_t* w13,
                            cudaStream_t s) {
  const int rows = swiglu_rows(ff);
  pack_w13_kernel<<<dim3(rows, N), 256, 0, s>>>(w1, w3, ff, d, rows, w13);
  return cudaGetLastError();
}

// -------------------------------------------------------- expert parallel
// send[p][i] = hidden_local[i] when global token rank*T_local+i has a slot on
// an expert owned by rank p, else zeros.
__global__ void ep_pack_kernel(const uint16_t* hidden, const int32_t* assigned, int T_local, int k, int N, int G,
                               int d, int rank, uint16_t* send) {
  const int i = blockIdx.x, p = blockIdx.y;
  const int t = rank * T_local + i;
  const int per = N / G;
  bool need = false;
  for (int c = 0; c < k; ++c) {
    const int e = assigned[t * k + c];
    need |= e >= 0 && e / per == p;
  }
  const uint4* src = reinterpret_cast<const uint4*>(hidden + static_cast<size_t>(i) * d);
  uint4* dst = reinterpret_cast<uint4*>(send + (static_cast<size_t>(p) * T_local + i) * d);
  for (int v = threadIdx.x; v < (d >> 3); v += blockDim.x) dst[v] = need ? src[v] : make_uint4(0, 0, 0, 0);
}

cudaError_t launch_ep_pack(const uint16_t* hidden_local, const int32_t* assigned, int T_local, int k, int N, int G,
                           int d, int rank, uint16_t* send, cudaStream_t s) {
  ep_pack_kernel<<<dim3(T_local, G), 128, 0, s>>>(hidden_local, assigned, T_local, k, N, G, d, rank, send);
  return cudaGetLastError();
}

// Keep only this rank's experts, renumbered locally; others become -1.
__global__ void ep_local_mask_kernel(const int32_t* assigned, const double* weights, int n, int N, int G, int rank,
                                     int32_t* assigned_local, double* weights_local) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int per = N / G;
  const int e = assigned[i];
  assigned_local[i] = e / per == rank ? e - rank * per : -1;
  weights_local[i] = weights[i];
}

cudaError_t launch_ep_local_mask(const int32_t* assigned, const double* weights, int T, int k, int N, int G,
                                 int rank, int32_t* assigned_local, double* weights_local, cudaStream_t s) {
  const int n = T * k;
  ep_local_mask_kernel<<<(n + 255) / 256, 256, 0, s>>>(assigned, weights, n, N, G, rank, assigned_local,
                                                       weights_local);
  return cudaGetLastError();
}

// out[i] = hidden_local[i] + sum_p recv[p][i], p ascending (= experts ascending).
__global__ void ep_combine_kernel(const uint16_t* hidden, const float* recv, int T_local, int G, int d,
                                  uint16_t* out) {
  const int i = blockIdx.x;
  for (int c = threadIdx.x * 2; c < d; c += blockDim.x * 2) {
    const float2 h = __bfloat1622float2(
        *reinterpret_cast<const __nv_bfloat162*>(hidden + static_cast<size_t>(i) * d + c));
    float sx = 0.f, sy = 0.f;
    for (int p = 0; p < G; ++p) {
      const float2 v = *reinterpret_cast<const float2*>(recv + (static_cast<size_t>(p) * T_local + i) * d + c);
      sx += v.x;
      sy += v.y;
    }
    *reinterpret_cast<__nv_bfloat162*>(out + static_cast<size_t>(i) * d + c) =
        __floats2bfloat162_rn(h.x + sx, h.y + sy);
  }
}

cudaError_t launch_ep_combine(const uint16_t* hidden_local, const float* recv, int T_local, int G, int d,
                              uint16_t* out, cudaStream_t s) {
  ep_combine_kernel<<<T_local, 256, 0, s>>>(hidden_local, recv, T_local, G, d, out);
  return cudaGetLastError();
}

}  // namespace lynx
