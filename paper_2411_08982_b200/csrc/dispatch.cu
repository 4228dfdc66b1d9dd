// dispatch.cu -- K2 gather of the dispatched rows, gate/up weight packing
// and the expert-parallel pack/combine helpers.
//
// Reference order (simulator.py:101-113): out = hidden.copy(); for each
// used expert e ascending (np.unique(assigned)), rows = the tokens with a
// slot on e, ascending; the row's gate weight is the sum of its slot
// weights on e in slot order; out[rows] += w * expert(hidden[rows]).
#include <cuda_bf16.h>
#include <stdint.h>

#include "lynx_internal.cuh"

namespace lynx {

// K2: gather the dispatched token rows into the permuted buffer (expert
// segments, 16-row padded) that K3's TMA tensor map covers.  One 16-byte
// vector per thread; padding rows are zero.  The permutation itself was
// planned by K1 (plan_dispatch in select.cu).
__global__ void __launch_bounds__(256) gather_kernel(GatherArgs a) {
  griddep_launch_dependents();
  griddep_wait();
  const int rows = *a.n_rows;
  const int nvec = a.d >> 3;
  const uint4* src = reinterpret_cast<const uint4*>(a.hidden);
  uint4* dst = reinterpret_cast<uint4*>(a.x_perm);
  const int total = rows * nvec;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int r = i / nvec, v = i - r * nvec;
    const int t = a.perm_token[r];
    dst[i] = t >= 0 ? src[static_cast<size_t>(t) * nvec + v] : make_uint4(0, 0, 0, 0);
  }
}

cudaError_t launch_gather(const GatherArgs& a, int sm_count, cudaStream_t s) {
  const long total = static_cast<long>(a.rows_cap) * (a.d >> 3);
  long grid = (total + 255) / 256;
  if (grid > 4L * sm_count) grid = 4L * sm_count;
  if (grid < 1) grid = 1;
  return launch_pdl(gather_kernel, dim3(static_cast<unsigned>(grid)), dim3(256), 0, s, a);
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
