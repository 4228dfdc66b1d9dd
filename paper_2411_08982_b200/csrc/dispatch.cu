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
#include "p2p.cuh"

namespace lynx {

// K2: gather the dispatched token rows into the permuted buffer (expert
// segments, 16-row padded) that K3's TMA tensor map covers.  One 16-byte
// vector per thread; padding rows are zero.  The permutation itself was
// planned by K1 (plan_dispatch in select.cu).
__global__ void __launch_bounds__(256) gather_kernel(const __grid_constant__ GatherArgs a) {
  griddep_launch_dependents();
  warm_params(a);
  griddep_wait();
  if (a.ep.enabled) {  // peer-memory EP: every rank's dispatched rows have landed
    if (threadIdx.x == 0) wait_peers(a.ep.P, a.ep.kind, *a.ep.P.epoch + 1);
    __syncthreads();
  }
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

// ------------------------------------------------------------------- K4
// out[t] = hidden[t] + sum_j w_tj * (slot0 + slot1 + ... + slot_{S-1})[row_tj],
// j over the token's experts ascending and s in order: the reference's
// accumulation order (simulator.py:101-112) with a fixed split-K order, so
// the layer output is bit-reproducible.  One CTA per (token, 512 columns);
// the token's rows are staged once, then the slot loads issue in groups.
// SPLIT = the split-K slot count when it is 1 or 2 (every BASELINE shape),
// 0 = any: with a compile-time count the k x SPLIT loads are straight-line
// (no per-entry index arithmetic) and all issue before the first use.
template <int SPLIT>
__global__ void __launch_bounds__(128, SPLIT == 1 ? 6 : 10) combine_kernel(const __grid_constant__ CombineArgs a) {
  constexpr int kMaxEntries = LYNX_MAX_TOPK + LYNX_MAX_SHARED;
  __shared__ int s_rows[kMaxEntries];
  __shared__ float s_w[kMaxEntries];
  griddep_launch_dependents();
  warm_params(a);
  // K3 releases this launch only after its own wait: the plan (token rows,
  // weights) and the residual are complete, so they load before our wait --
  // only the split-K slots need K3 to have finished
  const int t = blockIdx.y;
  if (threadIdx.x < a.k) {
    s_rows[threadIdx.x] = a.tok_rows[t * a.k + threadIdx.x];
    s_w[threadIdx.x] = a.tok_weight[t * a.k + threadIdx.x];
  }
  const int c0 = (blockIdx.x * blockDim.x + threadIdx.x) * 4;
  const bool live = c0 < a.d;
  const int c = live ? c0 : 0;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  if (a.hidden) {
    const __nv_bfloat162* h =
        reinterpret_cast<const __nv_bfloat162*>(a.hidden + static_cast<size_t>(t) * a.d + c);
    const float2 h0 = __bfloat1622float2(h[0]), h1 = __bfloat1622float2(h[1]);
    acc = make_float4(h0.x, h0.y, h1.x, h1.y);
  }
  __syncthreads();
  griddep_wait();  // partial slots come from K3
  auto slot = [&](int s, int row) {
    return *reinterpret_cast<const float4*>(a.partial + s * a.slot_stride + static_cast<size_t>(row) * a.d + c);
  };
  if (SPLIT > 0) {
    // entries in groups whose loads issue together, with registers low enough
    // for high occupancy (the slots come from HBM: occupancy is the MLP)
    constexpr int S = SPLIT > 0 ? SPLIT : 1;
    // one split slot: every entry's load in flight at once (C4: 8 rows);
    // two: four entries (eight loads) per group, registers for 10 CTAs per SM
    constexpr int G = S == 1 ? kMaxEntries : 4;
#pragma unroll 1
    for (int j0 = 0; j0 < a.k; j0 += G) {
      float4 v[G][S];
#pragma unroll
      for (int g = 0; g < G; ++g)
#pragma unroll
        for (int s = 0; s < S; ++s)
          if (j0 + g < a.k && s_rows[j0 + g] >= 0) v[g][s] = slot(s, s_rows[j0 + g]);
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const int j = j0 + g;
        if (j < a.k && s_rows[j] >= 0) {
          float4 y = v[g][0];
#pragma unroll
          for (int s = 1; s < S; ++s) {
            y.x += v[g][s].x;
            y.y += v[g][s].y;
            y.z += v[g][s].z;
            y.w += v[g][s].w;
          }
          const float w = s_w[j];
          acc.x += w * y.x;
          acc.y += w * y.y;
          acc.z += w * y.z;
          acc.w += w * y.w;
        }
      }
    }
  } else {
    for (int j = 0; j < a.k; ++j) {
      const int row = s_rows[j];
      if (row < 0) continue;
      float4 y = slot(0, row);
      for (int s = 1; s < a.split2; ++s) {
        const float4 u = slot(s, row);
        y.x += u.x;
        y.y += u.y;
        y.z += u.z;
        y.w += u.w;
      }
      const float w = s_w[j];
      acc.x += w * y.x;
      acc.y += w * y.y;
      acc.z += w * y.z;
      acc.w += w * y.w;
    }
  }
  if (a.discard_partials) {
    // this warp's 8-thread groups have consumed their 128-byte lines of every
    // slot row: drop them from L2 unwritten (K4 is their only reader)
    __syncwarp();
    if (live && (threadIdx.x & 7) == 0)
      for (int j = 0; j < a.k; ++j) {
        const int row = s_rows[j];
        if (row < 0) continue;
        for (int s2 = 0; s2 < a.split2; ++s2)
          asm volatile("discard.global.L2 [%0], 128;" ::"l"(a.partial + s2 * a.slot_stride +
                                                             static_cast<size_t>(row) * a.d + c)
                       : "memory");
      }
  }
  const size_t o = static_cast<size_t>(t) * a.d + c;
  if (a.peer_mode) {
    // the token's owner gathers every rank's partial in slot [rank]
    const int Tl = a.peers.tokens_per_rank;
    float* dst = a.peers.back[t / Tl] + (static_cast<size_t>(a.peers.rank) * Tl + t % Tl) * a.d + c;
    if (live) *reinterpret_cast<float4*>(dst) = acc;
    if (last_cta(a.peers.counters + 1)) {
      if (threadIdx.x == 0) signal_peers(a.peers, kSigBack, *a.peers.epoch + 1);
    }
  } else if (!live) {
  } else if (a.out_f32) {
    *reinterpret_cast<float4*>(a.out_f32 + o) = acc;
  } else {
    __nv_bfloat162* out = reinterpret_cast<__nv_bfloat162*>(a.out_bf16 + o);
    out[0] = __floats2bfloat162_rn(acc.x, acc.y);
    out[1] = __floats2bfloat162_rn(acc.z, acc.w);
  }
  if (a.discard_rows) {
    // K3 is complete: the H rows and gathered token rows it used are dead --
    // drop them from L2 unwritten (the plan's row count, not the capacity)
    const size_t rows = static_cast<size_t>(*a.discard_rows);
    const size_t nthr = static_cast<size_t>(gridDim.x) * gridDim.y * blockDim.x;
    const size_t me = (static_cast<size_t>(blockIdx.y) * gridDim.x + blockIdx.x) * blockDim.x + threadIdx.x;
#pragma unroll
    for (int r = 0; r < 2; ++r)
      for (size_t i = me; i < rows * a.discard_row_bytes[r] / 128; i += nthr)
        asm volatile("discard.global.L2 [%0], 128;" ::"l"(a.discard_base[r] + i * 128) : "memory");
  }
}

cudaError_t launch_combine(const CombineArgs& a, cudaStream_t s) {
  const dim3 grid((a.d + 511) / 512, a.T);
  if (a.split2 == 1) return launch_pdl(combine_kernel<1>, grid, dim3(128), 0, s, a);
  if (a.split2 == 2) return launch_pdl(combine_kernel<2>, grid, dim3(128), 0, s, a);
  return launch_pdl(combine_kernel<0>, grid, dim3(128), 0, s, a);
}

// ------------------------------------------------------------ trace ring
// Copy one layer's routing event into the device ring at slot (*pos) % cap.
struct TraceAppendArgs {
  lynx_trace_ring_t r;
  const int32_t* pos;
  int layer;
  lynx_selection_t sel;
};

__global__ void __launch_bounds__(256) trace_append_kernel(const __grid_constant__ TraceAppendArgs a) {
  griddep_launch_dependents();
  griddep_wait();
  const lynx_trace_ring_t& r = a.r;
  const int p = *a.pos;
  const int slot = p % r.capacity;
  const size_t ev = static_cast<size_t>(slot) * r.num_layers + a.layer;
  const int T = r.T, k = r.k, N = r.N;
  for (int i = threadIdx.x; i < T * k; i += blockDim.x) {
    r.original[ev * T * k + i] = a.sel.expert_ids[i];
    r.assigned[ev * T * k + i] = a.sel.assigned[i];
    r.weights[ev * T * k + i] = a.sel.weights[i];
  }
  for (int t = threadIdx.x; t < T; t += blockDim.x) {
    double m = a.sel.full_probs[static_cast<size_t>(t) * N];
    for (int e = 1; e < N; ++e) m = fmax(m, a.sel.full_probs[static_cast<size_t>(t) * N + e]);
    r.conf[ev * T + t] = m;
    r.important[ev * T + t] = a.sel.important ? a.sel.important[t] : 0;
  }
  for (int e = threadIdx.x; e < N; e += blockDim.x) r.retained[ev * N + e] = a.sel.retained[e];
  if (threadIdx.x == 0) {
    r.flags[ev] = a.sel.flags[0];
    if (a.layer == 0) r.positions[slot] = p;
  }
}

cudaError_t launch_trace_append(const lynx_trace_ring_t& r, const int32_t* pos, int layer,
                                const lynx_selection_t& sel, cudaStream_t s) {
  TraceAppendArgs a;
  a.r = r;
  a.pos = pos;
  a.layer = layer;
  a.sel = sel;
  return launch_pdl(trace_append_kernel, dim3(1), dim3(256), 0, s, a);
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
