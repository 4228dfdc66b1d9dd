// ep_p2p.cu -- expert parallelism over NVLink peer memory:
// the logits all-gather, the token dispatch and the partial-sum return are
// plain stores into the peers' symmetric buffers issued by the kernels that
// produce the data (K0, the dispatch kernel, K4), each followed by one
// release-signal per peer; the consuming kernels (K1, K2, the combine)
// acquire-wait on those signals at their start.  No NCCL call, no staging
// copy, no extra launch: the "collective" is fused into the producer and
// consumer kernels.
//
// Buffers (identical layout on every rank, peers reach them through the
// pointer arrays of lynx_ep_peers_t):
//   logits[G*Tl, N]  f64   rows r*Tl.. written by rank r (all-gather)
//   recv  [G*Tl, d]  bf16  rows r*Tl.. = rank r's tokens this rank needs
//   back  [G*Tl, d]  f32   rows r*Tl.. = rank r's partial sums for this
//                          rank's tokens (zeros where r has no expert)
//   flags [3*G]      int32 signal slot (kind, source rank) = epoch
// A layer call uses epoch = *epoch + 1; the combine's last CTA advances
// *epoch, so slots never need resetting and a captured graph replays.
#include <cuda_bf16.h>
#include <stdint.h>

#include "p2p.cuh"

namespace lynx {

// route: K0 itself stores its logits rows into every rank and signals
// (router_logits_kernel with an EpLink); K1 waits for them at its start.

// ------------------------------------------------------------- dispatch
// Row i of this rank goes to peer p's recv buffer (rows rank*Tl + i) iff
// global token rank*Tl + i has a slot on one of p's experts.  One CTA per
// (row, peer); the last CTA signals.
__global__ void __launch_bounds__(128) ep_dispatch_kernel(const __grid_constant__ lynx_ep_peers_t P,
                                                          const uint16_t* hidden_local, const int32_t* assigned,
                                                          int k, int N, int d) {
  griddep_launch_dependents();
  griddep_wait();
  const int i = blockIdx.x, p = blockIdx.y;
  const int Tl = P.tokens_per_rank, G = P.world_size;
  const int t = P.rank * Tl + i, per = N / G;
  bool need = false;
  for (int c = 0; c < k; ++c) {
    const int e = assigned[t * k + c];
    need |= e >= 0 && e / per == p;
  }
  if (need) {
    const uint4* src = reinterpret_cast<const uint4*>(hidden_local + static_cast<size_t>(i) * d);
    uint4* dst = reinterpret_cast<uint4*>(P.recv[p] + static_cast<size_t>(t) * d);
    for (int v = threadIdx.x; v < (d >> 3); v += blockDim.x) dst[v] = src[v];
  }
  if (last_cta(P.counters + 0)) {
    if (threadIdx.x == 0) signal_peers(P, kSigDispatch, *P.epoch + 1);
  }
}

// -------------------------------------------------------------- combine
// out[i] = hidden[i] + sum_p back[p*Tl + i], p ascending (= experts
// ascending); waits for every peer's return first; the last CTA advances
// the epoch.
__global__ void __launch_bounds__(256) ep_p2p_combine_kernel(const __grid_constant__ lynx_ep_peers_t P,
                                                             const uint16_t* hidden_local, int d, uint16_t* out) {
  griddep_launch_dependents();
  griddep_wait();
  __shared__ int s_epoch;
  if (threadIdx.x == 0) {
    s_epoch = *P.epoch + 1;
    wait_peers(P, kSigBack, s_epoch);
  }
  __syncthreads();
  const int i = blockIdx.x, Tl = P.tokens_per_rank;
  const float* back = P.back_local;
  for (int c = threadIdx.x * 2; c < d; c += blockDim.x * 2) {
    const float2 h = __bfloat1622float2(
        *reinterpret_cast<const __nv_bfloat162*>(hidden_local + static_cast<size_t>(i) * d + c));
    float sx = 0.f, sy = 0.f;
    for (int p = 0; p < P.world_size; ++p) {
      const float2 v = *reinterpret_cast<const float2*>(back + (static_cast<size_t>(p) * Tl + i) * d + c);
      sx += v.x;
      sy += v.y;
    }
    *reinterpret_cast<__nv_bfloat162*>(out + static_cast<size_t>(i) * d + c) =
        __floats2bfloat162_rn(h.x + sx, h.y + sy);
  }
  if (last_cta(P.counters + 2)) {
    if (threadIdx.x == 0) *P.epoch = s_epoch;
  }
}

cudaError_t launch_ep_dispatch(const lynx_ep_peers_t& P, const uint16_t* hidden_local, const int32_t* assigned, int k,
                               int N, int d, cudaStream_t s) {
  return launch_pdl(ep_dispatch_kernel, dim3(P.tokens_per_rank, P.world_size), dim3(128), 0, s, P, hidden_local,
                    assigned, k, N, d);
}
cudaError_t launch_ep_p2p_combine(const lynx_ep_peers_t& P, const uint16_t* hidden_local, int d, uint16_t* out,
                                  cudaStream_t s) {
  return launch_pdl(ep_p2p_combine_kernel, dim3(P.tokens_per_rank), dim3(256), 0, s, P, hidden_local, d, out);
}

}  // namespace lynx
