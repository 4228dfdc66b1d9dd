// p2p.cuh -- peer-memory signalling for the fused expert-parallel path
// (ep_p2p.cu, and K4's peer mode in dispatch.cu).  See ep_p2p.cu.
#pragma once

#include <stdint.h>

#include "lynx_internal.cuh"
#include "ptx.cuh"

namespace lynx {

enum { kSigLogits = 0, kSigDispatch = 1, kSigBack = 2 };

__device__ __forceinline__ void st_release_sys(int32_t* p, int v) {
  asm volatile("st.release.sys.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_acquire_sys(const int32_t* p) {
  int v;
  asm volatile("ld.acquire.sys.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Tell every peer that this rank's `kind` data for `epoch` is in place.
__device__ __forceinline__ void signal_peers(const lynx_ep_peers_t& P, int kind, int epoch) {
  __threadfence_system();
  for (int p = 0; p < P.world_size; ++p) st_release_sys(P.flags[p] + kind * P.world_size + P.rank, epoch);
}

// Last-arriving CTA of a grid: every CTA fences its (peer) stores and counts
// itself in; returns true on the last one, which also re-arms the counter.
// Must be reached by every thread of every CTA.
__device__ __forceinline__ bool last_cta(int32_t* counter) {
  __shared__ int s_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    const int total = gridDim.x * gridDim.y * gridDim.z;
    const int t = atomicAdd(counter, 1);
    s_last = t == total - 1;
    if (s_last) *counter = 0;  // the next launch is stream-ordered after this one
  }
  __syncthreads();
  return s_last;
}

// Spin (one thread) until every peer has signalled `kind` for `epoch`.
__device__ __forceinline__ void wait_peers(const lynx_ep_peers_t& P, int kind, int epoch) {
  const int32_t* f = P.flags_local + kind * P.world_size;
  Watchdog wd;
  for (int p = 0; p < P.world_size; ++p)
    while (ld_acquire_sys(f + p) < epoch) {
      __nanosleep(64);
      wd.tick(40 + kind);
    }
}

}  // namespace lynx
