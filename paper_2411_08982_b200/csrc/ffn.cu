// ffn.cu -- K3: grouped expert FFN over the USED experts only, on the
// 5th-gen tensor cores (tcgen05.mma, accumulators in TMEM), operands staged
// by TMA into 128B-swizzled shared memory.
//
// Reference: forward_layer (simulator.py:86-113) calls expert_mlp
// (simulator.py:77-79) once per used expert on that expert's token rows.
// Here every used expert becomes a "segment" of <= 256 token rows (planned by
// K1, gathered by K2), and the whole layer's expert work is one persistent
// launch over a device-side queue of work units:
//
//   phase-0 unit (seg, mt):     D[128 x n] = W1[e][mt*128 : +128, :] . X_seg^T
//        SwiGLU: rows interleave gate/up in 16-row groups (lynx_pack_w13),
//        epilogue h = silu(gate) * up -> H[seg rows, 64 features] (bf16).
//        TANH2:  epilogue h = tanh(acc) -> H[seg rows, 128 features].
//   phase-1 unit (seg, mt, s):  D[128 x n] = W2[e][mt*128 : +128, K_s] . H_seg[:, K_s]^T
//        epilogue -> slot[s][seg rows][mt*128 : +128] (f32).  K4 sums the
//        slots in the fixed order 0..S-1 (bit-reproducible, no float
//        atomics) fused with the weighted combine.
//
// Swap-AB: weight rows are the MMA M (=128) dimension, a segment's tokens the
// MMA N dimension (16..256, rounded to 16), so decode streams each used
// expert's weights from HBM exactly once while the tiny activation tiles
// come from L2.  Units are dequeued from a device ticket counter in the order
// [all phase-0 units][all phase-1 units]; a phase-1 unit waits (acquire)
// until its segment's phase-0 tiles are published (release), which queue
// order makes ready by the time it is dequeued.  Split-K keeps phase-1 units
// at 512 KB so the dynamic queue balances the tail.
//
// Measured lessons kept in this design: the epilogue never runs
// latency-bound L2 traffic (split sums / combine done in the epilogue or by
// in-kernel reducer warps under a saturated HBM cost 1.5-2x: every dependent
// round trip waits behind ~20 MB of in-flight TMA loads), so the reduction
// lives in K4, after the stream.
//
// Warp roles (256 threads, one CTA per SM):
//   warp 0      TMA producer + unit scheduler (one elected lane)
//   warp 1      tcgen05.mma issuer (one lane)
//   warp 2      TMEM allocator
//   warps 4..7  epilogue: TMEM -> registers -> activation -> global
#include <cuda_bf16.h>
#include <stdint.h>
#include <stdlib.h>

#include "lynx_internal.cuh"
#include "ptx.cuh"

namespace lynx {

constexpr int kFfnThreads = 256;
// CTA-pair kernel: 12 warps, epilogue warps 4..11 = two per TMEM lane
// quarter, each draining half of a tile's token columns
constexpr int kPairThreads = 384;
constexpr int kPairEpiWarps = 8;
constexpr int kUnitRing = 4;
constexpr int kTileA = 128 * 64 * 2;  // 128 weight rows x 64 bf16 (one 128B-swizzled k block)
constexpr int kBoxB = 16 * 64 * 2;    // 16 token rows x 64 bf16
// Stage geometry is set at run time from the plan's widest segment: the
// launch's template BN (from T) sizes shared memory and TMEM, but a stage
// only needs 16 KB of weights + 2 KB per 16 rows of the widest segment, so a
// batch whose experts got few rows each runs more stages in the same bytes.
constexpr int kMaxStages = 12;
constexpr int kAccSlots = 4;  // TMEM accumulator slots of the CTA-pair kernel

struct Unit {
  int phase, seg, mt, split, kb0, kb1, expert, row0, n, nmma;
};

__device__ __forceinline__ bool decode_unit(const FfnParams& p, int nseg, int u, Unit& U) {
  if (u < 0) return false;
  const int nA = nseg * p.tiles1;
  int slot;
  if (u < nA) {
    U.phase = 0;
    slot = u / p.tiles1;
    U.mt = u - slot * p.tiles1;
    U.split = 0;
    U.kb0 = 0;
    U.kb1 = p.kb1;
  } else {
    const int v = u - nA;
    const int per = p.tiles2 * p.split2;
    U.phase = 1;
    slot = v / per;
    const int r = v - slot * per;
    U.mt = r / p.split2;
    U.split = r - U.mt * p.split2;
    U.kb0 = U.split * p.kb2_per;
    U.kb1 = min(p.kb2_total, U.kb0 + p.kb2_per);
  }
  // queue slots run the largest segments first (LPT), so the last units of
  // the launch -- and the phase-1 units waiting on the last phase-0 tiles --
  // are the cheapest ones
  U.seg = p.seg_order[slot];
  U.expert = p.seg_expert[U.seg];
  U.row0 = p.seg_row[U.seg];
  U.n = p.seg_count[U.seg];
  U.nmma = (U.n + 15) & ~15;
  return true;
}

__device__ __forceinline__ float silu_mul(float g, float u) { return g / (1.f + __expf(-g)) * u; }

// ------------------------------------------------ optional timeline trace
// Built only into the diagnostic library (-DLYNX_TRACE): one record per unit
// with globaltimer start and end, read back by lynx_debug_trace().  The
// production library compiles these to nothing.
#ifdef LYNX_TRACE
__device__ unsigned long long g_trace[4 * 65536];
__device__ unsigned int g_trace_n;
__device__ __forceinline__ void trace(int role, int id, uint64_t t0, uint64_t t1) {
  const unsigned i = atomicAdd(&g_trace_n, 1u);
  if (i < 65536) {
    g_trace[4 * i + 0] = (static_cast<unsigned long long>(blockIdx.x) << 32) | static_cast<unsigned>(role);
    g_trace[4 * i + 1] = static_cast<unsigned long long>(id);
    g_trace[4 * i + 2] = t0;
    g_trace[4 * i + 3] = t1;
  }
}
#define LYNX_TRACE_T0 const uint64_t trace_t0 = globaltimer()
#define LYNX_TRACE_REC(role, id) trace((role), (id), trace_t0, globaltimer())
#else
#define LYNX_TRACE_T0 (void)0
#define LYNX_TRACE_REC(role, id) (void)0
#endif

// Epilogue stores of one unit: this warp's 32 TMEM lanes (weight rows of
// 128-row tile `tile`) x the segment's tokens.  Phase 0 applies the
// activation and writes H (bf16); phase 1 writes the split-K partial (f32).
// `real` = false masks the stores of a padding tile (CTA-pair kernel).
__device__ __forceinline__ void epilogue_store(const FfnParams& p, const Unit& U, int tile, bool real, int q, int lane,
                                               uint32_t tb, int c_lo, int c_hi) {
  if (U.phase == 0) {
    __nv_bfloat16* H = reinterpret_cast<__nv_bfloat16*>(p.h);
    if (p.act == LYNX_ACT_SWIGLU) {
      // lanes 0-15: gate rows, lanes 16-31: up rows of the same 16 features
      const int f = tile * 64 + q * 16 + (lane & 15);
      const bool upper = lane >= 16;
      for (int c0 = c_lo; c0 < c_hi; c0 += 16) {
        uint32_t v[16];
        tmem_ld16(tb + c0, v);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float send = __uint_as_float(upper ? v[j] : v[8 + j]);
          const float recv = __shfl_xor_sync(0xffffffffu, send, 16);
          const float g = upper ? recv : __uint_as_float(v[j]);
          const float uu = upper ? __uint_as_float(v[8 + j]) : recv;
          const int tok = c0 + (upper ? 8 : 0) + j;
          if (real && tok < U.n && f < p.ff)
            H[static_cast<size_t>(U.row0 + tok) * p.ff + f] = __float2bfloat16_rn(silu_mul(g, uu));
        }
      }
    } else {
      const int f = tile * 128 + q * 32 + lane;
      for (int c0 = c_lo; c0 < c_hi; c0 += 16) {
        uint32_t v[16];
        tmem_ld16(tb + c0, v);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const int tok = c0 + j;
          if (real && tok < U.n && f < p.ff)
            H[static_cast<size_t>(U.row0 + tok) * p.ff + f] = __float2bfloat16_rn(tanhf(__uint_as_float(v[j])));
        }
      }
    }
  } else {
    // phase 1: split-K partial for 32 output columns -> slot[s]
    const int r = tile * 128 + q * 32 + lane;
    float* dst = p.partial + (static_cast<size_t>(U.split) * p.rows_cap + U.row0) * p.d + r;
    for (int c0 = c_lo; c0 < c_hi; c0 += 16) {
      uint32_t v[16];
      tmem_ld16(tb + c0, v);
      tmem_ld_wait();
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (c0 + j < U.n && r < p.d) dst[static_cast<size_t>(c0 + j) * p.d] = __uint_as_float(v[j]);
    }
  }
}

template <int BN, int STAGES>
__global__ void __launch_bounds__(kFfnThreads, 1) ffn_kernel(const __grid_constant__ FfnParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr int kRing = STAGES * (kTileA + BN * 128);
  constexpr uint32_t kTmemCols = 2 * BN;
  uint8_t* ring = smem;  // stage s: [weights 16 KB | token rows], s * stage_bytes
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kRing);
  uint64_t* empty = full + kMaxStages;
  uint64_t* tfull = empty + kMaxStages;
  uint64_t* tempty = tfull + 2;
  uint64_t* ufull = tempty + 2;
  uint64_t* uempty = ufull + kUnitRing;
  int* uring = reinterpret_cast<int*>(uempty + kUnitRing);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(uring + kUnitRing);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kMaxStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 4);
    }
    for (int i = 0; i < kUnitRing; ++i) {
      mbar_init(&ufull[i], 1);
      mbar_init(&uempty[i], 5);  // MMA lane + 4 epilogue warps
    }
    fence_mbar_init();
  }
  if (threadIdx.x == 32) {
    tma_prefetch_desc(&p.map_w1);
    tma_prefetch_desc(&p.map_w2);
    tma_prefetch_desc(&p.map_x);
    tma_prefetch_desc(&p.map_h);
  }
  warm_params(p);
  if (warp == 2) tmem_alloc(tmem_slot, kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  // Everything above overlapped the previous kernel (programmatic launch);
  // the dispatch plan and gathered rows are only read after this point.
  griddep_wait();
  // Let K4 (combine) launch now: its CTAs are small enough to sit beside this
  // one and wait in griddepcontrol.wait, so its launch latency leaves the
  // critical path.  Released only after our own wait, so K4 starts after the
  // plan's writer completed and may read the plan (token rows, weights)
  // before its own wait; the split-K slots it reads only after this grid.
  griddep_launch_dependents();
#ifdef LYNX_TRACE
  const uint64_t cta_t0 = globaltimer();
#endif
  const uint32_t tmem_base = *tmem_slot;
  const int nseg = *p.n_seg;
  const int width = p.max_rows ? min(BN, max(16, (*p.max_rows + 15) & ~15)) : BN;
  const int stage_bytes = kTileA + width * 128;
  const int nstages = min(kMaxStages, kRing / stage_bytes);
  const int total = nseg * (p.tiles1 + p.tiles2 * p.split2);

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------ TMA producer
      const uint64_t pol_w = policy_evict_first();
      const uint64_t pol_act = policy_evict_last();
      int stage = 0, slot = 0;
      uint32_t phase = 0, uphase = 0;
      // the first ticket is the CTA's own index (no atomic round trip before
      // the first load); the counter then hands out tickets from gridDim.x on
      bool first = true;
      while (true) {
        int u = first ? static_cast<int>(blockIdx.x) : atomicAdd(&p.counters[0], 1) + static_cast<int>(gridDim.x);
        first = false;
        if (u >= total) u = -1;
        mbar_wait(&uempty[slot], uphase ^ 1, 1);
        uring[slot] = u;
        mbar_arrive(&ufull[slot]);
        if (++slot == kUnitRing) {
          slot = 0;
          uphase ^= 1;
        }
        Unit U;
        if (!decode_unit(p, nseg, u, U)) break;
        const CUtensorMap* ma = U.phase == 0 ? &p.map_w1 : &p.map_w2;
        const CUtensorMap* mb = U.phase == 0 ? &p.map_x : &p.map_h;
        if (U.phase == 1) {
          LYNX_TRACE_T0;
          const int* done = p.counters + 1 + U.seg;
          Watchdog wd;
          while (ld_acquire_gpu(done) < 4 * p.tiles1) {
            __nanosleep(100);
            wd.tick(2);
          }
          fence_proxy_async();  // H was written by generic stores; TMA reads it
          LYNX_TRACE_REC(1, u);
        }
        const int nb = U.nmma >> 4;
        const uint32_t bytes = kTileA + nb * kBoxB;
        for (int kb = U.kb0; kb < U.kb1; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1, 3);
          mbar_expect_tx(&full[stage], bytes);
          uint8_t* sa = ring + stage * stage_bytes;
          tma_load_3d(sa, ma, &full[stage], kb * 64, U.mt * 128, U.expert, pol_w);
          for (int j = 0; j < nb; ++j)
            tma_load_2d(sa + kTileA + j * kBoxB, mb, &full[stage], kb * 64, U.row0 + 16 * j, pol_act);
          if (++stage == nstages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ------------------------------------------------ MMA issuer
      int stage = 0, slot = 0, acc = 0;
      uint32_t phase = 0, uphase = 0, aphase = 0;
      while (true) {
        mbar_wait(&ufull[slot], uphase, 4);
        const int u = uring[slot];
        mbar_arrive(&uempty[slot]);
        if (++slot == kUnitRing) {
          slot = 0;
          uphase ^= 1;
        }
        Unit U;
        if (!decode_unit(p, nseg, u, U)) break;
        const uint32_t idesc = idesc_bf16_f32(128, U.nmma);
        mbar_wait(&tempty[acc], aphase ^ 1, 5);
        LYNX_TRACE_T0;
        tc_fence_after();
        const uint32_t dt = tmem_base + static_cast<uint32_t>(acc * BN);
        for (int kb = U.kb0; kb < U.kb1; ++kb) {
          mbar_wait(&full[stage], phase, 6);
          tc_fence_after();
          const uint32_t sa = smem_u32(ring + stage * stage_bytes);
          const uint64_t ad = sdesc_kmajor_sw128(sa);
          const uint64_t bd = sdesc_kmajor_sw128(sa + kTileA);
#pragma unroll
          for (int k = 0; k < 4; ++k)  // 4 x K16 per 64-wide block; +32 B = +2 in the address field
            umma_bf16_ss(dt, ad + 2 * k, bd + 2 * k, idesc, (kb > U.kb0 || k > 0) ? 1u : 0u);
          umma_commit(&empty[stage]);
          if (++stage == nstages) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit(&tfull[acc]);
        LYNX_TRACE_REC(4, u);
        acc ^= 1;
        if (acc == 0) aphase ^= 1;
      }
    }
  } else if (warp >= 4) {
    // -------------------------------------------------- epilogue
    const int q = warp - 4;  // TMEM lane quarter (warp_id % 4)
    int slot = 0, acc = 0;
    uint32_t uphase = 0, aphase = 0;
    while (true) {
      mbar_wait(&ufull[slot], uphase, 7);
      const int u = uring[slot];
      __syncwarp();
      if (lane == 0) mbar_arrive(&uempty[slot]);
      if (++slot == kUnitRing) {
        slot = 0;
        uphase ^= 1;
      }
      Unit U;
      if (!decode_unit(p, nseg, u, U)) break;
      mbar_wait(&tfull[acc], aphase, 8);
      LYNX_TRACE_T0;
      tc_fence_after();
      const uint32_t tb = tmem_base + static_cast<uint32_t>(acc * BN) + (static_cast<uint32_t>(q * 32) << 16);
      epilogue_store(p, U, U.mt, true, q, lane, tb, 0, U.nmma);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
      if (U.phase == 0) {
        // publish this warp's slice of H to phase-1 consumers on other SMs
        __threadfence();
        fence_proxy_async();
        __syncwarp();
        if (lane == 0) red_release_gpu_add(p.counters + 1 + U.seg, 1);
      }
      if (lane == 0) LYNX_TRACE_REC(2, u);
      acc ^= 1;
      if (acc == 0) aphase ^= 1;
    }
  }
  tc_fence_before();
  __syncthreads();
#ifdef LYNX_TRACE
  if (threadIdx.x == 0) trace(5, nseg, cta_t0, globaltimer());
#endif
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, kTmemCols);
  }
}

// ------------------------------------------- CTA-pair variant (large T)
// The same unit queue, run by clusters of two CTAs on one TPC with
// tcgen05.mma.cta_group::2: a unit is 256 weight rows (CTA r stages rows
// 128r..128r+127 of it) against the segment's tokens, of which each CTA
// stages half.  The leader (rank 0) issues the M=256 MMA; every CTA's TMEM
// holds its 128 weight rows x all tokens, so the epilogue is per CTA as in
// the single-CTA kernel.  Per weight byte each SM stages half the token rows
// of the single-CTA kernel: at large batches the activation tiles are as
// large as the weight tiles and their L2 traffic caps the stream.
//
// Handshakes: the leader's producer takes the tickets and writes them into
// both CTAs' unit rings; both producers wait for their own ring stage to be
// empty (the MMA commit is multicast to both CTAs) and complete their bytes
// on the leader's full barrier; both CTAs' epilogues arrive on the leader's
// accumulator-empty and unit-empty barriers.
__device__ __forceinline__ bool decode_unit_pair(const FfnParams& p, int nseg, int u, int tp1, int tp2, Unit& U) {
  if (u < 0) return false;
  const int nA = nseg * tp1;
  int slot;
  if (u < nA) {
    U.phase = 0;
    slot = u / tp1;
    U.mt = u - slot * tp1;  // pair tile: CTA r takes 128-row tile 2 * mt + r
    U.split = 0;
    U.kb0 = 0;
    U.kb1 = p.kb1;
  } else {
    const int v = u - nA;
    const int per = tp2 * p.split2;
    U.phase = 1;
    slot = v / per;
    const int r = v - slot * per;
    U.mt = r / p.split2;
    U.split = r - U.mt * p.split2;
    U.kb0 = U.split * p.kb2_per;
    U.kb1 = min(p.kb2_total, U.kb0 + p.kb2_per);
  }
  U.seg = p.seg_order[slot];
  U.expert = p.seg_expert[U.seg];
  U.row0 = p.seg_row[U.seg];
  U.n = p.seg_count[U.seg];
  U.nmma = (U.n + 31) & ~31;  // even split of the token rows over the pair
  return true;
}

// Ring bytes of the CTA-pair kernel: STAGES stages of the widest stage
// (MT = 1), or the shared-memory budget carved at run time (MT = 2: 4 stages
// at 256 token rows, 5 at 128, 6 at 64).
constexpr int pair_ring_bytes(int BN, int STAGES, int MT) {
  return MT == 1 ? STAGES * (kTileA + BN * 64) : 216 * 1024;
}

// MT weight tiles per CTA per stage: a pair unit covers 256 * MT weight rows
// (MMA j takes rows 256 j + 128 r .. of the unit on CTA r), all against the
// same activation tile.  Each SM then pulls 1/MT of the activation bytes per
// weight byte through L2: at large batches the L2 -> SM traffic (weights +
// activations) is what caps the weight stream, not HBM.  The MT accumulators
// of a unit take MT * N TMEM columns; they are double-buffered when two
// units' worth fit (N <= 256 / MT), else the epilogue drains one unit while
// the MMA waits for it.
template <int BN, int STAGES, int MT>
__global__ void __launch_bounds__(kPairThreads, 1) ffn_pair_kernel(const __grid_constant__ FfnParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr int kRing = pair_ring_bytes(BN, STAGES, MT);
  constexpr uint32_t kTmemCols = 512;
  static_assert(MT * BN <= 512, "a unit's accumulators must fit TMEM");
  uint8_t* ring = smem;  // stage s: [MT weight tiles x 16 KB | this CTA's half of the token rows]
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kRing);
  uint64_t* empty = full + kMaxStages;
  uint64_t* tfull = empty + kMaxStages;  // per accumulator slot (kAccSlots)
  uint64_t* tempty = tfull + kAccSlots;
  uint64_t* ufull = tempty + kAccSlots;
  uint64_t* uempty = ufull + kUnitRing;
  int* uring = reinterpret_cast<int*>(uempty + kUnitRing);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(uring + kUnitRing);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kMaxStages; ++s) {
      mbar_init(&full[s], 1);   // leader: its producer's arrive + both CTAs' bytes
      mbar_init(&empty[s], 1);  // multicast MMA commit
    }
    for (int i = 0; i < kAccSlots; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 2 * kPairEpiWarps);  // leader: the epilogue warps of both CTAs
    }
    for (int i = 0; i < kUnitRing; ++i) {
      mbar_init(&ufull[i], 1);
      mbar_init(&uempty[i], 2 + 2 * kPairEpiWarps);  // leader: MMA + epilogue warps, peer: producer + epilogue warps
    }
    fence_mbar_init();
  }
  if (threadIdx.x == 32) {
    tma_prefetch_desc(&p.map_w1);
    tma_prefetch_desc(&p.map_w2);
    tma_prefetch_desc(&p.map_x);
    tma_prefetch_desc(&p.map_h);
  }
  warm_params(p);
  if (warp == 2) tmem_alloc_pair(tmem_slot, kTmemCols);
  tc_fence_before();
  cluster_sync();  // both CTAs' barriers initialised and TMEM allocated
  tc_fence_after();
  griddep_wait();
  griddep_launch_dependents();  // K4 may launch now (see ffn_kernel)
  const uint32_t tmem_base = *tmem_slot;
  const int nseg = *p.n_seg;
  const int tp1 = (p.tiles1 + 2 * MT - 1) / (2 * MT), tp2 = (p.tiles2 + 2 * MT - 1) / (2 * MT);
  const int total = nseg * (tp1 + tp2 * p.split2);
  const int width = p.max_rows ? min(BN, max(32, (*p.max_rows + 31) & ~31)) : BN;
  const int stage_bytes = MT * kTileA + (width >> 1) * 128;
  const int nstages = min(kMaxStages, kRing / stage_bytes);
  // TMEM as a ring of `nslot` accumulator slots of `width` columns; unit u's
  // tile m accumulates in slot (MT u + m) % nslot.  The epilogue frees a
  // slot as soon as it has drained that tile, so the next unit's MMAs wait
  // only for the slots they reuse: with 3 slots (width <= 170) the second
  // tile's drain overlaps the next unit instead of stalling it.
  const int nslot = min(kAccSlots, static_cast<int>(kTmemCols) / width);
  const uint32_t peer_ufull = mapa_shared(ufull, 1), peer_uring = mapa_shared(uring, 1);
  const uint32_t lead_uempty = mapa_shared(uempty, 0), lead_tempty = mapa_shared(tempty, 0);

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------ TMA producers (both CTAs)
      const uint64_t pol_w = policy_evict_first();
      const uint64_t pol_act = policy_evict_last();
      int stage = 0, slot = 0;
      uint32_t phase = 0, uphase = 0;
      bool first = true;  // first ticket = the pair's index, as in ffn_kernel
      while (true) {
        int u;
        if (leader) {
          const int npairs = static_cast<int>(gridDim.x) / 2;
          u = first ? static_cast<int>(blockIdx.x) / 2 : atomicAdd(&p.counters[0], 1) + npairs;
          first = false;
          if (u >= total) u = -1;
          mbar_wait(&uempty[slot], uphase ^ 1, 1);
          uring[slot] = u;
          st_cluster_u32(peer_uring + 4 * slot, static_cast<uint32_t>(u));
          mbar_arrive(&ufull[slot]);
          mbar_arrive_cluster(peer_ufull + 8 * slot);
        } else {
          mbar_wait_cluster(&ufull[slot], uphase, 1);
          u = uring[slot];
          mbar_arrive_cluster(lead_uempty + 8 * slot);
        }
        if (++slot == kUnitRing) {
          slot = 0;
          uphase ^= 1;
        }
        Unit U;
        if (!decode_unit_pair(p, nseg, u, tp1, tp2, U)) break;
        const CUtensorMap* ma = U.phase == 0 ? &p.map_w1 : &p.map_w2;
        const CUtensorMap* mb = U.phase == 0 ? &p.map_x : &p.map_h;
        if (U.phase == 1) {
          const int* done = p.counters + 1 + U.seg;
          Watchdog wd;
          while (ld_acquire_gpu(done) < kPairEpiWarps * p.tiles1) {
            __nanosleep(100);
            wd.tick(2);
          }
          fence_proxy_async();  // H was written by generic stores; TMA reads it
        }
        const int half = U.nmma >> 1;  // token rows per CTA
        const int nb = half >> 4;
        const uint32_t bytes = 2 * (MT * kTileA + nb * kBoxB);  // both CTAs' bytes land on the leader's barrier
        const int wrow = (2 * MT * U.mt + static_cast<int>(rank)) * 128;
        const int trow = U.row0 + static_cast<int>(rank) * half;
        for (int kb = U.kb0; kb < U.kb1; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1, 3);
          if (leader) mbar_expect_tx(&full[stage], bytes);
          uint8_t* sa = ring + stage * stage_bytes;
#pragma unroll
          for (int m = 0; m < MT; ++m)
            tma_load_3d_pair(sa + m * kTileA, ma, &full[stage], kb * 64, wrow + 256 * m, U.expert, pol_w);
          for (int j = 0; j < nb; ++j)
            tma_load_2d_pair(sa + MT * kTileA + j * kBoxB, mb, &full[stage], kb * 64, trow + 16 * j, pol_act);
          if (++stage == nstages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && leader) {
      // ------------------------------------------------ MMA issuer (leader only)
      int stage = 0, slot = 0, acc = 0;  // acc: the next accumulator slot
      uint32_t phase = 0, uphase = 0, aphase = 0;  // aphase: parity bit per accumulator slot
      while (true) {
        mbar_wait(&ufull[slot], uphase, 4);
        const int u = uring[slot];
        mbar_arrive(&uempty[slot]);
        if (++slot == kUnitRing) {
          slot = 0;
          uphase ^= 1;
        }
        Unit U;
        if (!decode_unit_pair(p, nseg, u, tp1, tp2, U)) break;
        const uint32_t idesc = idesc_bf16_f32(256, U.nmma);
        int as[MT];
#pragma unroll
        for (int m = 0; m < MT; ++m) {
          as[m] = acc;
          mbar_wait_cluster(&tempty[acc], ((aphase >> acc) & 1u) ^ 1u, 5);
          if (++acc == nslot) acc = 0;
        }
        tc_fence_after();
        for (int kb = U.kb0; kb < U.kb1; ++kb) {
          mbar_wait(&full[stage], phase, 6);
          tc_fence_after();
          const uint32_t sa = smem_u32(ring + stage * stage_bytes);
          const uint64_t bd = sdesc_kmajor_sw128(sa + MT * kTileA);
#pragma unroll
          for (int m = 0; m < MT; ++m) {
            const uint64_t ad = sdesc_kmajor_sw128(sa + m * kTileA);
            const uint32_t dt = tmem_base + static_cast<uint32_t>(as[m] * width);
#pragma unroll
            for (int k = 0; k < 4; ++k)  // 4 x K16 per 64-wide block; +32 B = +2 in the address field
              umma_bf16_ss_pair(dt, ad + 2 * k, bd + 2 * k, idesc, (kb > U.kb0 || k > 0) ? 1u : 0u);
          }
          umma_commit_pair(&empty[stage]);
          if (++stage == nstages) {
            stage = 0;
            phase ^= 1;
          }
        }
#pragma unroll
        for (int m = 0; m < MT; ++m) {
          umma_commit_pair(&tfull[as[m]]);
          aphase ^= 1u << as[m];
        }
      }
    }
  } else if (warp >= 4) {
    // -------------------------------------------------- epilogue (both CTAs)
    const int q = (warp - 4) & 3;  // TMEM lane quarter (warp_id % 4)
    const int half = (warp - 4) >> 2;  // which half of the token columns
    int slot = 0, acc = 0;
    uint32_t uphase = 0, aphase = 0;
    while (true) {
      if (leader) mbar_wait(&ufull[slot], uphase, 7);
      else mbar_wait_cluster(&ufull[slot], uphase, 7);
      const int u = uring[slot];
      __syncwarp();
      if (lane == 0) {
        if (leader) mbar_arrive(&uempty[slot]);
        else mbar_arrive_cluster(lead_uempty + 8 * slot);
      }
      if (++slot == kUnitRing) {
        slot = 0;
        uphase ^= 1;
      }
      Unit U;
      if (!decode_unit_pair(p, nseg, u, tp1, tp2, U)) break;
      int published = 0;
      LYNX_TRACE_T0;
#pragma unroll 1
      for (int m = 0; m < MT; ++m) {
        mbar_wait(&tfull[acc], (aphase >> acc) & 1u, 8);
        tc_fence_after();
        const int tile = 2 * (MT * U.mt + m) + static_cast<int>(rank);
        const uint32_t tb = tmem_base + static_cast<uint32_t>(acc * width) + (static_cast<uint32_t>(q * 32) << 16);
        const bool real = tile < (U.phase == 0 ? p.tiles1 : p.tiles2);  // tiles past the end are padding
        const int hc = U.nmma >> 1;  // nmma is a multiple of 32: halves of 16-column steps
        epilogue_store(p, U, tile, real, q, lane, tb, half * hc, (half + 1) * hc);
        published += real ? 1 : 0;
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {  // this slot is free for the next unit's MMAs
          if (leader) mbar_arrive(&tempty[acc]);
          else mbar_arrive_cluster(lead_tempty + 8 * acc);
        }
        aphase ^= 1u << acc;
        if (++acc == nslot) acc = 0;
      }
      if (U.phase == 0 && published) {  // publish this warp's slices of H to phase-1 consumers on other SMs
        __threadfence();
        fence_proxy_async();
        __syncwarp();
        if (lane == 0) red_release_gpu_add(p.counters + 1 + U.seg, published);
      }
      if (threadIdx.x == 128) LYNX_TRACE_REC(4, u);  // unit drained (trace build: per-CTA unit timeline)
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // the peer's TMEM and barriers outlive every MMA / remote arrive
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc_pair(tmem_base, kTmemCols);
  }
}

template <int BN, int STAGES, int MT>
static cudaError_t launch_ffn_pair_t(const FfnParams& p, int sm_count, cudaStream_t s) {
  constexpr size_t smem = 1024 + pair_ring_bytes(BN, STAGES, MT) + (2 * kMaxStages + 2 * kAccSlots + 2 * kUnitRing) * 8 +
                          kUnitRing * 4 + 16;
  static_assert(smem <= 227 * 1024, "shared memory budget");
  static int configured_device = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (configured_device != dev) {
    cudaError_t e = cudaFuncSetAttribute(ffn_pair_kernel<BN, STAGES, MT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    configured_device = dev;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(sm_count & ~1);
  cfg.blockDim = dim3(kPairThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = 2;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, ffn_pair_kernel<BN, STAGES, MT>, p);
}

// The CTA pair halves each SM's activation tiles but couples two SMs per
// stage.  Measured on B200 (K3, CUDA events): it wins once the segments are
// wide -- Mixtral-8x22B at T=256 (~128 rows per used expert) 638 -> 520 us,
// T=128 (~64 rows) 478 -> 437 us, Mixtral-8x7B without Lynx at T=256 (~64
// rows) 549 -> 515 us -- and loses on narrow ones (T=128 without Lynx, ~32
// rows: 468 -> 474 us; DeepSeek-MoE C4, ~37 rows: 76.5 -> 83.2 us).  The host
// only knows the expected rows per used expert, so that picks the kernel.
// LYNX_FFN_PAIR=0/1 forces either kernel (A/B switch); unset or "auto": by rows.
bool ffn_use_pair(int bn, int rows_hint) {
  static int force = -2;
  if (force == -2) {
    const char* e = getenv("LYNX_FFN_PAIR");
    force = (e && e[0] == '0' && !e[1]) ? 0 : (e && e[0] == '1' && !e[1]) ? 1 : -1;
  }
  if (bn < 128) return false;  // T <= 64: decode batches stay on the single-CTA kernel
  if (force >= 0) return force == 1;
  return rows_hint >= 64;
}

template <int BN, int STAGES>
static cudaError_t launch_ffn_t(const FfnParams& p, int sm_count, cudaStream_t s) {
  constexpr size_t smem =
      1024 + STAGES * (kTileA + BN * 128) + (2 * kMaxStages + 4 + 2 * kUnitRing) * 8 + kUnitRing * 4 + 16;
  static_assert(smem <= 227 * 1024, "shared memory budget");
  static int configured_device = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (configured_device != dev) {
    cudaError_t e = cudaFuncSetAttribute(ffn_kernel<BN, STAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    configured_device = dev;
  }
  return launch_pdl(ffn_kernel<BN, STAGES>, dim3(sm_count), dim3(kFfnThreads), smem, s, p);
}

// Weight tiles per CTA per stage of the CTA-pair kernel (LYNX_FFN_MT=1/2 A/B switch).
static int pair_mt() {
  static int mt = 0;
  if (!mt) {
    const char* e = getenv("LYNX_FFN_MT");
    mt = (e && e[0] == '1' && !e[1]) ? 1 : 2;
  }
  return mt;
}

cudaError_t launch_ffn(const FfnParams& p, int bn, int rows_hint, int sm_count, cudaStream_t s) {
  const bool pair = ffn_use_pair(bn, rows_hint);
  switch (bn) {
    case 32:
      return launch_ffn_t<32, 10>(p, sm_count, s);
    case 64:
      return launch_ffn_t<64, 9>(p, sm_count, s);
    case 128:
      if (!pair) return launch_ffn_t<128, 7>(p, sm_count, s);
      return pair_mt() == 2 ? launch_ffn_pair_t<128, 5, 2>(p, sm_count, s) : launch_ffn_pair_t<128, 9, 1>(p, sm_count, s);
    default:
      if (!pair) return launch_ffn_t<256, 4>(p, sm_count, s);
      return pair_mt() == 2 ? launch_ffn_pair_t<256, 4, 2>(p, sm_count, s) : launch_ffn_pair_t<256, 7, 1>(p, sm_count, s);
  }
}

}  // namespace lynx

#ifdef LYNX_TRACE
// Diagnostic library only: copy out and reset the timeline trace.
extern "C" int lynx_debug_trace(unsigned long long* host, int max_records) {
  unsigned n = 0;
  if (cudaMemcpyFromSymbol(&n, lynx::g_trace_n, sizeof(n)) != cudaSuccess) return -1;
  if (n > 65536u) n = 65536u;
  if (static_cast<int>(n) > max_records) n = static_cast<unsigned>(max_records);
  if (n && cudaMemcpyFromSymbol(host, lynx::g_trace, n * 4 * sizeof(unsigned long long)) != cudaSuccess) return -1;
  unsigned z = 0;
  cudaMemcpyToSymbol(lynx::g_trace_n, &z, sizeof(z));
  return static_cast<int>(n);
}
#endif
