// ffn.cu -- K3: grouped expert FFN over the USED experts only, on the
// 5th-gen tensor cores (tcgen05.mma, accumulators in TMEM), operands staged
// by TMA into 128B-swizzled shared memory.
//
// Reference: forward_layer (simulator.py:86-113) calls expert_mlp
// (simulator.py:77-79) once per used expert on that expert's token rows.
// Here every used expert becomes a "segment" of <= 256 token rows (built by
// K2), and the whole layer's expert work is one persistent launch:
//
//   phase-0 unit (seg, mt):       D[128 x n] = W1[e][mt*128 : +128, :] . X_seg^T
//        SwiGLU: rows interleave gate/up in 16-row groups (lynx_pack_w13),
//        epilogue h = silu(gate) * up -> H[seg rows, 64 features] (bf16).
//        TANH2:  epilogue h = tanh(acc) -> H[seg rows, 128 features].
//   phase-1 unit (seg, mt, s):    D[128 x n] = W2[e][mt*128 : +128, K_s] . H_seg[:, K_s]^T
//        epilogue: slot[s][seg rows][mt*128 : +128] = D (f32), no waiting.
//        The epilogue warp whose split lands last for (segment, m-tile, warp
//        quarter) queues a task for this CTA's reducer warps, which sum the
//        slots in the fixed order 0..S-1 into slot 0 -- bit-reproducible
//        without float atomics -- and, for the last segment to finish a
//        column slice, apply the combine (simulator.py:101-112) for its 32
//        columns: out[t] = hidden[t] + sum_j w_tj * Y[row_tj], experts
//        ascending.  Nothing on the streaming path blocks on another CTA
//        except phase-1 loads of H (which queue order makes ready), and no
//        latency-bound L2 traffic sits in the epilogue (measured: doing the
//        reductions in the epilogue under a saturated HBM cost 2x).
//
// Swap-AB: weight rows are the MMA M (=128) dimension, the segment's tokens
// the MMA N dimension (16..256, rounded to 16), so decode streams each used
// expert's weights from HBM exactly once while the tiny activation tiles
// come from L2.  Units are dequeued from a device ticket counter in order
// [all phase-0 units][all phase-1 units]; a phase-1 unit waits (acquire)
// until its segment's phase-0 tiles are published (release), which by
// queue order has almost always already happened.
//
// Warp roles (256 threads, one CTA per SM):
//   warp 0      TMA producer + unit scheduler (one elected lane)
//   warp 1      tcgen05.mma issuer (one lane)
//   warp 2      TMEM allocator, then reducer
//   warp 3      reducer (split-K sums + fused combine, fed by the epilogue)
//   warps 4..7  epilogue: TMEM -> registers -> activation -> global
#include <cuda_bf16.h>
#include <stdint.h>

#include "lynx_internal.cuh"
#include "ptx.cuh"

namespace lynx {

constexpr int kFfnThreads = 256;
constexpr int kUnitRing = 4;
constexpr int kTileA = 128 * 64 * 2;  // 128 weight rows x 64 bf16 (one 128B-swizzled k block)
constexpr int kBoxB = 16 * 64 * 2;    // 16 token rows x 64 bf16

struct Unit {
  int phase, seg, mt, split, kb0, kb1, expert, row0, n, nmma;
};

__device__ __forceinline__ bool decode_unit(const FfnParams& p, int nseg, int u, Unit& U) {
  if (u < 0) return false;
  const int nA = nseg * p.tiles1;
  if (u < nA) {
    U.phase = 0;
    U.seg = u / p.tiles1;
    U.mt = u - U.seg * p.tiles1;
    U.split = 0;
    U.kb0 = 0;
    U.kb1 = p.kb1;
  } else {
    const int v = u - nA;
    const int per = p.tiles2 * p.split2;
    U.phase = 1;
    U.seg = v / per;
    const int r = v - U.seg * per;
    U.mt = r / p.split2;
    U.split = r - U.mt * p.split2;
    U.kb0 = U.split * p.kb2_per;
    U.kb1 = min(p.kb2_total, U.kb0 + p.kb2_per);
  }
  U.expert = p.seg_expert[U.seg];
  U.row0 = p.seg_row[U.seg];
  U.n = p.seg_count[U.seg];
  U.nmma = (U.n + 15) & ~15;
  return true;
}

__device__ __forceinline__ float silu_mul(float g, float u) { return g / (1.f + __expf(-g)) * u; }

// Scalars and pointers the reducer paths need, copied once into registers:
// reading FfnParams fields through a reference inside a non-inlined helper
// turns every access into a generic load and serialises the load chain
// (measured: ~1 L2 round trip per element).
struct ReduceCtx {
  float* __restrict__ partial;
  const __nv_bfloat16* __restrict__ hidden;
  const int32_t* __restrict__ tok_rows;
  const float* __restrict__ tok_weight;
  __nv_bfloat16* __restrict__ out_bf16;
  float* __restrict__ out_f32;
  size_t stride;  // one split slot: rows_cap * d floats
  int d, split2, T, k;
};

__device__ __forceinline__ ReduceCtx reduce_ctx(const FfnParams& p) {
  ReduceCtx c;
  c.partial = p.partial;
  c.hidden = reinterpret_cast<const __nv_bfloat16*>(p.hidden);
  c.tok_rows = p.tok_rows;
  c.tok_weight = p.tok_weight;
  c.out_bf16 = reinterpret_cast<__nv_bfloat16*>(p.out_bf16);
  c.out_f32 = p.out_f32;
  c.stride = static_cast<size_t>(p.rows_cap) * p.d;
  c.d = p.d;
  c.split2 = p.split2;
  c.T = p.T;
  c.k = p.k;
  return c;
}

// slot0[row][r] = ((slot0 + slot1) + slot2) + ... for the segment's rows:
// split-K partials summed in a fixed order (bit-reproducible).  Loads use
// clamped in-bounds addresses so they issue unconditionally (64 in flight).
__device__ __noinline__ void reduce_splits(const ReduceCtx c, int row0, int n, int r, bool rv) {
  float* base = c.partial + static_cast<size_t>(row0) * c.d + r;
  for (int t0 = 0; t0 < n; t0 += 8) {
    float acc[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) acc[u] = __ldcg(base + static_cast<size_t>(min(t0 + u, n - 1)) * c.d);
    for (int s0 = 1; s0 < c.split2; s0 += 8) {
      float v[8][8];
#pragma unroll
      for (int s = 0; s < 8; ++s)
#pragma unroll
        for (int u = 0; u < 8; ++u)
          v[s][u] = __ldcg(base + min(s0 + s, c.split2 - 1) * c.stride +
                           static_cast<size_t>(min(t0 + u, n - 1)) * c.d);
#pragma unroll
      for (int s = 0; s < 8; ++s)
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (s0 + s < c.split2) acc[u] += v[s][u];
    }
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (rv && t0 + u < n) __stcg(base + static_cast<size_t>(t0 + u) * c.d, acc[u]);
  }
}

// Combine for one output column r (all tokens): residual + experts in
// ascending order, the reference's accumulation order (simulator.py:101-112).
// Token rows/weights are fetched lane-parallel (lane = token) and broadcast.
// Called by all 32 lanes of a warp (r clamped in bounds, rv = column valid).
__device__ __noinline__ void combine_column(const ReduceCtx c, int r, bool rv) {
  const float* Y = c.partial + r;
  const int lane = threadIdx.x & 31;
  for (int t0 = 0; t0 < c.T; t0 += 32) {
    int rows[LYNX_MAX_TOPK];
    float wts[LYNX_MAX_TOPK];
    const int tl = min(t0 + lane, c.T - 1);
#pragma unroll
    for (int j = 0; j < LYNX_MAX_TOPK; ++j) {
      const int jj = min(j, c.k - 1);
      const int row = c.tok_rows[tl * c.k + jj];
      rows[j] = j < c.k ? row : -1;
      wts[j] = c.tok_weight[tl * c.k + jj];
    }
    const int tn = min(32, c.T - t0);
    for (int u0 = 0; u0 < tn; u0 += 8) {
      float acc[8], y[8][LYNX_MAX_TOPK], w[8][LYNX_MAX_TOPK];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int src = min(u0 + u, tn - 1);
        const int t = t0 + src;
        acc[u] = c.hidden ? __bfloat162float(c.hidden[static_cast<size_t>(t) * c.d + r]) : 0.f;
#pragma unroll
        for (int j = 0; j < LYNX_MAX_TOPK; ++j) {
          const int row = __shfl_sync(0xffffffffu, rows[j], src);
          w[u][j] = row >= 0 ? __shfl_sync(0xffffffffu, wts[j], src) : 0.f;
          y[u][j] = __ldcg(Y + static_cast<size_t>(max(row, 0)) * c.d);
        }
      }
#pragma unroll
      for (int u = 0; u < 8; ++u)
#pragma unroll
        for (int j = 0; j < LYNX_MAX_TOPK; ++j)
          if (j < c.k) acc[u] += w[u][j] * y[u][j];  // -1 rows carry weight 0
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        if (u0 + u >= tn || !rv) break;
        const size_t o = static_cast<size_t>(t0 + u0 + u) * c.d + r;
        if (c.out_f32)
          c.out_f32[o] = acc[u];
        else
          c.out_bf16[o] = __float2bfloat16_rn(acc[u]);
      }
    }
  }
}

// ------------------------------------------------ optional timeline trace
// Built only into the diagnostic library (-DLYNX_TRACE): one record per
// unit / task with globaltimer start and end, read back by
// lynx_debug_trace().  The production library compiles these to nothing.
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

// ------------------------------------------------ epilogue -> reducer tasks
// Bounded MPMC ticket queue in shared memory (epilogue warps push, the two
// reducer warps pop).  seq[i] == t: slot free for ticket t; == t + 1: task
// of ticket t ready.
constexpr int kTaskRing = 32;
constexpr int kTaskReduce = 0, kTaskCombine = 1;

struct TaskQueue {
  int seq[kTaskRing];
  int ring[kTaskRing];
  int head, tail, epi_done;
};

__device__ __forceinline__ int make_task(int kind, int seg, int mt, int q) {
  return (kind << 30) | (seg << 16) | (mt << 2) | q;
}

__device__ __forceinline__ int* seg_done_counter(const FfnParams& p, int mt, int q) {
  return p.counters + 1 + p.max_seg + p.max_seg * p.tiles2 * 4 + mt * 4 + q;
}

__device__ __noinline__ void task_push(TaskQueue* q, int task) {
  const int t = atomicAdd(&q->tail, 1);
  volatile int* seq = q->seq;
  Watchdog wd;
  while (seq[t % kTaskRing] != t) {  // wait for the slot's previous lap to drain
    __nanosleep(32);
    wd.tick(10);
  }
  reinterpret_cast<volatile int*>(q->ring)[t % kTaskRing] = task;
  __threadfence_block();
  seq[t % kTaskRing] = t + 1;
}

// Returns -1 once every epilogue warp is done and the queue is drained.
__device__ __noinline__ int task_pop(TaskQueue* q) {
  const int h = atomicAdd(&q->head, 1);
  volatile int* seq = q->seq;
  volatile int* vq = reinterpret_cast<volatile int*>(q);
  while (true) {
    if (seq[h % kTaskRing] == h + 1) {
      __threadfence_block();
      const int task = reinterpret_cast<volatile int*>(q->ring)[h % kTaskRing];
      seq[h % kTaskRing] = h + kTaskRing;
      return task;
    }
    const int done = vq[offsetof(TaskQueue, epi_done) / 4];
    const int tail = vq[offsetof(TaskQueue, tail) / 4];
    if (done == 4 && h >= tail) return -1;
    __nanosleep(64);
  }
}

template <int BN, int STAGES>
__global__ void __launch_bounds__(kFfnThreads, 1) ffn_kernel(const __grid_constant__ FfnParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr int kTileB = BN * 128;
  constexpr uint32_t kTmemCols = 2 * BN;
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * kTileA;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * kTileB);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* ufull = tempty + 2;
  uint64_t* uempty = ufull + kUnitRing;
  int* uring = reinterpret_cast<int*>(uempty + kUnitRing);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(uring + kUnitRing);
  TaskQueue* tq = reinterpret_cast<TaskQueue*>(tmem_slot + 4);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x < kTaskRing) tq->seq[threadIdx.x] = threadIdx.x;
  if (threadIdx.x == 0) {
    tq->head = 0;
    tq->tail = 0;
    tq->epi_done = 0;
    for (int s = 0; s < STAGES; ++s) {
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
  if (warp == 2) tmem_alloc(tmem_slot, kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  // Everything above overlapped the previous kernel (programmatic launch);
  // the dispatch plan and gathered rows are only read after this point.
  griddep_wait();
#ifdef LYNX_TRACE
  const uint64_t cta_t0 = globaltimer();
#endif
  const uint32_t tmem_base = *tmem_slot;
  const int nseg = *p.n_seg;
  const int total = nseg * (p.tiles1 + p.tiles2 * p.split2);
  if (nseg == 0) {
    // No token routed here (an expert-parallel shard can receive none):
    // the output is the residual (or zeros for a partial).
    if (warp >= 4)
      for (int r0 = blockIdx.x * 128 + (warp - 4) * 32; r0 < p.d; r0 += gridDim.x * 128)
        combine_column(reduce_ctx(p), min(r0 + lane, p.d - 1), r0 + lane < p.d);
  }

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------ TMA producer
      const uint64_t pol_w = policy_evict_first();
      const uint64_t pol_act = policy_evict_last();
      int stage = 0, slot = 0;
      uint32_t phase = 0, uphase = 0;
      while (true) {
        int u = atomicAdd(&p.counters[0], 1);
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
          tma_load_3d(sA + stage * kTileA, ma, &full[stage], kb * 64, U.mt * 128, U.expert, pol_w);
          for (int j = 0; j < nb; ++j)
            tma_load_2d(sB + stage * kTileB + j * kBoxB, mb, &full[stage], kb * 64, U.row0 + 16 * j, pol_act);
          if (++stage == STAGES) {
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
          const uint64_t ad = sdesc_kmajor_sw128(smem_u32(sA + stage * kTileA));
          const uint64_t bd = sdesc_kmajor_sw128(smem_u32(sB + stage * kTileB));
#pragma unroll
          for (int k = 0; k < 4; ++k)  // 4 x K16 per 64-wide block; +32 B = +2 in the address field
            umma_bf16_ss(dt, ad + 2 * k, bd + 2 * k, idesc, (kb > U.kb0 || k > 0) ? 1u : 0u);
          umma_commit(&empty[stage]);
          if (++stage == STAGES) {
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
      if (U.phase == 0) {
        __nv_bfloat16* H = reinterpret_cast<__nv_bfloat16*>(p.h);
        if (p.act == LYNX_ACT_SWIGLU) {
          // lanes 0-15: gate rows, lanes 16-31: up rows of the same 16 features
          const int f = U.mt * 64 + q * 16 + (lane & 15);
          const bool upper = lane >= 16;
          for (int c0 = 0; c0 < U.nmma; c0 += 16) {
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
              if (tok < U.n && f < p.ff)
                H[static_cast<size_t>(U.row0 + tok) * p.ff + f] = __float2bfloat16_rn(silu_mul(g, uu));
            }
          }
        } else {
          const int f = U.mt * 128 + q * 32 + lane;
          for (int c0 = 0; c0 < U.nmma; c0 += 16) {
            uint32_t v[16];
            tmem_ld16(tb + c0, v);
            tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              const int tok = c0 + j;
              if (tok < U.n && f < p.ff)
                H[static_cast<size_t>(U.row0 + tok) * p.ff + f] = __float2bfloat16_rn(tanhf(__uint_as_float(v[j])));
            }
          }
        }
      } else {
        // ---- phase 1: split-K partial -> slot s; the last split of this
        //      (segment, m-tile, warp quarter) to land sums slots 0..S-1 in
        //      order into slot 0; the last segment then applies the combine.
        const int r = U.mt * 128 + q * 32 + lane;  // output column (d index)
        const bool rv = r < p.d;
        const size_t slot_stride = static_cast<size_t>(p.rows_cap) * p.d;
        float* mine = p.partial + U.split * slot_stride + static_cast<size_t>(U.row0) * p.d + r;
        for (int c0 = 0; c0 < U.nmma; c0 += 16) {
          uint32_t v[16];
          tmem_ld16(tb + c0, v);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 16; ++j)
            if (c0 + j < U.n && rv) __stcg(mine + static_cast<size_t>(c0 + j) * p.d, __uint_as_float(v[j]));
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[acc]);
        acc ^= 1;
        if (acc == 0) aphase ^= 1;
        // Publish the slot; whoever completes a reduction hands the
        // latency-bound follow-up (split sum, combine) to the reducer warps
        // so this warp is back on TMEM without waiting on L2.
        __threadfence();
        __syncwarp();
        if (lane == 0) {
          if (p.split2 > 1) {
            int* cnt = p.counters + 1 + p.max_seg + (U.seg * p.tiles2 + U.mt) * 4 + q;
            if (atom_add_acq_rel_gpu(cnt, 1) == p.split2 - 1) task_push(tq, make_task(kTaskReduce, U.seg, U.mt, q));
          } else if (atom_add_acq_rel_gpu(seg_done_counter(p, U.mt, q), 1) == nseg - 1) {
            task_push(tq, make_task(kTaskCombine, 0, U.mt, q));
          }
        }
        __syncwarp();
        if (lane == 0) LYNX_TRACE_REC(2, u);
        continue;
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
      // publish this warp's slice of H to phase-1 consumers on other SMs
      __threadfence();
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) red_release_gpu_add(p.counters + 1 + U.seg, 1);
      if (lane == 0) LYNX_TRACE_REC(2, u);
      acc ^= 1;
      if (acc == 0) aphase ^= 1;
    }
    if (lane == 0) atomicAdd(&tq->epi_done, 1);
  } else if (warp == 2 || warp == 3) {
    // -------------------------------------------------- reducers
    // Split-K sums and the final combine are chains of dependent L2 loads;
    // with HBM saturated by the weight stream their latency is long, so
    // they run here, overlapped with streaming, never in the epilogue.
    const ReduceCtx ctx = reduce_ctx(p);
    while (true) {
      int task = 0;
      if (lane == 0) task = task_pop(tq);
      task = __shfl_sync(0xffffffffu, task, 0);
      if (task < 0) break;
      LYNX_TRACE_T0;
      const int kind = task >> 30, seg = (task >> 16) & 0x3FFF, mt = (task >> 2) & 0x3FFF, q = task & 3;
      const int r = mt * 128 + q * 32 + lane;
      const bool rv = r < p.d;
      fence_acq_rel_gpu();
      int last = 1;
      if (kind == kTaskReduce) {
        reduce_splits(ctx, p.seg_row[seg], p.seg_count[seg], min(r, p.d - 1), rv);
        __threadfence();
        __syncwarp();
        if (lane == 0) last = atom_add_acq_rel_gpu(seg_done_counter(p, mt, q), 1) == nseg - 1;
        last = __shfl_sync(0xffffffffu, last, 0);
        if (last) fence_acq_rel_gpu();
      }
      if (last) combine_column(ctx, min(r, p.d - 1), rv);
      __syncwarp();
      if (lane == 0) LYNX_TRACE_REC(last ? 6 : 3, task);
    }
  }
  tc_fence_before();
  __syncthreads();
#ifdef LYNX_TRACE
  if (threadIdx.x == 0) trace(5, nseg, cta_t0, globaltimer());
#endif
  griddep_launch_dependents();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, kTmemCols);
  }
}

template <int BN, int STAGES>
static cudaError_t launch_ffn_t(const FfnParams& p, int sm_count, cudaStream_t s) {
  constexpr size_t smem =
      1024 + STAGES * (kTileA + BN * 128) + (2 * STAGES + 4 + 2 * kUnitRing) * 8 + kUnitRing * 4 + 16 +
      sizeof(TaskQueue);
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

cudaError_t launch_ffn(const FfnParams& p, int bn, int sm_count, cudaStream_t s) {
  switch (bn) {
    case 32:
      return launch_ffn_t<32, 10>(p, sm_count, s);
    case 64:
      return launch_ffn_t<64, 8>(p, sm_count, s);
    case 128:
      return launch_ffn_t<128, 6>(p, sm_count, s);
    default:
      return launch_ffn_t<256, 4>(p, sm_count, s);
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
