// lynx_internal.cuh -- kernel argument structs, programmatic-dependent-launch
// helpers and launchers shared by the translation units behind the C ABI
// (include/lynx_b200.h).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <utility>

#include "../../include/lynx_b200.h"

namespace lynx {

constexpr int kSelectThreads = 1024;  // one warp per token, 32 tokens at a time
constexpr size_t kSelectMaxSmem = 200 * 1024;

// ------------------------------------------------- programmatic dependent launch
// Every kernel of the layer chain is launched with programmatic stream
// serialization: it may start while its predecessor drains, runs its
// prologue, and calls griddep_wait() before touching anything the
// predecessor (or anything before it) wrote.  Because every kernel waits
// before it completes, completion stays transitive along the stream.
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void griddep_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// Touch every 32-byte line of a __grid_constant__ kernel argument before
// griddep_wait(): the constant-cache misses of a cold SM then overlap the
// predecessor's tail instead of stalling the kernel's first uses.
template <typename A>
__device__ __forceinline__ void warm_params(const A& a) {
  constexpr int kLines = static_cast<int>((sizeof(A) + 31) / 32);
  __shared__ int s_sink[kLines];  // one word per thread: a store keeps ptxas from dropping the load
  if (static_cast<int>(threadIdx.x) < kLines)
    *static_cast<volatile int*>(&s_sink[threadIdx.x]) = reinterpret_cast<const int*>(&a)[threadIdx.x * 8];
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// Peer-memory EP hooks inside the layer kernels (ep_p2p.cu): K0 stores its
// logits rows into every peer and signals; K1 / K2 wait for every peer's
// logits / rows before reading them.  enabled = 0: plain single-GPU kernels.
struct EpLink {
  int enabled;
  int kind;  // the signal this kernel waits for (K1: logits, K2: dispatch)
  lynx_ep_peers_t P;
};

// Dispatch plan written by K1 (or the standalone plan kernel).
struct PlanOut {
  int enabled;
  int n_shared;         // S always-on experts N..N+S-1 over all T tokens (tok_rows stride k+S)
  int32_t* n_seg;
  int32_t* n_used;
  int32_t* n_rows;      // rows of the permuted buffer in use (16-padded per expert)
  int32_t* max_rows;    // rows of the largest segment (K3's stage width), or null
  int32_t* seg_expert;
  int32_t* seg_row;
  int32_t* seg_count;
  int32_t* seg_order;   // [max_seg] K3 queue order: segments by rows desc (LPT), or null
  int32_t* perm_token;  // [rows_cap] source token, -1 = padding
  float* perm_weight;
  int32_t* tok_rows;    // [T,k+S] permuted rows per token: routed experts ascending (-1 padded),
  float* tok_weight;    //   then the S shared experts (weight 1)
  int* counters;        // FFN scheduler words zeroed for the next K3 launch
  int n_counters;
};

struct SelectArgs {
  const double* logits;  // null: the selection (ids/probs/full) is an input
  int T, N, k, decode;
  lynx_policy_t pol;
  int floor_keep;  // resolved min_experts (>= k)
  int stage;       // stage per-token arrays in shared memory
  int routed_top;  // given selection came from K0's routing: probs[:, :2] are the row's top two
  int32_t* ids;
  double* probs;
  double* full;
  double* conf;
  double* counts;
  uint8_t* retained;
  int32_t* assigned;
  double* weights;
  uint8_t* important;
  int32_t* flags;
  PlanOut plan;
  EpLink ep;  // peer-memory EP: wait for every peer's logits first
};

// Grouped expert FFN (K3).  Phase 0 = gate/up (or tanh w1) over d, phase 1 =
// down projection over ff, split-K into `split2` partial slots that K4 sums.
struct FfnParams {
  CUtensorMap map_w1;  // (d, rows1, E)   box (64, 128, 1)
  CUtensorMap map_w2;  // (ff, d, E)      box (64, 128, 1)
  CUtensorMap map_x;   // (d, rows_cap)   box (64, 16)
  CUtensorMap map_h;   // (ff, rows_cap)  box (64, 16)
  const int32_t* n_seg;
  const int32_t* seg_expert;
  const int32_t* seg_row;
  const int32_t* seg_count;
  const int32_t* seg_order;  // queue slot -> segment (largest first)
  const int32_t* max_rows;   // rows of the largest segment, or null (-> the launch's BN)
  uint16_t* h;      // [rows_cap, ff] bf16
  float* partial;   // [split2, rows_cap, d] f32
  int* counters;    // [0] unit ticket, [1 + s] phase-0 tiles done for segment s
  int d, ff, act;
  int tiles1, kb1;  // phase 0: 128-row tiles per segment, 64-wide k blocks
  int tiles2, split2, kb2_per, kb2_total;
  int rows_cap;
};

// K4: split-K sum + weighted combine (+ residual).
struct CombineArgs {
  const uint16_t* hidden;  // residual; null -> no residual (EP partial)
  int peer_mode;           // 1: row t goes to peers.back[t / Tl] rows rank*Tl + t % Tl, then signal
  lynx_ep_peers_t peers;
  const float* partial;    // [split2][rows_cap][d]
  size_t slot_stride;      // rows_cap * d
  int split2, T, k, d;  // k = entries per token in tok_rows (top_k + shared)
  const int32_t* tok_rows;
  const float* tok_weight;
  uint16_t* out_bf16;  // exactly one of the outputs is set
  float* out_f32;
  // K3's scratch, dead once K3 completes (H, the gathered token rows):
  // dropped from L2 without write-back (discard.global.L2), and the split-K
  // slots after K4 reads them (discard_partials; needs d % 32 == 0 so no
  // 128-byte line spans two rows)
  const int32_t* discard_rows;  // rows of both regions in use (the plan's n_rows), or null: no discard
  uint8_t* discard_base[2];
  size_t discard_row_bytes[2];
  int discard_partials;
};

struct GatherArgs {
  const uint16_t* hidden;
  const int32_t* perm_token;
  const int32_t* n_rows;
  int rows_cap, d;
  uint16_t* x_perm;
  EpLink ep;  // peer-memory EP: wait for every peer's dispatched rows first
};

// Attention stand-in (attention.cu).
struct AttnArgs {
  const uint16_t* h_in;  // [B*Tn, d]
  const uint16_t* wqkv;  // [3*dh, d]
  const uint16_t* wo;    // [dh, d]
  float* kcache;         // [B, max_len, dh]
  float* vcache;
  float* q;              // [B*Tn, dh] scratch
  const int32_t* pos;
  int B, Tn, d, dh, max_len, norm_input;
  uint16_t* h_out;
  // fused router (router_wt != null): per-(row, column chunk) partial dots
  // and sum of squares, the row's last chunk finishes the logits
  const uint16_t* router_wt;
  int N;
  double* logits;
  float* rpart;       // [B*Tn, chunks, N + 1]
  int* row_arrivals;  // [B*Tn], zero; re-armed by the last chunk
};
size_t attn_out_smem(int d, int dh, int max_len);
cudaError_t launch_attention(const AttnArgs& a, cudaStream_t s);
cudaError_t launch_advance_position(int32_t* pos, int by, cudaStream_t s);

cudaError_t launch_trace_append(const lynx_trace_ring_t& r, const int32_t* pos, int layer,
                                const lynx_selection_t& sel, cudaStream_t s);

cudaError_t launch_ep_dispatch(const lynx_ep_peers_t& P, const uint16_t* hidden_local, const int32_t* assigned, int k,
                               int N, int d, cudaStream_t s);
cudaError_t launch_ep_p2p_combine(const lynx_ep_peers_t& P, const uint16_t* hidden_local, int d, uint16_t* out,
                                  cudaStream_t s);

cudaError_t launch_router_logits(const uint16_t* hidden, const uint16_t* wt, int T, int d, int N, double* logits,
                                 cudaStream_t s, const EpLink* put = nullptr);
// K0 + routing for 16 < N <= 64 (clusters of ceil(N/8) CTAs per token):
// writes full/ids/probs (and logits if non-null); K1 then runs on the given selection.
cudaError_t launch_router_route(const uint16_t* hidden, const uint16_t* wt, int T, int d, int N, int k,
                                double* logits, double* full, int32_t* ids, double* probs, cudaStream_t s);
// Fused K0 + K1 + K2 for N <= 8, T <= 256, no shared experts (select.cu front_kernel).
size_t front_smem_bytes(int T, int N, int k, int d);

cudaError_t launch_front(const SelectArgs& a, const uint16_t* hidden, const uint16_t* router_wt, int d,
                         uint16_t* x_perm, int* sync, const double* logits_in, cudaStream_t s);
size_t select_smem_bytes(int T, int N, int k, bool stage, bool plan);
bool select_can_stage(int T, int N, int k, bool plan);
cudaError_t launch_route_select(const SelectArgs& a, cudaStream_t s);
cudaError_t launch_plan(const int32_t* asg, const double* w, int T, int N, int k, const PlanOut& o, cudaStream_t s);
cudaError_t launch_remap(const int32_t* ids, const double* full, int T, int N, int k, const uint8_t* retained,
                         int32_t* assigned, double* weights, int32_t* flags, cudaStream_t s);
cudaError_t launch_topk(const double* vals, int T, int N, int k, int32_t* ids, double* out, cudaStream_t s);
cudaError_t launch_vote(const int32_t* ids, int T, int k, int N, const lynx_policy_t& w, double* counts,
                        cudaStream_t s);
cudaError_t launch_gather(const GatherArgs& a, int sm_count, cudaStream_t s);
// rows_hint: expected token rows per used expert (picks the CTA-pair kernel for wide segments)
cudaError_t launch_ffn(const FfnParams& p, int bn, int rows_hint, int sm_count, cudaStream_t s);
// K3 kernel choice: true -> ffn_pair_kernel (cta_group::2), false -> ffn_kernel
bool ffn_use_pair(int bn, int rows_hint);
cudaError_t launch_combine(const CombineArgs& a, cudaStream_t s);
cudaError_t launch_pack_w13(const uint16_t* w1, const uint16_t* w3, int N, int ff, int d, uint16_t* w13,
                            cudaStream_t s);
cudaError_t launch_ep_pack(const uint16_t* hidden_local, const int32_t* assigned, int T_local, int k, int N, int G,
                           int d, int rank, uint16_t* send, cudaStream_t s);
cudaError_t launch_ep_local_mask(const int32_t* assigned, const double* weights, int T, int k, int N, int G,
                                 int rank, int32_t* assigned_local, double* weights_local, cudaStream_t s);
cudaError_t launch_ep_combine(const uint16_t* hidden_local, const float* recv, int T_local, int G, int d,
                              uint16_t* out, cudaStream_t s);

// 2*ceil64(ff): rows of the packed gate/up matrix per expert.
inline int swiglu_rows(int ff) { return 2 * ((ff + 63) / 64) * 64; }

}  // namespace lynx
