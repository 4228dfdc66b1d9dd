// lynx_internal.cuh -- kernel argument structs and launchers shared by the
// translation units behind the C ABI (include/lynx_b200.h).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/lynx_b200.h"

namespace lynx {

constexpr int kSelectThreads = 512;

struct SelectArgs {
  const double* logits;
  int T, N, k, decode;
  lynx_policy_t pol;
  int floor_keep;  // resolved min_experts (>= k)
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
};

// Dispatch bookkeeping the FFN and combine kernels read.
struct DispatchView {
  int32_t* n_seg;
  int32_t* n_used;
  int32_t* seg_expert;
  int32_t* seg_row;
  int32_t* seg_count;
  int32_t* perm_token;
  float* perm_weight;
  int32_t* tok_rows;
  float* tok_weight;
  uint16_t* x_perm;
};

struct PermuteArgs {
  const int32_t* assigned;
  const double* weights;
  const uint16_t* hidden;
  int T, N, k, d;
  int max_seg, rows_cap;
  DispatchView out;
  int* counters;   // FFN scheduler words to zero (may be null)
  int n_counters;
};

// Grouped expert FFN (K3).  Phase 0 = gate/up (or tanh w1) over d,
// phase 1 = down projection over ff, split-K into `split2` partials.
struct FfnParams {
  CUtensorMap map_w1;  // (d, rows1, E)   box (64, 128, 1)
  CUtensorMap map_w2;  // (ff, d, E)      box (64, 128, 1)
  CUtensorMap map_x;   // (d, rows_cap)   box (64, 16)
  CUtensorMap map_h;   // (ff, rows_cap)  box (64, 16)
  const int32_t* n_seg;
  const int32_t* seg_expert;
  const int32_t* seg_row;
  const int32_t* seg_count;
  uint16_t* h;      // [rows_cap, ff] bf16
  float* partial;   // [split2, rows_cap, d] f32
  int* counters;    // [0] unit ticket, [1 + s] phase-0 tiles done for segment s
  int d, ff, act;
  int tiles1, kb1;  // phase 0: 128-row tiles per segment, 64-wide k blocks
  int tiles2, split2, kb2_per, kb2_total;
  int rows_cap;
};

struct CombineArgs {
  const uint16_t* hidden;  // residual (null -> no residual)
  const float* partial;
  int split2, rows_cap, T, k, d;
  const int32_t* tok_rows;
  const float* tok_weight;
  uint16_t* out_bf16;  // one of these is set
  float* out_f32;
};

cudaError_t launch_router_logits(const uint16_t* hidden, const uint16_t* wt, int T, int d, int N, double* logits,
                                 cudaStream_t s);
cudaError_t launch_route_select(const SelectArgs& a, cudaStream_t s);
cudaError_t launch_remap(const int32_t* ids, const double* full, int T, int N, int k, const uint8_t* retained,
                         int32_t* assigned, double* weights, int32_t* flags, cudaStream_t s);
cudaError_t launch_topk(const double* vals, int T, int N, int k, int32_t* ids, double* out, cudaStream_t s);
cudaError_t launch_vote(const int32_t* ids, int T, int k, int N, const lynx_policy_t& w, double* counts,
                        cudaStream_t s);
cudaError_t launch_permute(const PermuteArgs& a, int sm_count, cudaStream_t s);
cudaError_t launch_ffn(const FfnParams& p, int bn, int sm_count, cudaStream_t s);
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
