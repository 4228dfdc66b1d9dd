// capi.cu -- extern "C" entry points of include/lynx_b200.h: argument
// validation mirroring the reference's ValidationError sites, workspace
// planning, TMA descriptor encoding and the kernel chain
//
//   K0 router GEMV -> K1 route + policy + remap + dispatch plan ->
//   K2 gather -> K3 grouped expert GEMM (tcgen05) + fused combine
//
// launched back to back with programmatic dependent launch (no host sync).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include <algorithm>

#include "lynx_internal.cuh"
#include "p2p.cuh"

using namespace lynx;

namespace {

constexpr int kAbiVersion = 5;

int sm_count_cached() {
  static int cached_dev = -1, cached = 0;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  if (dev != cached_dev) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 0;
    cached = n;
    cached_dev = dev;
  }
  return cached;
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// bf16 tensor, dim0 contiguous, 128B swizzle, OOB -> zero.
bool encode_bf16(CUtensorMap* m, const void* ptr, int rank, const uint64_t* dims, const uint32_t* box) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t gdim[3], gstride[2];
  cuuint32_t bdim[3], estride[3] = {1, 1, 1};
  uint64_t stride = 2;
  for (int i = 0; i < rank; ++i) {
    gdim[i] = dims[i];
    bdim[i] = box[i];
    if (i > 0) gstride[i - 1] = stride;
    stride *= dims[i];
  }
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, const_cast<void*>(ptr), gdim, gstride, bdim, estride,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// k blocks (64 wide) per phase-1 unit.  Default: the down projection split
// in two halves (at least 32 blocks), so the expert stream ends in
// 2*tiles2 units per segment and K4 sums two partial slots.  Measured on
// B200 at Mixtral shape (kb2_total = 224): split 2 beat 3, 4, 7, 14 and 1 by
// 1.5-5% at T = 32 and 64 (fewer unit transitions and partial writes while
// the queue still balances); LYNX_KB2_PER overrides it for experiments.
int kb2_per_unit(int kb2_total) {
  static int env = -1;
  if (env < 0) {
    const char* s = getenv("LYNX_KB2_PER");
    env = s ? atoi(s) : 0;
    if (env < 0) env = 0;
  }
  if (env) return env;
  return std::max(32, (kb2_total + 1) / 2);
}

size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

// LYNX_FUSED_FRONT=0 runs K0, K1 and K2 as separate kernels for N <= 8 (A/B switch).
bool fused_front_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("LYNX_FUSED_FRONT");
    v = (e && e[0] == '0' && !e[1]) ? 0 : 1;
  }
  return v == 1;
}

// LYNX_L2_DISCARD=0 keeps K3's dead scratch in L2 (written back when evicted); 2 / 3 drop only
// the split-K slots / only H and the gathered rows (A/B switch).
int l2_discard_mode() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("LYNX_L2_DISCARD");
    v = e ? atoi(e) : 1;
  }
  return v;
}

// LYNX_ROUTE_IN_K1=1 keeps the routing in K1 for N > 16 (A/B switch).
bool route_in_k0_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("LYNX_ROUTE_IN_K1");
    v = (e && atoi(e)) ? 0 : 1;
  }
  return v == 1;
}

struct Caps {
  int max_seg, rows_cap;
};

// S shared experts add S segments-per-256-tokens and S 16-padded copies of
// the T token rows after the routed experts.
Caps caps_for(int T, int N, int k, int S = 0) {
  const int slots = T * k;
  const int seg_per_shared = (T + LYNX_SEG_ROWS - 1) / LYNX_SEG_ROWS;
  Caps c;
  c.max_seg = std::min(N, slots) + slots / LYNX_SEG_ROWS + 1 + S * seg_per_shared;
  c.rows_cap = static_cast<int>(align_up(static_cast<size_t>(slots) + 15 * std::min(N, slots), 16) +
                                static_cast<size_t>(S) * align_up(T, 16));
  return c;
}

struct Geometry {
  int rows1, tiles1, kb1, tiles2, kb2_total, kb2_per, split2, bn;
};

Geometry geometry(const lynx_layer_t* L, int T) {
  Geometry g;
  g.rows1 = L->activation == LYNX_ACT_SWIGLU ? swiglu_rows(L->d_ff) : L->d_ff;
  g.tiles1 = (g.rows1 + 127) / 128;
  g.kb1 = (L->d_model + 63) / 64;
  g.tiles2 = (L->d_model + 127) / 128;
  g.kb2_total = (L->d_ff + 63) / 64;
  g.kb2_per = std::min(g.kb2_total, kb2_per_unit(g.kb2_total));
  g.split2 = (g.kb2_total + g.kb2_per - 1) / g.kb2_per;
  const int rows = std::min(T, LYNX_SEG_ROWS);
  g.bn = rows <= 32 ? 32 : rows <= 64 ? 64 : rows <= 128 ? 128 : 256;
  return g;
}

// Workspace carve-up.  Selection region only for the whole-layer call.
struct Plan {
  size_t sync;  // fused-front barrier words (zero before the first call; every call leaves them zero)
  size_t logits, ids, probs, full, conf, counts, retained, assigned, weights, important, flags;
  size_t n_seg, n_used, n_rows, max_rows, seg_expert, seg_row, seg_count, seg_order, perm_token, perm_weight, tok_rows,
      tok_weight;
  size_t counters, x_perm, h, y;
  size_t total;
  int n_counters;
};

Plan plan_for(const lynx_layer_t* L, int T, bool selection) {
  const int N = L->num_experts, k = L->top_k, d = L->d_model, ff = L->d_ff, S = L->num_shared;
  const Caps c = caps_for(T, N, k, S);
  const Geometry g = geometry(L, T);
  Plan p{};
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const size_t o = off;
    off = align_up(off + bytes, 256);
    return o;
  };
  if (selection) {
    p.sync = take(64);
    p.logits = take(sizeof(double) * T * N);
    p.ids = take(sizeof(int32_t) * T * k);
    p.probs = take(sizeof(double) * T * k);
    p.full = take(sizeof(double) * T * N);
    p.conf = take(sizeof(double) * T);
    p.counts = take(sizeof(double) * N);
    p.retained = take(N);
    p.assigned = take(sizeof(int32_t) * T * k);
    p.weights = take(sizeof(double) * T * k);
    p.important = take(T);
    p.flags = take(sizeof(int32_t));
  }
  p.n_seg = take(sizeof(int32_t));
  p.n_used = take(sizeof(int32_t));
  p.n_rows = take(sizeof(int32_t));
  p.max_rows = take(sizeof(int32_t));
  p.seg_expert = take(sizeof(int32_t) * c.max_seg);
  p.seg_row = take(sizeof(int32_t) * c.max_seg);
  p.seg_count = take(sizeof(int32_t) * c.max_seg);
  p.seg_order = take(sizeof(int32_t) * c.max_seg);
  p.perm_token = take(sizeof(int32_t) * c.rows_cap);
  p.perm_weight = take(sizeof(float) * c.rows_cap);
  p.tok_rows = take(sizeof(int32_t) * T * (k + S));
  p.tok_weight = take(sizeof(float) * T * (k + S));
  // unit ticket + phase-0 tiles published per segment
  p.n_counters = 1 + c.max_seg;
  p.counters = take(sizeof(int32_t) * p.n_counters);
  p.x_perm = take(sizeof(uint16_t) * static_cast<size_t>(c.rows_cap) * d);
  p.h = take(sizeof(uint16_t) * static_cast<size_t>(c.rows_cap) * ff);
  // split-K partial slots [split2][rows_cap][d]; slot 0 ends up holding Y
  p.y = take(sizeof(float) * static_cast<size_t>(g.split2) * c.rows_cap * d);
  p.total = off + 256;  // slack for base alignment
  return p;
}

template <typename T>
T* at(void* base, size_t off) {
  return reinterpret_cast<T*>(static_cast<char*>(base) + off);
}

// slots_exceed_ok: an expert-parallel shard holds fewer experts than the
// routing width; its mask has top_k slots per token, most of them -1.
int check_layer(const lynx_layer_t* L, int T, bool slots_exceed_ok = false) {
  if (!L) return LYNX_ERR_SHAPE;
  if (T < 1 || L->num_experts < 1 || L->d_model < 8 || L->d_ff < 8) return LYNX_ERR_SHAPE;
  if (L->top_k < 1 || (!slots_exceed_ok && L->top_k > L->num_experts)) return LYNX_ERR_TOPK;
  if (L->num_experts > LYNX_MAX_EXPERTS || L->top_k > LYNX_MAX_TOPK || T > LYNX_MAX_TOKENS)
    return LYNX_ERR_UNSUPPORTED;
  if (L->d_model % 8 || L->d_ff % 8) return LYNX_ERR_UNSUPPORTED;  // TMA 16-byte strides
  if (L->activation != LYNX_ACT_SWIGLU && L->activation != LYNX_ACT_TANH2) return LYNX_ERR_CONFIG;
  if (L->num_shared < 0) return LYNX_ERR_SHAPE;
  if (L->num_shared > LYNX_MAX_SHARED) return LYNX_ERR_UNSUPPORTED;
  if (!L->w13 || !L->w2) return LYNX_ERR_SHAPE;
  return LYNX_OK;
}

// PolicyConfig.__post_init__ (policy.py:40-55) + the checks the reference
// performs lazily on the decode path (policy.py:61-64, 130-133).
int check_policy(const lynx_policy_t* pol, int k, int decode, int* floor_keep) {
  *floor_keep = k;
  if (!pol || pol->mode == LYNX_POLICY_NONE) return LYNX_OK;
  if (pol->mode != LYNX_POLICY_LATENCY && pol->mode != LYNX_POLICY_ACCURACY) return LYNX_ERR_CONFIG;
  if (pol->drop_count < 0 || !(pol->confidence_threshold >= 0.0 && pol->confidence_threshold <= 1.0) ||
      pol->sample_threshold < 1 || pol->min_experts < 0 || pol->freq_keep_budget < 1 ||
      (pol->confidence_metric != LYNX_CONF_TOP1 && pol->confidence_metric != LYNX_CONF_MARGIN) ||
      pol->n_rank_weights < 0 || pol->n_rank_weights > LYNX_MAX_TOPK)
    return LYNX_ERR_CONFIG;
  for (int r = 0; r < pol->n_rank_weights; ++r)
    if (!(pol->rank_weights[r] >= 0.0)) return LYNX_ERR_CONFIG;
  if (!decode) return LYNX_OK;
  if (pol->min_experts > 0 && pol->min_experts < k) return LYNX_ERR_MIN_EXPERTS;
  if (pol->n_rank_weights != 0 && pol->n_rank_weights != k) return LYNX_ERR_CONFIG;
  if (pol->min_experts > 0) *floor_keep = pol->min_experts;
  return LYNX_OK;
}

int cuda_status(cudaError_t e) { return e == cudaSuccess ? LYNX_OK : LYNX_ERR_CUDA; }

PlanOut plan_out(void* ws, const Plan& P, int n_shared) {
  PlanOut o{};
  o.enabled = 1;
  o.n_shared = n_shared;
  o.n_seg = at<int32_t>(ws, P.n_seg);
  o.n_used = at<int32_t>(ws, P.n_used);
  o.n_rows = at<int32_t>(ws, P.n_rows);
  o.max_rows = at<int32_t>(ws, P.max_rows);
  o.seg_expert = at<int32_t>(ws, P.seg_expert);
  o.seg_row = at<int32_t>(ws, P.seg_row);
  o.seg_count = at<int32_t>(ws, P.seg_count);
  o.seg_order = at<int32_t>(ws, P.seg_order);
  o.perm_token = at<int32_t>(ws, P.perm_token);
  o.perm_weight = at<float>(ws, P.perm_weight);
  o.tok_rows = at<int32_t>(ws, P.tok_rows);
  o.tok_weight = at<float>(ws, P.tok_weight);
  o.counters = at<int>(ws, P.counters);
  o.n_counters = P.n_counters;
  return o;
}

inline void record(cudaEvent_t const* ev, int i, cudaStream_t s) {
  if (ev) cudaEventRecord(ev[i], s);
}

// K2 gather -> K3 expert GEMM + combine, on a plan already in the workspace.
// ev (optional): [0] before K2 (gather), [1] before K3 (FFN), [2] before K4 (combine).
// kept_hint: experts expected to stay in use (the policy's kept-set size;
// N when unknown), for K3's kernel choice only.
int gather_and_ffn(const lynx_layer_t* L, const uint16_t* hidden, int T, uint16_t* out_bf16, float* out_f32,
                   void* ws, const Plan& P, cudaStream_t s, cudaEvent_t const* ev,
                   const lynx_ep_peers_t* peers = nullptr, int kept_hint = 0, bool gathered = false) {
  const int N = L->num_experts, k = L->top_k, d = L->d_model, ff = L->d_ff, S = L->num_shared;
  const int sms = sm_count_cached();
  if (sms <= 0) return LYNX_ERR_CUDA;
  const Caps c = caps_for(T, N, k, S);
  const Geometry g = geometry(L, T);
  const PlanOut o = plan_out(ws, P, S);

  GatherArgs ga{};
  if (peers) {
    ga.ep.enabled = 1;
    ga.ep.kind = kSigDispatch;
    ga.ep.P = *peers;
  }
  ga.hidden = hidden;
  ga.perm_token = o.perm_token;
  ga.n_rows = o.n_rows;
  ga.rows_cap = c.rows_cap;
  ga.d = d;
  ga.x_perm = at<uint16_t>(ws, P.x_perm);
  record(ev, 0, s);
  int st = gathered ? LYNX_OK : cuda_status(launch_gather(ga, sms, s));  // the fused front gathered already
  if (st) return st;

  FfnParams fp{};
  {
    const uint64_t dw1[3] = {static_cast<uint64_t>(d), static_cast<uint64_t>(g.rows1), static_cast<uint64_t>(N + S)};
    const uint64_t dw2[3] = {static_cast<uint64_t>(ff), static_cast<uint64_t>(d), static_cast<uint64_t>(N + S)};
    const uint64_t dx[2] = {static_cast<uint64_t>(d), static_cast<uint64_t>(c.rows_cap)};
    const uint64_t dh[2] = {static_cast<uint64_t>(ff), static_cast<uint64_t>(c.rows_cap)};
    const uint32_t bw[3] = {64, 128, 1};
    const uint32_t ba[2] = {64, 16};
    if (!encode_bf16(&fp.map_w1, L->w13, 3, dw1, bw) || !encode_bf16(&fp.map_w2, L->w2, 3, dw2, bw))
      return LYNX_ERR_CUDA;
    if (!encode_bf16(&fp.map_x, ga.x_perm, 2, dx, ba) || !encode_bf16(&fp.map_h, at<uint16_t>(ws, P.h), 2, dh, ba))
      return LYNX_ERR_CUDA;
  }
  fp.n_seg = o.n_seg;
  fp.seg_expert = o.seg_expert;
  fp.seg_row = o.seg_row;
  fp.seg_count = o.seg_count;
  fp.seg_order = o.seg_order;
  fp.max_rows = o.max_rows;
  fp.h = at<uint16_t>(ws, P.h);
  fp.partial = at<float>(ws, P.y);
  fp.counters = o.counters;
  fp.d = d;
  fp.ff = ff;
  fp.act = L->activation;
  fp.tiles1 = g.tiles1;
  fp.kb1 = g.kb1;
  fp.tiles2 = g.tiles2;
  fp.split2 = g.split2;
  fp.kb2_per = g.kb2_per;
  fp.kb2_total = g.kb2_total;
  fp.rows_cap = c.rows_cap;
  record(ev, 1, s);
  const int kept = kept_hint > 0 ? std::min(kept_hint, N) : N;
  st = cuda_status(launch_ffn(fp, g.bn, T * k / kept, sms, s));
  if (st) return st;

  CombineArgs ca{};
  ca.hidden = (out_f32 || peers) ? nullptr : hidden;
  if (peers) {
    ca.peer_mode = 1;
    ca.peers = *peers;
  }
  ca.partial = fp.partial;
  ca.slot_stride = static_cast<size_t>(c.rows_cap) * d;
  ca.split2 = g.split2;
  ca.T = T;
  ca.k = k + S;
  ca.d = d;
  ca.tok_rows = o.tok_rows;
  ca.tok_weight = o.tok_weight;
  ca.out_bf16 = out_bf16;
  ca.out_f32 = out_f32;
  // Dropping K3's dead scratch from L2 (instead of writing it back while the
  // next layer streams) pays where the scratch is large next to K4's own
  // work: the wide-d_ff layers whose down projection K4 sums from two split-K
  // slots (C2 -1.6 us, C5 T=256 -16 us); at C4 (one slot, 8 rows per token)
  // the discards lengthen K4 more than they save (+1 us).  LYNX_L2_DISCARD:
  // 0 off, 1 on (default, this rule), 2 slots only, 3 scratch only.
  const int dmode = g.split2 >= 2 ? l2_discard_mode() : 0;
  if (dmode == 1 || dmode == 3) {
    ca.discard_rows = o.n_rows;
    ca.discard_base[0] = reinterpret_cast<uint8_t*>(fp.h);
    ca.discard_row_bytes[0] = sizeof(uint16_t) * static_cast<size_t>(ff);
    ca.discard_base[1] = reinterpret_cast<uint8_t*>(ga.x_perm);
    ca.discard_row_bytes[1] = sizeof(uint16_t) * static_cast<size_t>(d);
  }
  if (dmode == 1 || dmode == 2) ca.discard_partials = d % 32 == 0 ? 1 : 0;
  record(ev, 2, s);
  return cuda_status(launch_combine(ca, s));
}

void* aligned_ws(void* ws) {
  return reinterpret_cast<void*>((reinterpret_cast<uintptr_t>(ws) + 255) & ~uintptr_t(255));
}

SelectArgs select_args(const double* logits, int T, int N, int k, int decode, const lynx_policy_t* policy,
                       int floor_keep) {
  SelectArgs a{};
  a.logits = logits;
  a.T = T;
  a.N = N;
  a.k = k;
  a.decode = decode;
  if (policy) {
    a.pol = *policy;
  } else {
    a.pol = lynx_policy_t{};
    a.pol.mode = LYNX_POLICY_NONE;
  }
  a.floor_keep = floor_keep;
  a.plan.enabled = 0;
  return a;
}

int moe_forward_common(const lynx_layer_t* layer, const uint16_t* hidden, int T, const int32_t* assigned,
                       const double* weights, uint16_t* out_bf16, float* out_f32, void* workspace,
                       size_t workspace_bytes, cudaStream_t stream, const lynx_ep_peers_t* peers = nullptr) {
  const bool partial = out_f32 != nullptr || peers != nullptr;
  int st = check_layer(layer, T, partial);
  if (st) return st;
  if (partial && layer->num_shared) return LYNX_ERR_UNSUPPORTED;
  const Plan P = plan_for(layer, T, false);
  if (!workspace || workspace_bytes < P.total) return LYNX_ERR_WORKSPACE;
  void* ws = aligned_ws(workspace);
  st = cuda_status(launch_plan(assigned, weights, T, layer->num_experts, layer->top_k,
                               plan_out(ws, P, layer->num_shared), stream));
  if (st) return st;
  return gather_and_ffn(layer, hidden, T, out_bf16, out_f32, ws, P, stream, nullptr, peers);
}

int check_peers(const lynx_ep_peers_t* P) {
  if (!P || P->world_size < 1 || P->rank < 0 || P->rank >= P->world_size || P->tokens_per_rank < 1)
    return LYNX_ERR_SHAPE;
  if (!P->logits || !P->recv || !P->back || !P->flags || !P->logits_local || !P->recv_local || !P->back_local ||
      !P->flags_local || !P->counters || !P->epoch)
    return LYNX_ERR_SHAPE;
  return LYNX_OK;
}

// Experts the policy is expected to keep: K3's kernel choice only (no effect on results).
int kept_hint(const lynx_policy_t* policy, int decode, int N, int floor_keep) {
  if (policy && decode && policy->mode == LYNX_POLICY_LATENCY) return std::max(floor_keep, N - policy->drop_count);
  if (policy && decode && policy->mode == LYNX_POLICY_ACCURACY) return std::max(floor_keep, policy->freq_keep_budget);
  return N;
}

int moe_layer_impl(const lynx_layer_t* layer, const uint16_t* hidden, int T, int decode, const lynx_policy_t* policy,
                   uint16_t* out, const lynx_selection_t* sel, void* workspace, size_t workspace_bytes,
                   cudaStream_t stream, cudaEvent_t const* ev, const double* given_logits = nullptr) {
  int st = check_layer(layer, T);
  if (st) return st;
  if (!layer->router_wt && !given_logits) return LYNX_ERR_SHAPE;
  const int N = layer->num_experts, k = layer->top_k;
  int floor_keep = k;
  st = check_policy(policy, k, decode, &floor_keep);
  if (st) return st;
  const Plan P = plan_for(layer, T, true);
  if (!workspace || workspace_bytes < P.total) return LYNX_ERR_WORKSPACE;
  void* ws = aligned_ws(workspace);

  const double* logits = given_logits;
  record(ev, 0, stream);
  // N <= 8, T <= 256 (Mixtral): K0 + K1 + K2 as one fused launch (front_kernel).
  const bool fused = N <= 8 && T <= LYNX_SEG_ROWS && layer->num_shared == 0 && fused_front_enabled() &&
                     front_smem_bytes(T, N, k, layer->d_model) <= 48 * 1024 && (logits || layer->router_wt);
  // N > 16: the routing itself runs inside K0 (clusters per token) and K1
  // takes the selection as given; N <= 16 keeps it in K1's thread-per-token path.
  const bool route_in_k0 = !logits && N > 16 && route_in_k0_enabled();
  if (!logits && !route_in_k0 && !fused) {
    double* lg = at<double>(ws, P.logits);
    st = cuda_status(launch_router_logits(hidden, layer->router_wt, T, layer->d_model, N, lg, stream));
    if (st) return st;
    logits = lg;
  }

  SelectArgs a = select_args(logits, T, N, k, decode, policy, floor_keep);
  a.stage = select_can_stage(T, N, k, true) ? 1 : 0;
#define LYNX_PICK(field, off, type) ((sel && sel->field) ? sel->field : at<type>(ws, P.off))
  a.ids = LYNX_PICK(expert_ids, ids, int32_t);
  a.probs = LYNX_PICK(probs, probs, double);
  a.full = LYNX_PICK(full_probs, full, double);
  a.conf = LYNX_PICK(conf, conf, double);
  a.counts = LYNX_PICK(counts, counts, double);
  a.retained = LYNX_PICK(retained, retained, uint8_t);
  a.assigned = LYNX_PICK(assigned, assigned, int32_t);
  a.weights = LYNX_PICK(weights, weights, double);
  a.important = LYNX_PICK(important, important, uint8_t);
  a.flags = LYNX_PICK(flags, flags, int32_t);
#undef LYNX_PICK
  a.plan = plan_out(ws, P, layer->num_shared);
  a.routed_top = route_in_k0 ? 1 : 0;
  if (fused) {
    a.logits = nullptr;
    st = cuda_status(launch_front(a, hidden, layer->router_wt, layer->d_model, at<uint16_t>(ws, P.x_perm),
                                  at<int>(ws, P.sync), logits, stream));
    if (st) return st;
    record(ev, 1, stream);
    st = gather_and_ffn(layer, hidden, T, out, nullptr, ws, P, stream, ev ? ev + 2 : nullptr, nullptr,
                        kept_hint(policy, decode, N, floor_keep), true);
    record(ev, 5, stream);
    return st;
  }
  if (route_in_k0) {
    st = cuda_status(launch_router_route(hidden, layer->router_wt, T, layer->d_model, N, k, nullptr, a.full, a.ids,
                                         a.probs, stream));
    if (st) return st;
  }
  record(ev, 1, stream);
  st = cuda_status(launch_route_select(a, stream));
  if (st) return st;
  st = gather_and_ffn(layer, hidden, T, out, nullptr, ws, P, stream, ev ? ev + 2 : nullptr, nullptr,
                      kept_hint(policy, decode, N, floor_keep));
  record(ev, 5, stream);
  return st;
}

int route_select_common(SelectArgs a, const lynx_selection_t* out, cudaStream_t stream) {
  a.conf = out->conf;
  a.counts = out->counts;
  a.retained = out->retained;
  a.assigned = out->assigned;
  a.weights = out->weights;
  a.important = out->important;
  a.flags = out->flags;
  a.stage = select_can_stage(a.T, a.N, a.k, false) ? 1 : 0;
  return cuda_status(launch_route_select(a, stream));
}

}  // namespace

extern "C" {

int lynx_abi_version(void) { return kAbiVersion; }

const char* lynx_status_string(int status) {
  switch (status) {
    case LYNX_OK:
      return "ok";
    case LYNX_ERR_SHAPE:
      return "invalid shape";
    case LYNX_ERR_TOPK:
      return "k out of range";
    case LYNX_ERR_MIN_EXPERTS:
      return "min_experts must be >= top_k";
    case LYNX_ERR_RETAINED:
      return "retained set empty or out of range";
    case LYNX_ERR_TOKENS:
      return "token count mismatch";
    case LYNX_ERR_CUDA:
      return "CUDA error";
    case LYNX_ERR_UNSUPPORTED:
      return "shape outside build limits";
    case LYNX_ERR_WORKSPACE:
      return "workspace too small";
    case LYNX_ERR_CONFIG:
      return "invalid policy config";
    default:
      return "unknown status";
  }
}

int lynx_dispatch_caps(int T, int N, int k, int32_t* max_seg, int32_t* rows_cap) {
  if (T < 1 || N < 1 || k < 1) return LYNX_ERR_SHAPE;
  const Caps c = caps_for(T, N, k);
  if (max_seg) *max_seg = c.max_seg;
  if (rows_cap) *rows_cap = c.rows_cap;
  return LYNX_OK;
}

size_t lynx_moe_workspace_bytes(const lynx_layer_t* layer, int T) {
  if (!layer || T < 1) return 0;
  return plan_for(layer, T, true).total;
}

int lynx_router_logits(const uint16_t* hidden, const uint16_t* router_wt, int T, int d, int N, double* logits,
                       lynx_stream_t stream) {
  if (T < 1 || N < 1 || d < 8) return LYNX_ERR_SHAPE;
  if (d % 8 || N > LYNX_MAX_EXPERTS) return LYNX_ERR_UNSUPPORTED;
  return cuda_status(launch_router_logits(hidden, router_wt, T, d, N, logits, stream));
}

int lynx_route_select(const double* logits, int T, int N, int k, int decode, const lynx_policy_t* policy,
                      const lynx_selection_t* out, lynx_stream_t stream) {
  if (T < 1 || N < 1) return LYNX_ERR_SHAPE;
  if (k < 1 || k > N) return LYNX_ERR_TOPK;
  if (N > LYNX_MAX_EXPERTS || k > LYNX_MAX_TOPK || T > LYNX_MAX_TOKENS) return LYNX_ERR_UNSUPPORTED;
  if (!out || !out->expert_ids || !out->probs || !out->full_probs || !out->conf || !out->assigned ||
      !out->weights || !out->flags)
    return LYNX_ERR_SHAPE;
  int floor_keep = k;
  const int st = check_policy(policy, k, decode, &floor_keep);
  if (st) return st;
  SelectArgs a = select_args(logits, T, N, k, decode, policy, floor_keep);
  a.ids = out->expert_ids;
  a.probs = out->probs;
  a.full = out->full_probs;
  return route_select_common(a, out, stream);
}

int lynx_apply_policy(const int32_t* expert_ids, const double* probs, const double* full_probs, int T, int N, int k,
                      int decode, const lynx_policy_t* policy, const lynx_selection_t* out, lynx_stream_t stream) {
  if (T < 1 || N < 1) return LYNX_ERR_SHAPE;
  if (k < 1 || k > N) return LYNX_ERR_TOPK;
  if (N > LYNX_MAX_EXPERTS || k > LYNX_MAX_TOPK || T > LYNX_MAX_TOKENS) return LYNX_ERR_UNSUPPORTED;
  if (!out || !expert_ids || !probs || !full_probs || !out->conf || !out->assigned || !out->weights || !out->flags)
    return LYNX_ERR_SHAPE;
  int floor_keep = k;
  const int st = check_policy(policy, k, decode, &floor_keep);
  if (st) return st;
  SelectArgs a = select_args(nullptr, T, N, k, decode, policy, floor_keep);
  a.ids = const_cast<int32_t*>(expert_ids);
  a.probs = const_cast<double*>(probs);
  a.full = const_cast<double*>(full_probs);
  return route_select_common(a, out, stream);
}

int lynx_topk(const double* values, int T, int N, int k, int32_t* ids, double* out, lynx_stream_t stream) {
  if (T < 1 || N < 1) return LYNX_ERR_SHAPE;
  if (k < 1 || k > N) return LYNX_ERR_TOPK;
  if (N > LYNX_MAX_EXPERTS) return LYNX_ERR_UNSUPPORTED;
  return cuda_status(launch_topk(values, T, N, k, ids, out, stream));
}

int lynx_vote(const int32_t* expert_ids, int T, int k, int N, const lynx_policy_t* rank_weights, double* counts,
              lynx_stream_t stream) {
  if (T < 1 || N < 1 || k < 1) return LYNX_ERR_SHAPE;
  if (N > LYNX_MAX_EXPERTS || k > LYNX_MAX_TOPK) return LYNX_ERR_UNSUPPORTED;
  lynx_policy_t w{};
  if (rank_weights && rank_weights->n_rank_weights) {
    if (rank_weights->n_rank_weights != k) return LYNX_ERR_CONFIG;
    w = *rank_weights;
  }
  return cuda_status(launch_vote(expert_ids, T, k, N, w, counts, stream));
}

int lynx_remap(const int32_t* expert_ids, const double* full_probs, int T, int N, int k, const uint8_t* retained,
               int32_t* assigned, double* weights, int32_t* flags, lynx_stream_t stream) {
  if (T < 1 || N < 1) return LYNX_ERR_SHAPE;
  if (k < 1 || k > N) return LYNX_ERR_TOPK;
  if (N > LYNX_MAX_EXPERTS || k > LYNX_MAX_TOPK) return LYNX_ERR_UNSUPPORTED;
  if (!retained) return LYNX_ERR_RETAINED;
  return cuda_status(launch_remap(expert_ids, full_probs, T, N, k, retained, assigned, weights, flags, stream));
}

int lynx_permute(const int32_t* assigned, const double* weights, const uint16_t* hidden, int T, int N, int k, int d,
                 const lynx_dispatch_t* out, lynx_stream_t stream) {
  if (T < 1 || N < 1 || d < 8) return LYNX_ERR_SHAPE;
  if (k < 1 || k > N) return LYNX_ERR_TOPK;
  if (N > LYNX_MAX_EXPERTS || k > LYNX_MAX_TOPK || T > LYNX_MAX_TOKENS || d % 8) return LYNX_ERR_UNSUPPORTED;
  if (!out) return LYNX_ERR_SHAPE;
  const int sms = sm_count_cached();
  if (sms <= 0) return LYNX_ERR_CUDA;
  const Caps c = caps_for(T, N, k);
  PlanOut o{};
  o.enabled = 1;
  o.n_shared = 0;
  o.n_seg = out->n_seg;
  o.n_used = out->n_used;
  o.n_rows = out->n_rows;
  o.seg_expert = out->seg_expert;
  o.seg_row = out->seg_row;
  o.seg_count = out->seg_count;
  o.seg_order = nullptr;
  o.perm_token = out->perm_token;
  o.perm_weight = out->perm_weight;
  o.tok_rows = out->tok_rows;
  o.tok_weight = out->tok_weight;
  o.counters = nullptr;
  o.n_counters = 0;
  int st = cuda_status(launch_plan(assigned, weights, T, N, k, o, stream));
  if (st) return st;
  GatherArgs ga{};
  ga.hidden = hidden;
  ga.perm_token = out->perm_token;
  ga.n_rows = out->n_rows;
  ga.rows_cap = c.rows_cap;
  ga.d = d;
  ga.x_perm = out->x_perm;
  return cuda_status(launch_gather(ga, sms, stream));
}

int lynx_moe_forward(const lynx_layer_t* layer, const uint16_t* hidden, int T, const int32_t* assigned,
                     const double* weights, uint16_t* out, void* workspace, size_t workspace_bytes,
                     lynx_stream_t stream) {
  return moe_forward_common(layer, hidden, T, assigned, weights, out, nullptr, workspace, workspace_bytes, stream);
}

int lynx_moe_forward_partial(const lynx_layer_t* layer, const uint16_t* hidden, int T, const int32_t* assigned,
                             const double* weights, float* partial_out, void* workspace, size_t workspace_bytes,
                             lynx_stream_t stream) {
  return moe_forward_common(layer, hidden, T, assigned, weights, nullptr, partial_out, workspace, workspace_bytes,
                            stream);
}

int lynx_moe_layer(const lynx_layer_t* layer, const uint16_t* hidden, int T, int decode, const lynx_policy_t* policy,
                   uint16_t* out, const lynx_selection_t* sel, void* workspace, size_t workspace_bytes,
                   lynx_stream_t stream) {
  return moe_layer_impl(layer, hidden, T, decode, policy, out, sel, workspace, workspace_bytes, stream, nullptr);
}

int lynx_moe_layer_logits(const lynx_layer_t* layer, const uint16_t* hidden, const double* logits, int T, int decode,
                          const lynx_policy_t* policy, uint16_t* out, const lynx_selection_t* sel, void* workspace,
                          size_t workspace_bytes, lynx_stream_t stream) {
  if (!logits) return LYNX_ERR_SHAPE;
  return moe_layer_impl(layer, hidden, T, decode, policy, out, sel, workspace, workspace_bytes, stream, nullptr,
                        logits);
}

int lynx_moe_layer_profiled(const lynx_layer_t* layer, const uint16_t* hidden, int T, int decode,
                            const lynx_policy_t* policy, uint16_t* out, const lynx_selection_t* sel, void* workspace,
                            size_t workspace_bytes, lynx_stream_t stream, void* const* events, int n_events) {
  if (!events || n_events != LYNX_PROFILE_EVENTS) return LYNX_ERR_SHAPE;
  return moe_layer_impl(layer, hidden, T, decode, policy, out, sel, workspace, workspace_bytes, stream,
                        reinterpret_cast<cudaEvent_t const*>(events));
}

int lynx_moe_ffn_kernel(const lynx_layer_t* layer, int T, int decode, const lynx_policy_t* policy,
                        int32_t* stage_rows) {
  int st = check_layer(layer, T);
  if (st) return st;
  int floor_keep = layer->top_k;
  st = check_policy(policy, layer->top_k, decode, &floor_keep);
  if (st) return st;
  const Geometry g = geometry(layer, T);
  const int N = layer->num_experts;
  const int kept = std::min(kept_hint(policy, decode, N, floor_keep), N);
  if (stage_rows) *stage_rows = g.bn;
  return ffn_use_pair(g.bn, T * layer->top_k / kept) ? 1 : 0;
}

int lynx_pack_w13(const uint16_t* w1, const uint16_t* w3, int N, int ff, int d, uint16_t* w13,
                  lynx_stream_t stream) {
  if (N < 1 || ff < 1 || d < 1) return LYNX_ERR_SHAPE;
  return cuda_status(launch_pack_w13(w1, w3, N, ff, d, w13, stream));
}

// q scratch | fused-router chunk partials (d <= 8192: <= 8 chunks of N+1 <= 17) | row counters
constexpr int kRouterChunksMax = 8;

size_t lynx_attention_workspace_bytes(int rows, int d_head) {
  if (rows < 1 || d_head < 1) return 0;
  const size_t q = align_up(sizeof(float) * static_cast<size_t>(rows) * d_head, 256);
  const size_t part = align_up(sizeof(float) * static_cast<size_t>(rows) * kRouterChunksMax *
                                   (LYNX_MAX_FUSED_ROUTER + 1), 256);
  return q + part + sizeof(int) * static_cast<size_t>(rows) + 512;
}

int lynx_attention(const lynx_attention_t* attn, const uint16_t* h_in, int B, int Tn, int norm_input,
                   const int32_t* pos, uint16_t* h_out, void* workspace, size_t workspace_bytes,
                   lynx_stream_t stream) {
  if (!attn || !h_in || !h_out || !pos || B < 1 || Tn < 1) return LYNX_ERR_SHAPE;
  if (attn->d_model < 8 || attn->d_head < 1 || attn->max_len < Tn) return LYNX_ERR_SHAPE;
  if (!attn->wqkv || !attn->wo || !attn->k_cache || !attn->v_cache) return LYNX_ERR_SHAPE;
  if (attn->d_model % 8 || attn->d_head > LYNX_MAX_DHEAD ||
      attn_out_smem(attn->d_model, attn->d_head, attn->max_len) > 200 * 1024)
    return LYNX_ERR_UNSUPPORTED;
  if (!workspace || workspace_bytes < lynx_attention_workspace_bytes(B * Tn, attn->d_head)) return LYNX_ERR_WORKSPACE;
  AttnArgs a{};
  a.h_in = h_in;
  a.wqkv = attn->wqkv;
  a.wo = attn->wo;
  a.kcache = attn->k_cache;
  a.vcache = attn->v_cache;
  a.q = static_cast<float*>(aligned_ws(workspace));
  a.pos = pos;
  a.B = B;
  a.Tn = Tn;
  a.d = attn->d_model;
  a.dh = attn->d_head;
  a.max_len = attn->max_len;
  a.norm_input = norm_input ? 1 : 0;
  a.h_out = h_out;
  a.router_wt = attn->router_wt;
  a.N = attn->num_experts;
  a.logits = attn->logits;
  a.rpart = nullptr;
  a.row_arrivals = nullptr;
  if (attn->router_wt) {
    if (!attn->logits || attn->num_experts < 1) return LYNX_ERR_SHAPE;
    if (attn->num_experts > LYNX_MAX_FUSED_ROUTER || attn->d_model > kRouterChunksMax * 1024)
      return LYNX_ERR_UNSUPPORTED;
    const int rows = B * Tn;
    char* base = static_cast<char*>(aligned_ws(workspace));
    const size_t q = align_up(sizeof(float) * static_cast<size_t>(rows) * attn->d_head, 256);
    const size_t part = align_up(sizeof(float) * static_cast<size_t>(rows) * kRouterChunksMax *
                                     (LYNX_MAX_FUSED_ROUTER + 1), 256);
    a.rpart = reinterpret_cast<float*>(base + q);
    a.row_arrivals = reinterpret_cast<int*>(base + q + part);
  }
  return cuda_status(launch_attention(a, stream));
}

int lynx_advance_position(int32_t* pos, int by, lynx_stream_t stream) {
  if (!pos) return LYNX_ERR_SHAPE;
  return cuda_status(launch_advance_position(pos, by, stream));
}

int lynx_trace_append(const lynx_trace_ring_t* ring, const int32_t* pos, int layer, const lynx_selection_t* sel,
                      lynx_stream_t stream) {
  if (!ring || !pos || !sel || ring->capacity < 1 || layer < 0 || layer >= ring->num_layers) return LYNX_ERR_SHAPE;
  if (ring->T < 1 || ring->k < 1 || ring->N < 1) return LYNX_ERR_SHAPE;
  if (!ring->positions || !ring->original || !ring->assigned || !ring->weights || !ring->conf || !ring->retained ||
      !ring->important || !ring->flags)
    return LYNX_ERR_SHAPE;
  if (!sel->expert_ids || !sel->full_probs || !sel->assigned || !sel->weights || !sel->retained || !sel->flags)
    return LYNX_ERR_SHAPE;
  return cuda_status(launch_trace_append(*ring, pos, layer, *sel, stream));
}

int lynx_ep_pack(const uint16_t* hidden_local, const int32_t* assigned, int T_local, int k, int N, int G, int d,
                 int rank, uint16_t* send, lynx_stream_t stream) {
  if (T_local < 1 || G < 1 || N % G || rank < 0 || rank >= G || d % 8) return LYNX_ERR_SHAPE;
  return cuda_status(launch_ep_pack(hidden_local, assigned, T_local, k, N, G, d, rank, send, stream));
}

int lynx_ep_local_mask(const int32_t* assigned, const double* weights, int T, int k, int N, int G, int rank,
                       int32_t* assigned_local, double* weights_local, lynx_stream_t stream) {
  if (T < 1 || G < 1 || N % G || rank < 0 || rank >= G) return LYNX_ERR_SHAPE;
  return cuda_status(launch_ep_local_mask(assigned, weights, T, k, N, G, rank, assigned_local, weights_local, stream));
}

int lynx_ep_combine(const uint16_t* hidden_local, const float* recv_partial, int T_local, int G, int d,
                    uint16_t* out, lynx_stream_t stream) {
  if (T_local < 1 || G < 1 || d % 2) return LYNX_ERR_SHAPE;
  return cuda_status(launch_ep_combine(hidden_local, recv_partial, T_local, G, d, out, stream));
}

int lynx_enable_peer_access(int peer_device) {
  int cur = 0;
  if (cudaGetDevice(&cur) != cudaSuccess) return LYNX_ERR_CUDA;
  if (peer_device == cur) return LYNX_OK;
  int can = 0;
  if (cudaDeviceCanAccessPeer(&can, cur, peer_device) != cudaSuccess) return LYNX_ERR_CUDA;
  if (!can) return LYNX_ERR_UNSUPPORTED;
  const cudaError_t e = cudaDeviceEnablePeerAccess(peer_device, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();  // clear the sticky-free "already enabled" status
    return LYNX_OK;
  }
  return cuda_status(e);
}

int lynx_ep_p2p_route(const uint16_t* router_wt, const uint16_t* hidden_local, int d, int N,
                      const lynx_ep_peers_t* peers, lynx_stream_t stream) {
  int st = check_peers(peers);
  if (st) return st;
  if (!router_wt || !hidden_local || d < 8 || N < 1 || N % peers->world_size) return LYNX_ERR_SHAPE;
  if (d % 8 || N > LYNX_MAX_EXPERTS || peers->world_size * peers->tokens_per_rank > LYNX_MAX_TOKENS)
    return LYNX_ERR_UNSUPPORTED;
  // K0 stores this rank's logits rows into every rank's buffer and signals
  EpLink put{};
  put.enabled = 1;
  put.P = *peers;
  return cuda_status(launch_router_logits(hidden_local, router_wt, peers->tokens_per_rank, d, N,
                                          peers->logits_local, stream, &put));
}

int lynx_ep_p2p_dispatch(const uint16_t* hidden_local, int N, int k, int d, int decode, const lynx_policy_t* policy,
                         const lynx_selection_t* sel, const lynx_ep_peers_t* peers, lynx_stream_t stream) {
  int st = check_peers(peers);
  if (st) return st;
  const int T = peers->world_size * peers->tokens_per_rank;
  if (!hidden_local || N < 1 || d < 8 || N % peers->world_size) return LYNX_ERR_SHAPE;
  if (k < 1 || k > N) return LYNX_ERR_TOPK;
  if (N > LYNX_MAX_EXPERTS || k > LYNX_MAX_TOPK || T > LYNX_MAX_TOKENS || d % 8) return LYNX_ERR_UNSUPPORTED;
  if (!sel || !sel->expert_ids || !sel->probs || !sel->full_probs || !sel->conf || !sel->assigned ||
      !sel->weights || !sel->flags)
    return LYNX_ERR_SHAPE;
  int floor_keep = k;
  st = check_policy(policy, k, decode, &floor_keep);
  if (st) return st;
  SelectArgs a = select_args(peers->logits_local, T, N, k, decode, policy, floor_keep);
  a.ep.enabled = 1;  // K1 waits for every rank's logits itself
  a.ep.kind = kSigLogits;
  a.ep.P = *peers;
  a.ids = sel->expert_ids;
  a.probs = sel->probs;
  a.full = sel->full_probs;
  st = route_select_common(a, sel, stream);
  if (st) return st;
  return cuda_status(launch_ep_dispatch(*peers, hidden_local, sel->assigned, k, N, d, stream));
}

int lynx_ep_p2p_expert(const lynx_layer_t* local_layer, int N, const int32_t* assigned, const double* weights,
                       int32_t* assigned_local, double* weights_local, const lynx_ep_peers_t* peers, void* workspace,
                       size_t workspace_bytes, lynx_stream_t stream) {
  int st = check_peers(peers);
  if (st) return st;
  if (!local_layer || !assigned || !weights || !assigned_local || !weights_local) return LYNX_ERR_SHAPE;
  const int G = peers->world_size, T = G * peers->tokens_per_rank;
  if (N % G || local_layer->num_experts * G != N) return LYNX_ERR_SHAPE;
  // the gather kernel (K2) waits for every rank's rows itself
  st = cuda_status(launch_ep_local_mask(assigned, weights, T, local_layer->top_k, N, G, peers->rank, assigned_local,
                                        weights_local, stream));
  if (st) return st;
  return moe_forward_common(local_layer, peers->recv_local, T, assigned_local, weights_local, nullptr, nullptr,
                            workspace, workspace_bytes, stream, peers);
}

int lynx_ep_p2p_combine(const uint16_t* hidden_local, int d, uint16_t* out, const lynx_ep_peers_t* peers,
                        lynx_stream_t stream) {
  const int st = check_peers(peers);
  if (st) return st;
  if (!hidden_local || !out || d < 2 || d % 2) return LYNX_ERR_SHAPE;
  return cuda_status(launch_ep_p2p_combine(*peers, hidden_local, d, out, stream));
}

}  // extern "C"
