/*
 * lynx_b200.h -- C ABI of the B200-native Lynx MoE decode hot path.
 *
 * The reference (moetrim, /root/reference/pkg/src/moetrim) is a pure-Python
 * package with no FFI; its "operator API" for this path is three Python
 * calls, which this library replaces one-for-one:
 *
 *   route_batch(logits, k)                    router.py:174-187
 *   apply_policy(selection, phase, config)    policy.py:341-350
 *     (latency_policy 232-264, accuracy_policy 287-338,
 *      remap_tokens 151-212, full_retain_mask 215-229)
 *   forward_layer(hidden, model, layer, mask) simulator.py:86-113
 *     (router_logits 82-83, rms_norm 26-27, expert_mlp 77-79)
 *
 * Python binds these entry points with ctypes
 * (paper_2411_08982_b200/_native.py); INTEGRATION.md shows the binding.
 *
 * Conventions
 *   - Every pointer argument is a DEVICE pointer owned by the caller,
 *     except the const struct pointers (lynx_policy_t, lynx_layer_t,
 *     lynx_selection_t, lynx_dispatch_t), which are host structs holding
 *     device pointers.  The library never allocates or frees and keeps no
 *     global mutable state; calls are re-entrant and stream-ordered.
 *   - bf16 tensors are passed as uint16_t* (raw bfloat16 bits).
 *   - Return value: LYNX_OK (0) or a negative lynx_status.  Preconditions
 *     the reference rejects with ValidationError map to distinct codes;
 *     data-dependent conditions found on the device (non-finite logits,
 *     zero probability mass, clipped drop) are reported through the
 *     caller's int32 `flags` word, read back only when the caller asks.
 *   - No host synchronisation inside any call; all calls are capturable
 *     into CUDA graphs.
 *   - Build target: sm_100a only (B200).
 */
#ifndef LYNX_B200_H
#define LYNX_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st *lynx_stream_t; /* == cudaStream_t */

enum lynx_status {
  LYNX_OK = 0,
  LYNX_ERR_SHAPE = -1,         /* bad T/N/d/ff, RoutingLogits shape (router.py:67-70) */
  LYNX_ERR_TOPK = -2,          /* k outside [1, N] (router.py:176-179) */
  LYNX_ERR_MIN_EXPERTS = -3,   /* min_experts < top_k (policy.py:61-64) */
  LYNX_ERR_RETAINED = -4,      /* empty / out-of-range retained (policy.py:164-167) */
  LYNX_ERR_TOKENS = -5,        /* mask/hidden token mismatch (simulator.py:97-100) */
  LYNX_ERR_CUDA = -6,          /* a CUDA launch or driver call failed */
  LYNX_ERR_UNSUPPORTED = -7,   /* shape outside this build's limits (see LYNX_MAX_*) */
  LYNX_ERR_WORKSPACE = -8,     /* workspace smaller than lynx_*_workspace_bytes() */
  LYNX_ERR_CONFIG = -9         /* invalid PolicyConfig field (policy.py:40-55) */
};

/* Device flag bits (int32 word written by the selection kernel). */
#define LYNX_FLAG_CLIPPED 1      /* ExpertMask.clipped (policy.py:100, 250-251, 337) */
#define LYNX_FLAG_NONFINITE 2    /* logits contain NaN/Inf (router.py:71-72) */
#define LYNX_FLAG_ZERO_MASS 4    /* token has zero mass on assigned experts (policy.py:206-209) */

/* Build limits. */
#define LYNX_MAX_EXPERTS 64
#define LYNX_MAX_TOPK 8
#define LYNX_MAX_SHARED 4         /* always-on shared experts per layer (DeepSeek-MoE style) */
#define LYNX_MAX_DHEAD 64         /* attention stand-in head width */
#define LYNX_MAX_TOKENS 4096
#define LYNX_SEG_ROWS 256        /* max token rows one expert segment feeds one MMA */

enum lynx_policy_mode { LYNX_POLICY_NONE = 0, LYNX_POLICY_LATENCY = 1, LYNX_POLICY_ACCURACY = 2 };
enum lynx_conf_metric { LYNX_CONF_TOP1 = 0, LYNX_CONF_MARGIN = 1 };
enum lynx_activation { LYNX_ACT_SWIGLU = 0, LYNX_ACT_TANH2 = 1 };

/* PolicyConfig (policy.py:26-37).  mode NONE = full_retain_mask. */
typedef struct lynx_policy {
  int32_t mode;
  int32_t drop_count;
  double confidence_threshold;
  int32_t sample_threshold;
  int32_t min_experts;        /* 0 = unset -> resolves to top_k (policy.py:57-65) */
  int32_t freq_keep_budget;
  int32_t confidence_metric;  /* lynx_conf_metric */
  int32_t n_rank_weights;     /* 0 = one vote per slot, else == top_k */
  int32_t reserved;
  double rank_weights[LYNX_MAX_TOPK];
} lynx_policy_t;

/* ExpertSelection + ExpertMask outputs (router.py:84-123, policy.py:83-113).
 * Any pointer except expert_ids/assigned/weights/flags may be NULL. */
typedef struct lynx_selection {
  int32_t *expert_ids;  /* [T,k] rank order, ties -> smaller index */
  double *probs;        /* [T,k] */
  double *full_probs;   /* [T,N] float64 softmax */
  double *conf;         /* [T]   confidence(metric) */
  double *counts;       /* [N]   vote tally the policy used */
  uint8_t *retained;    /* [N]   1 = expert retained */
  int32_t *assigned;    /* [T,k] remap_assigned */
  double *weights;      /* [T,k] remap_weights (renormalised) */
  uint8_t *important;   /* [T]   accuracy policy's important tokens */
  int32_t *flags;       /* [1]   LYNX_FLAG_* */
} lynx_selection_t;

/* One MoE layer's static description (weights are borrowed device memory). */
typedef struct lynx_layer {
  int32_t num_experts;    /* N */
  int32_t top_k;          /* k */
  int32_t d_model;        /* d, multiple of 8 */
  int32_t d_ff;           /* ff, multiple of 8 */
  int32_t activation;     /* lynx_activation */
  /* S shared experts (0..LYNX_MAX_SHARED): experts N..N+S-1 of w13/w2, applied
   * to every token with gate weight 1 after the routed experts, outside the
   * router and the policy.  The reference has none; 0
   * reproduces forward_layer exactly. */
  int32_t num_shared;
  /* SWIGLU: packed gate/up [N+S, 2*ceil64(ff), d] (lynx_pack_w13 layout).
   * TANH2:  w1^T [N+S, ff, d] (reference w1 is [N, d, ff], simulator.py:40). */
  const uint16_t *w13;
  const uint16_t *w2;        /* [N+S, d, ff]  (reference w2 [N, ff, d] transposed) */
  const uint16_t *router_wt; /* [N, d]      (reference router_w [d, N] transposed); may be NULL
                                if the caller routes itself */
} lynx_layer_t;

/* Dispatch produced by lynx_permute (simulator.py:104-112 order: experts
 * ascending, token rows ascending, duplicate slots of a token merged). */
typedef struct lynx_dispatch {
  int32_t *n_seg;       /* [1]  number of segments (used experts split at LYNX_SEG_ROWS) */
  int32_t *n_used;      /* [1]  number of used experts */
  int32_t *n_rows;      /* [1]  permuted rows in use (each expert padded to 16) */
  int32_t *seg_expert;  /* [max_seg] expert id of each segment */
  int32_t *seg_row;     /* [max_seg] first permuted row (16-aligned) */
  int32_t *seg_count;   /* [max_seg] token rows in the segment */
  int32_t *perm_token;  /* [rows_cap] source token of each permuted row, -1 = padding */
  float *perm_weight;   /* [rows_cap] merged gate weight of each permuted row */
  int32_t *tok_rows;    /* [T,k] permuted rows of token t, experts ascending, -1 padded */
  float *tok_weight;    /* [T,k] matching merged weights */
  uint16_t *x_perm;     /* [rows_cap, d] gathered hidden rows (bf16), padding rows zero */
} lynx_dispatch_t;

/* ---- sizes ---------------------------------------------------------- */
int lynx_abi_version(void);
const char *lynx_status_string(int status);
/* Upper bounds the caller uses to size dispatch buffers. */
int lynx_dispatch_caps(int T, int N, int k, int32_t *max_seg, int32_t *rows_cap);
/* Workspace for lynx_moe_forward / lynx_moe_layer. */
size_t lynx_moe_workspace_bytes(const lynx_layer_t *layer, int T);

/* ---- K0: router GEMV with fused RMSNorm (simulator.py:26-27, 82-83) -- */
int lynx_router_logits(const uint16_t *hidden, const uint16_t *router_wt, int T, int d, int N,
                       double *logits, lynx_stream_t stream);

/* ---- K1: route_batch + apply_policy (router.py:174-187, policy.py:341-350) */
int lynx_route_select(const double *logits, int T, int N, int k, int decode,
                      const lynx_policy_t *policy, const lynx_selection_t *out,
                      lynx_stream_t stream);

/* apply_policy / latency_policy / accuracy_policy / full_retain_mask on an
 * existing selection (policy.py:215-350).  expert_ids/probs/full_probs are
 * inputs ([T,k], [T,k], [T,N]); out->expert_ids/probs/full_probs are ignored.
 * policy NULL or mode NONE = full_retain_mask (also fills conf). */
int lynx_apply_policy(const int32_t *expert_ids, const double *probs, const double *full_probs,
                      int T, int N, int k, int decode, const lynx_policy_t *policy,
                      const lynx_selection_t *out, lynx_stream_t stream);

/* top_k_select (router.py:157-171) on float64 rows [T,N]: (value desc, index asc). */
int lynx_topk(const double *values, int T, int N, int k, int32_t *ids, double *out,
              lynx_stream_t stream);

/* vote_expert_frequencies (policy.py:116-138); policy may carry rank weights. */
int lynx_vote(const int32_t *expert_ids, int T, int k, int N, const lynx_policy_t *rank_weights,
              double *counts, lynx_stream_t stream);

/* remap_tokens on an arbitrary retained mask (policy.py:151-212). */
int lynx_remap(const int32_t *expert_ids, const double *full_probs, int T, int N, int k,
               const uint8_t *retained, int32_t *assigned, double *weights, int32_t *flags,
               lynx_stream_t stream);

/* ---- K2: dispatch plan (bitmap histogram + scan, simulator.py:104-112)
 * and gather of the token rows into expert segments */
int lynx_permute(const int32_t *assigned, const double *weights, const uint16_t *hidden,
                 int T, int N, int k, int d, const lynx_dispatch_t *out, lynx_stream_t stream);

/* ---- K3: grouped expert FFN over used experts + fused weighted combine --
 * forward_layer(hidden, model, layer, mask) for a given mask. */
int lynx_moe_forward(const lynx_layer_t *layer, const uint16_t *hidden, int T,
                     const int32_t *assigned, const double *weights, uint16_t *out,
                     void *workspace, size_t workspace_bytes, lynx_stream_t stream);

/* Same as lynx_moe_forward but writes the f32 sum of expert outputs WITHOUT
 * the residual; assigned entries < 0 are skipped (expert-parallel partial).
 * Shared experts are not part of an expert-parallel shard (num_shared must be 0). */
int lynx_moe_forward_partial(const lynx_layer_t *layer, const uint16_t *hidden, int T,
                             const int32_t *assigned, const double *weights, float *partial_out,
                             void *workspace, size_t workspace_bytes, lynx_stream_t stream);

/* ---- whole decode layer: K0 -> K1 -> K2 -> K3 -------------------------
 * _apply_routing + forward_layer (simulator.py:245-266, 86-113).
 * `sel` may be NULL; when given, the selection/mask outputs are copied out.
 * For N <= 8, T <= LYNX_SEG_ROWS and no shared experts, K0..K2 run as one
 * fused launch synchronised by a grid barrier whose words live in the
 * workspace: zero-fill the workspace once before its first use (every call
 * leaves those words ready for the next; a workspace serves calls in stream
 * order). */
int lynx_moe_layer(const lynx_layer_t *layer, const uint16_t *hidden, int T, int decode,
                   const lynx_policy_t *policy, uint16_t *out, const lynx_selection_t *sel,
                   void *workspace, size_t workspace_bytes, lynx_stream_t stream);

/* lynx_moe_layer with the router logits given (f64 [T, N], e.g. from the
 * fused router of lynx_attention): K1..K4 only. */
int lynx_moe_layer_logits(const lynx_layer_t *layer, const uint16_t *hidden, const double *logits, int T,
                          int decode, const lynx_policy_t *policy, uint16_t *out, const lynx_selection_t *sel,
                          void *workspace, size_t workspace_bytes, lynx_stream_t stream);

/* lynx_moe_layer that also records caller-created CUDA events (cudaEvent_t)
 * on `stream` around each kernel: events[0] before K0 (router), [1] before
 * K1 (select + plan), [2] before K2 (gather), [3] before K3 (expert FFN with
 * the fused combine), [4] after K3, [5] at the end.  n_events must be
 * LYNX_PROFILE_EVENTS.  Event records serialise the programmatic launches,
 * so bench.py uses this only to attribute time to kernels. */
#define LYNX_PROFILE_EVENTS 6
int lynx_moe_layer_profiled(const lynx_layer_t *layer, const uint16_t *hidden, int T, int decode,
                            const lynx_policy_t *policy, uint16_t *out, const lynx_selection_t *sel,
                            void *workspace, size_t workspace_bytes, lynx_stream_t stream,
                            void *const *events, int n_events);

/* Which K3 kernel lynx_moe_layer launches for this layer, batch and policy:
 * 0 = ffn_kernel (one CTA per SM, tcgen05 cta_group::1), 1 = ffn_pair_kernel
 * (CTA pairs, cta_group::2, for wide expert segments); negative = lynx_status.
 * *stage_rows (may be NULL) receives the launch's activation tile width. */
int lynx_moe_ffn_kernel(const lynx_layer_t *layer, int T, int decode, const lynx_policy_t *policy,
                        int32_t *stage_rows);

/* Pack HF-layout gate/up projections w1, w3 [N, ff, d] into the
 * interleaved w13 layout the SwiGLU kernel streams. */
int lynx_pack_w13(const uint16_t *w1, const uint16_t *w3, int N, int ff, int d, uint16_t *w13,
                  lynx_stream_t stream);

/* ---- decode stack around the layer -------------------
 * The reference model's single-head attention stand-in plus its residual,
 * h_out = h + attention(layer, h)  (simulator.py:308-326, 333), with a
 * per-layer KV cache.  A chunk of Tn new tokens per sequence (B sequences;
 * rows b*Tn+i of h_in/h_out) occupies cache positions *pos .. *pos+Tn-1 and
 * attends causally (simulator.py:318-321).  `pos` is device memory so a
 * captured decode step replays step after step; lynx_advance_position adds
 * `by` to it on the stream.  norm_input = 1 feeds rms_norm(h_in) as the
 * layer input (the decode step's rms_norm(prev), simulator.py:353). */
typedef struct lynx_attention {
  int32_t d_model;          /* d (multiple of 8) */
  int32_t d_head;           /* dh <= LYNX_MAX_DHEAD */
  int32_t max_len;          /* cache capacity in positions */
  int32_t num_experts;      /* N of the fused router (router_wt != NULL), <= LYNX_MAX_FUSED_ROUTER */
  const uint16_t *wqkv;     /* [3*dh, d] bf16: wq^T, wk^T, wv^T (reference [d, dh] each, simulator.py:35-37) */
  const uint16_t *wo;       /* [dh, d] bf16 (reference wo, simulator.py:38) */
  float *k_cache;           /* [B, max_len, dh] f32 */
  float *v_cache;           /* [B, max_len, dh] f32 */
  /* Optional router fused into the attention output: the
   * next MoE layer's logits rms_norm(h_out) . router (simulator.py:82-83)
   * are produced by the same kernel that produces h_out, written to
   * logits [B*Tn, N] f64; feed them to lynx_moe_layer_logits.  NULL = off. */
  const uint16_t *router_wt;  /* [N, d] bf16 */
  double *logits;             /* [B*Tn, N] f64 */
} lynx_attention_t;

#define LYNX_MAX_FUSED_ROUTER 16

/* q scratch plus, with the fused router, per-chunk partials and row counters. */
size_t lynx_attention_workspace_bytes(int rows, int d_head);
int lynx_attention(const lynx_attention_t *attn, const uint16_t *h_in, int B, int Tn, int norm_input,
                   const int32_t *pos, uint16_t *h_out, void *workspace, size_t workspace_bytes,
                   lynx_stream_t stream);
int lynx_advance_position(int32_t *pos, int by, lynx_stream_t stream);

/* ---- device trace ring -------------------------------
 * Routing events of a captured decode step are appended on the device, so
 * tracing costs no host sync per step; the host later serialises the ring
 * into the reference's trace JSONL (trace.py:24-35, 81-125).  Slot =
 * (*pos) % capacity, the slot's cache position goes to positions[slot].
 * conf is the top-1 confidence the reference traces (trace.py:90). */
typedef struct lynx_trace_ring {
  int32_t capacity;       /* steps held */
  int32_t num_layers;     /* L */
  int32_t T, k, N, reserved;
  int32_t *positions;     /* [cap] */
  int32_t *original;      /* [cap, L, T, k] remap_original */
  int32_t *assigned;      /* [cap, L, T, k] remap_assigned */
  double *weights;        /* [cap, L, T, k] remap_weights */
  double *conf;           /* [cap, L, T]    top-1 confidence */
  uint8_t *retained;      /* [cap, L, N] */
  uint8_t *important;     /* [cap, L, T] */
  int32_t *flags;         /* [cap, L]       LYNX_FLAG_* */
} lynx_trace_ring_t;

/* sel: the layer's selection outputs (expert_ids, full_probs, assigned,
 * weights, retained, important, flags must be set). */
int lynx_trace_append(const lynx_trace_ring_t *ring, const int32_t *pos, int layer,
                      const lynx_selection_t *sel, lynx_stream_t stream);

/* ---- expert parallel helpers -------------------------
 * Rank r of G owns experts [r*N/G, (r+1)*N/G).  Dispatch rows are sent with
 * a fixed per-peer capacity of T_local rows so the NCCL all-to-all needs no
 * count exchange; every rank holds the identical global selection. */
int lynx_ep_pack(const uint16_t *hidden_local, const int32_t *assigned, int T_local, int k,
                 int N, int G, int d, int rank, uint16_t *send, lynx_stream_t stream);
int lynx_ep_local_mask(const int32_t *assigned, const double *weights, int T, int k, int N,
                       int G, int rank, int32_t *assigned_local, double *weights_local,
                       lynx_stream_t stream);
int lynx_ep_combine(const uint16_t *hidden_local, const float *recv_partial, int T_local, int G,
                    int d, uint16_t *out, lynx_stream_t stream);

/* ---- expert parallel over NVLink peer memory -----------
 * The fused alternative to the NCCL path above: the logits all-gather, the
 * token dispatch and the partial-sum return are stores into the peers'
 * buffers issued by the kernels that produce the data (router, dispatch,
 * K4), each followed by a release signal per peer; consumers acquire-wait.
 * Buffers are symmetric (same layout on every rank, e.g. from
 * torch.distributed._symmetric_memory); the pointer arrays below are DEVICE
 * arrays of G pointers, the *_local fields this rank's own buffers.
 *   logits [G*Tl, N] f64    recv [G*Tl, d] bf16    back [G*Tl, d] f32
 *   flags  [3*G] int32 (zero-initialised)
 * counters (4 int32) and epoch (1 int32) are this rank's, zero-initialised.
 * A layer is the four calls in order (route -> dispatch -> expert ->
 * combine); each call only waits at its start for the previous call's data
 * of every peer, so ranks may also be driven phase by phase (tests run G
 * ranks on one GPU that way). */
typedef struct lynx_ep_peers {
  int32_t world_size;       /* G */
  int32_t rank;
  int32_t tokens_per_rank;  /* Tl */
  int32_t reserved;
  double *const *logits;
  uint16_t *const *recv;
  float *const *back;
  int32_t *const *flags;
  double *logits_local;
  uint16_t *recv_local;
  float *back_local;
  int32_t *flags_local;
  int32_t *counters;
  int32_t *epoch;
} lynx_ep_peers_t;

/* Let kernels on the calling thread's current device load/store memory of
 * device `peer_device` (cudaDeviceEnablePeerAccess; already enabled or the
 * same device: LYNX_OK; no P2P path: LYNX_ERR_UNSUPPORTED).  Peer buffers
 * opened over CUDA IPC are mapped for the owner's device only, so every rank
 * calls this for every other rank's device before the first layer. */
int lynx_enable_peer_access(int peer_device);

/* K0 on the local rows into logits_local rows rank*Tl.., then to every peer. */
int lynx_ep_p2p_route(const uint16_t *router_wt, const uint16_t *hidden_local, int d, int N,
                      const lynx_ep_peers_t *peers, lynx_stream_t stream);
/* Wait for every peer's logits; K1 (route + Lynx policy) on the global batch
 * into `sel` (identical on every rank); dispatch this rank's needed rows into
 * the owners' recv buffers. */
int lynx_ep_p2p_dispatch(const uint16_t *hidden_local, int N, int k, int d, int decode,
                         const lynx_policy_t *policy, const lynx_selection_t *sel,
                         const lynx_ep_peers_t *peers, lynx_stream_t stream);
/* Wait for every peer's rows; this rank's experts (local_layer: its N/G
 * experts, router_wt unused) over recv with the global mask renumbered into
 * assigned_local/weights_local [G*Tl, k] (caller buffers); K4 stores each
 * token's partial sum into its owner's back buffer. */
int lynx_ep_p2p_expert(const lynx_layer_t *local_layer, int N, const int32_t *assigned, const double *weights,
                       int32_t *assigned_local, double *weights_local, const lynx_ep_peers_t *peers,
                       void *workspace, size_t workspace_bytes, lynx_stream_t stream);
/* Wait for every peer's partial sums; out = hidden + sum over ranks (rank
 * order = experts ascending); advances the epoch. */
int lynx_ep_p2p_combine(const uint16_t *hidden_local, int d, uint16_t *out, const lynx_ep_peers_t *peers,
                        lynx_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* LYNX_B200_H */
