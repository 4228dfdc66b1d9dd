"""paper_2411_08982_b200 -- B200-native Lynx MoE decode hot path.

Drop-in for the hot path of moetrim (arXiv 2411.08982 "Lynx"): routing,
batch-aware expert retention, re-routing, dispatch, grouped expert FFN over
the used experts only, and the weighted combine -- hand-written sm_100a
CUDA behind the C ABI in include/lynx_b200.h.  The public names mirror
moetrim/__init__.py:35-73 for this path.
"""

from ._version import __version__
from .errors import NativeLibraryError, TraceFormatError, ValidationError
from .decode import AttentionWeights, DecodeStack, SimResult, attention_from_reference, build_attention
from .moe import (
    LynxMoELayer,
    MoEWeights,
    build_swiglu_model,
    forward_layer,
    forward_partial,
    from_hf_swiglu,
    from_reference,
    pack_w13,
    router_logits,
    unpack_w13,
)
from .policy import (
    POLICY_MODES,
    ExpertMask,
    PolicyConfig,
    VoteTally,
    accuracy_policy,
    apply_policy,
    full_retain_mask,
    latency_policy,
    remap_tokens,
    select_important_tokens,
    vote_expert_frequencies,
)
from .router import (
    ExpertSelection,
    MoEModelSpec,
    Phase,
    RoutingLogits,
    confidence,
    route_batch,
    softmax_probs,
    top_k_select,
)

from .trace import (
    MaskRecord,
    TraceRecord,
    TraceRecorder,
    masks_path_for,
    read_masks_jsonl,
    read_trace_jsonl,
    write_masks_jsonl,
    write_trace_jsonl,
)

__all__ = [
    "AttentionWeights", "DecodeStack", "SimResult", "attention_from_reference", "build_attention",
    "MaskRecord", "TraceRecord", "TraceRecorder", "masks_path_for", "read_masks_jsonl", "read_trace_jsonl",
    "write_masks_jsonl", "write_trace_jsonl",
    "__version__", "NativeLibraryError", "TraceFormatError", "ValidationError",
    "LynxMoELayer", "MoEWeights", "build_swiglu_model", "forward_layer", "forward_partial",
    "from_hf_swiglu", "from_reference", "pack_w13", "router_logits", "unpack_w13",
    "POLICY_MODES", "ExpertMask", "PolicyConfig", "VoteTally", "accuracy_policy", "apply_policy",
    "full_retain_mask", "latency_policy", "remap_tokens", "select_important_tokens",
    "vote_expert_frequencies", "ExpertSelection", "MoEModelSpec", "Phase", "RoutingLogits",
    "confidence", "route_batch", "softmax_probs", "top_k_select",
]
