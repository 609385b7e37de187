"""B200-native FastMoE (arXiv 2103.13262) MoE-layer hot path.

The compute lives in libfmoe_b200.so (hand-written sm_100a CUDA behind the
C-ABI in include/fmoe_b200.h); this package is its Python host, mirroring
the reference's operator and layer API.  Importing fails loudly if the
library is not built -- there is no CPU fallback.
"""
from .api import (  # noqa: F401
    Context,
    DispatchPlan,
    Experts,
    ExpertGradsT,
    GateGrads,
    GateOutput,
    MoEConfig,
    MoELayer,
    ProtocolError,
    ShapeError,
    TransportError,
    alloc_plan,
    build_plan,
    checkpoint_info,
    gate_backward,
    gate_forward,
    gather_combine,
    gather_combine_backward,
    launches,
    multi_expert_backward,
    multi_expert_forward,
    scatter,
    scatter_backward,
    version,
    World,
    ExchangePlan,
    exchange_counts,
    all_to_all_rows,
    all_to_all_rows_reverse,
    ep_layout,
    ep_routes,
    allreduce_sum,
    matmul,
    softmax_rows,
    topk_rows,
)
from ._lib import LIB_PATH  # noqa: F401
