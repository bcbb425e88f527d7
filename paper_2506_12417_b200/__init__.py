"""B200-native HarMoEny expert-parallel MoE block (arXiv 2506.12417).

Drop-in for the reference's scheduling API (``moesim``: core value types,
policies, ``build_schedule``) backed by hand-written sm_100a CUDA kernels in
``libharmoe.so`` (C ABI: include/harmoe.h), plus the MoE block itself
(``HarMoEnyBlock`` / ``MoEConfig`` / ``replace_moe_layer``).
"""

from .core import (
    ClusterSpec,
    ModelSpec,
    Placement,
    RoutingMatrix,
    ScheduleTensor,
    load_per_gpu,
    total_tokens,
    validate_against,
)
from .engine import SimFlags, build_schedule, static_placement
from .policies import (
    PlacementKind,
    PopularityProfile,
    SchedulerConfig,
    SchedulingPolicy,
    affinity_placement,
    blocked_placement,
    estimate_token_threshold,
    even_split_assign,
    initial_assign,
    rebalance,
    rebalance_with_stats,
    round_robin_placement,
    threshold_bound,
)
from .costmodel import MeasuredCostModel
from .trace import Trace, TraceBatch, TraceParseError, read_trace, write_trace
from .workload import (
    SkewSpec,
    WorkloadSpec,
    generate_trace,
    sample_routing,
    skew_probabilities,
    zipf_probabilities,
    zipf_routing_matrix,
)

__version__ = "0.1.0"


def __getattr__(name):
    # torch-dependent pieces load lazily so the value types import without CUDA
    if name in ("HarMoEnyBlock", "MoEConfig", "BlockStats"):
        from . import block

        return getattr(block, name)
    if name in ("replace_moe_layer", "HarMoEnyLayer"):
        from . import integration

        return getattr(integration, name)
    raise AttributeError(name)


__all__ = [
    "ClusterSpec", "ModelSpec", "Placement", "RoutingMatrix", "ScheduleTensor", "load_per_gpu", "total_tokens",
    "validate_against", "SimFlags", "build_schedule", "static_placement", "PlacementKind", "SchedulerConfig",
    "SchedulingPolicy", "blocked_placement", "estimate_token_threshold", "initial_assign", "rebalance",
    "rebalance_with_stats", "round_robin_placement", "threshold_bound", "skew_probabilities",
    "zipf_probabilities", "zipf_routing_matrix", "HarMoEnyBlock", "MoEConfig", "BlockStats", "replace_moe_layer",
    "HarMoEnyLayer", "MeasuredCostModel", "PopularityProfile", "affinity_placement", "even_split_assign",
    "SkewSpec", "WorkloadSpec", "generate_trace", "sample_routing", "Trace", "TraceBatch", "TraceParseError", "read_trace", "write_trace",
]
