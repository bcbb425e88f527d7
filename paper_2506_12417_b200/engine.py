"""Engine-level seam of the reference (moesim/engine.py) that the hot path plugs into.

``build_schedule`` is the function ``moesim.engine.simulate_layer`` calls for
step 3 of Alg. 1 (engine.py:287-299, called at engine.py:334).  Here it runs the
GPU scheduler kernel; patching ``moesim.engine.build_schedule`` (or
``moesim.engine.rebalance``) with these functions drops the B200 scheduler into
the reference's simulator.  Patching ``moesim.policies`` alone
is not seen by the engine because engine.py:40-51 binds the names at import.
"""

from __future__ import annotations

from dataclasses import dataclass

from .core import Placement, RoutingMatrix, ScheduleTensor
from .policies import (
    PlacementKind,
    SchedulerConfig,
    SchedulingPolicy,
    blocked_placement,
    round_robin_placement,
)


@dataclass(frozen=True)
class SimFlags:
    """Ablation switches (engine.py:73-79)."""

    rebalancing_enabled: bool = True
    async_loading_enabled: bool = True
    include_scheduler_walltime: bool = False


def build_schedule(m_all: RoutingMatrix, placement: Placement, config: SchedulerConfig,
                   flags: SimFlags) -> ScheduleTensor:
    """Policy dispatch of engine.py:287-299 in one GPU kernel launch: even_split_assign for
    EVEN_SPLIT, else initial_assign (+ rebalance when policy is REBALANCE and enabled)."""
    import numpy as np
    import torch

    from . import ops
    from .policies import _to_i32

    home = np.asarray(placement.home, np.int64)
    if config.policy is SchedulingPolicy.EVEN_SPLIT:  # even_split_assign(m_all, m_all.num_gpus), engine.py:293
        policy = ops.HM_POLICY_EVEN_SPLIT
        home = np.zeros(m_all.num_experts, np.int64)  # the even split ignores the placement
    else:
        if placement.num_experts != m_all.num_experts or placement.num_gpus != m_all.num_gpus:
            raise ValueError("placement dimensions do not match routing matrix")
        do_rebalance = config.policy is SchedulingPolicy.REBALANCE and flags.rebalancing_enabled
        policy = ops.HM_POLICY_REBALANCE if do_rebalance else ops.HM_POLICY_NONE
    S, _, _ = ops.schedule(_to_i32(m_all.counts, "build_schedule"),
                           _to_i32(home, "home"), config.token_threshold_q, rebalance=policy)
    torch.cuda.current_stream().synchronize()
    return ScheduleTensor(S.cpu().numpy().astype(np.int64))


def static_placement(config: SchedulerConfig, num_experts: int, num_gpus: int) -> Placement:
    """engine.py:387-390."""
    if config.placement is PlacementKind.BLOCKED:
        return blocked_placement(num_experts, num_gpus)
    return round_robin_placement(num_experts, num_gpus)
