"""HarMoEny scheduling policies with the reference's API (moesim/policies.py),
executed by the sm_100a scheduler kernel (K3).

``initial_assign``, ``rebalance`` and ``rebalance_with_stats`` keep the
reference signatures and value semantics (inputs never mutated, new
ScheduleTensor returned, ValueError on q < 1) but run ``hm_schedule`` /
``hm_rebalance`` on the GPU; there is no CPU fallback.  The numpy <-> device
int32 conversion happens at this boundary.

Placements and the Eq. 4 threshold are host-side closed forms, restated from
policies.py:91-106 and 232-255.  The baseline policies of the paper's ablations
 sit on the same seam: ``even_split_assign`` runs in the
same GPU scheduler kernel (HM_POLICY_EVEN_SPLIT), ``affinity_placement`` is a
host-side placement like round-robin/blocked (policies.py:206-229).
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from enum import Enum

import numpy as np

from .core import Placement, RoutingMatrix, ScheduleTensor

_I32_MAX = 2**31 - 1


class SchedulingPolicy(str, Enum):
    REBALANCE = "rebalance"
    ROUND_ROBIN = "round_robin"
    EVEN_SPLIT = "even_split"
    AFFINITY = "affinity"


class PlacementKind(str, Enum):
    ROUND_ROBIN = "round_robin"
    BLOCKED = "blocked"


@dataclass(frozen=True)
class SchedulerConfig:
    """Scheduling knobs (policies.py:42-65)."""

    token_threshold_q: int
    policy: SchedulingPolicy = SchedulingPolicy.REBALANCE
    placement: PlacementKind = PlacementKind.ROUND_ROBIN
    affinity_refresh_batches: int | None = None

    def __post_init__(self):
        object.__setattr__(self, "policy", SchedulingPolicy(self.policy))
        object.__setattr__(self, "placement", PlacementKind(self.placement))
        if self.token_threshold_q < 1:
            raise ValueError("token_threshold_q must be >= 1")
        if self.affinity_refresh_batches is not None and self.affinity_refresh_batches < 1:
            raise ValueError("affinity_refresh_batches must be >= 1 when set")


def round_robin_placement(num_experts: int, num_gpus: int) -> Placement:
    """home[e] = e mod G (policies.py:91-95)."""
    if num_experts < 1 or num_gpus < 1:
        raise ValueError("num_experts and num_gpus must be >= 1")
    return Placement(home=tuple(int(e) % num_gpus for e in range(num_experts)), num_gpus=num_gpus)


def blocked_placement(num_experts: int, num_gpus: int) -> Placement:
    """ceil(E/G) contiguous experts per GPU, clamped to the last GPU (policies.py:98-106)."""
    if num_experts < 1 or num_gpus < 1:
        raise ValueError("num_experts and num_gpus must be >= 1")
    per = (num_experts + num_gpus - 1) // num_gpus
    return Placement(home=tuple(min(e // per, num_gpus - 1) for e in range(num_experts)), num_gpus=num_gpus)


def _device():
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("the HarMoEny scheduler runs on the GPU (hm_schedule); no CUDA device is visible")
    return torch.device("cuda", torch.cuda.current_device())


def _to_i32(arr: np.ndarray, what: str):
    import torch

    if arr.size and int(arr.sum()) > _I32_MAX:
        raise ValueError(f"{what}: token totals exceed the int32 device representation")
    return torch.from_numpy(np.ascontiguousarray(arr, dtype=np.int32)).to(_device())


def initial_assign(m_all: RoutingMatrix, placement: Placement) -> ScheduleTensor:
    """S[g, e, home[e]] = m_all[g, e] (policies.py:109-117), on the GPU."""
    from . import ops

    if placement.num_experts != m_all.num_experts or placement.num_gpus != m_all.num_gpus:
        raise ValueError("placement dimensions do not match routing matrix")
    S, _, _ = ops.schedule(_to_i32(m_all.counts, "initial_assign"),
                           _to_i32(np.asarray(placement.home, np.int64), "home"), 1, rebalance=False)
    return ScheduleTensor(S.cpu().numpy().astype(np.int64))


def rebalance_with_stats(s_initial: ScheduleTensor, q: int) -> tuple[ScheduleTensor, int]:
    """Alg. 2 token rebalancing (policies.py:120-171) on the GPU; returns (S, moves)."""
    from . import ops

    if q < 1:
        raise ValueError("token threshold q must be >= 1")
    S = _to_i32(s_initial.counts, "rebalance")
    iters, _ = ops.rebalance_(S, int(q))
    return ScheduleTensor(S.cpu().numpy().astype(np.int64)), int(iters.item())


def rebalance(s_initial: ScheduleTensor, q: int) -> ScheduleTensor:
    """Greedy token rebalancing from overloaded to underloaded GPUs (policies.py:144-163)."""
    s, _ = rebalance_with_stats(s_initial, q)
    return s


def even_split_assign(m_all: RoutingMatrix, num_gpus: int) -> ScheduleTensor:
    """Each expert's pooled tokens split evenly over all GPUs (policies.py:174-203), on the GPU.

    Remainder to the lowest-index GPUs; sources fill the per-GPU targets in index order."""
    from . import ops

    if num_gpus != m_all.num_gpus:
        raise ValueError("num_gpus does not match routing matrix")
    home = np.zeros(m_all.num_experts, np.int64)  # unused by the even split
    S, _, _ = ops.schedule(_to_i32(m_all.counts, "even_split_assign"), _to_i32(home, "home"), 1,
                           rebalance=ops.HM_POLICY_EVEN_SPLIT)
    return ScheduleTensor(S.cpu().numpy().astype(np.int64))


@dataclass(frozen=True)
class PopularityProfile:
    """Cumulative per-expert token counts over a profiling window (policies.py:68-88)."""

    counts: np.ndarray
    window_batches: int

    def __post_init__(self):
        arr = np.array(self.counts, dtype=np.int64, copy=True)
        if arr.ndim != 1:
            raise ValueError("profile counts must be one-dimensional")
        if arr.size and arr.min() < 0:
            raise ValueError("profile counts must be non-negative")
        arr.setflags(write=False)
        object.__setattr__(self, "counts", arr)
        if self.window_batches < 0:
            raise ValueError("window_batches must be >= 0")

    @property
    def num_experts(self) -> int:
        return self.counts.shape[0]


def affinity_placement(profile: PopularityProfile, num_gpus: int, slots: int) -> Placement:
    """Greedy LPT packing by profiled popularity (policies.py:206-229).

    Experts in descending popularity (ties: lower id first) go to the GPU with the least
    accumulated mass that still has a free slot (ties: lower GPU index).  A stable sort plus a
    running per-GPU (mass, index) minimum gives the reference's choice in O(E log E + E*G)."""
    E = profile.num_experts
    if E > num_gpus * slots:
        raise ValueError(f"infeasible placement: {E} experts > {num_gpus} GPUs x {slots} slots")
    counts = profile.counts
    order = np.lexsort((np.arange(E), -counts))
    mass = np.zeros(num_gpus, np.int64)
    used = np.zeros(num_gpus, np.int64)
    home = np.zeros(E, np.int64)
    for e in order:
        free = used < slots
        masked = np.where(free, mass, np.iinfo(np.int64).max)
        g = int(np.argmin(masked))  # first minimum = lowest index among equal masses
        home[e] = g
        mass[g] += int(counts[e])
        used[g] += 1
    return Placement(home=tuple(int(h) for h in home), num_gpus=num_gpus)


def estimate_token_threshold(gpu_flops: float, dtype_bytes: float, pcie_bandwidth: float) -> int:
    """q = ceil(phi * d_type / (2 beta)) + 1 with the float-jitter guard (policies.py:232-248, Eq. 4)."""
    bound = threshold_bound(gpu_flops, dtype_bytes, pcie_bandwidth)
    near = round(bound)
    ceil_bound = int(near) if abs(bound - near) <= 1e-9 * max(1.0, abs(bound)) else math.ceil(bound)
    return max(ceil_bound + 1, 1)


def threshold_bound(gpu_flops: float, dtype_bytes: float, pcie_bandwidth: float) -> float:
    if gpu_flops <= 0 or dtype_bytes <= 0 or pcie_bandwidth <= 0:
        raise ValueError("gpu_flops, dtype_bytes, and pcie_bandwidth must be positive")
    return gpu_flops * dtype_bytes / (2.0 * pcie_bandwidth)
