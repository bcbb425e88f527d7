"""B200-measured cost model for the reference simulator's cost seam.

The reference replays traces through an analytic CostModel (engine.py:82-132): expert
compute = FLOPs / gpu_flops, expert fetch = bytes / pcie_bandwidth, a constant
metadata_time, and token_bytes for the all-to-all.  ``simulate_run(..., cost=...)``
(engine.py:399,415-416) takes any object exposing the attributes the engine reads:

* ``expert_compute_time(n)``   engine.py:248,270
* ``expert_load_time``         engine.py:258,266
* ``metadata_time``            engine.py:328-331
* ``token_bytes``              engine.py:341

:class:`MeasuredCostModel` provides exactly those, filled from B200 measurements of THIS
repo's kernels instead of peak-rate formulas:

* compute — the tcgen05 grouped GEMM pair (K5: gate/up+SwiGLU or W1+ReLU, then down) on
  ``probe_experts`` experts of n rows each, timed with CUDA events; per-expert time = total
  / probe_experts (the engine sums experts sequentially, so the amortised per-expert cost
  is the matching quantity).  Piecewise-linear in n between measured points, linear
  extrapolation past the last one;
* expert load — ``hm_fetch_expert`` of one expert's packed weights from pinned host memory
  ("host", the reference's PCIe path) or from another HBM buffer ("device"; the NVLink peer
  path needs two GPUs and is measured by ep.py);
* metadata — the fused plan kernel (histogram reduce + schedule + layout, K2-K3) at the
  config's G, plus the all-gather of hist when a process group with world > 1 is live.

The model serialises to JSON so it can be measured once on a B200 and fed to moesim on any
host.  Summary/breakdown reports (metrics.py:127-202) are then the reference's own writers
applied to the RunMetrics this cost model produces.
"""

from __future__ import annotations

import json
from dataclasses import asdict, dataclass

import numpy as np

DEFAULT_POINTS = (1, 32, 64, 128, 256, 512, 1024, 2048, 4096)


@dataclass(frozen=True)
class MeasuredCostModel:
    d_model: int
    d_ff: int
    dtype_bytes: int
    n_matrices: int  # 2 (ReLU expert) or 3 (SwiGLU expert)
    metadata_time: float  # seconds
    expert_load_time: float  # seconds per expert fetch
    token_points: tuple  # measured token counts, strictly increasing
    compute_seconds: tuple  # per-expert seconds at token_points
    device_name: str = ""
    load_source: str = "host"

    def __post_init__(self):
        pts = tuple(int(p) for p in self.token_points)
        secs = tuple(float(s) for s in self.compute_seconds)
        if len(pts) < 2 or len(pts) != len(secs):
            raise ValueError("need >= 2 measured (tokens, seconds) points")
        if any(b <= a for a, b in zip(pts, pts[1:])) or pts[0] < 1:
            raise ValueError("token_points must be positive and strictly increasing")
        if any(s < 0 for s in secs) or self.expert_load_time < 0 or self.metadata_time < 0:
            raise ValueError("measured times must be >= 0")
        object.__setattr__(self, "token_points", pts)
        object.__setattr__(self, "compute_seconds", secs)

    # ---- attributes the reference engine reads ----
    @property
    def expert_bytes(self) -> int:
        return self.n_matrices * self.d_model * self.d_ff * self.dtype_bytes

    @property
    def token_bytes(self) -> int:
        return self.d_model * self.dtype_bytes

    @property
    def pcie_bandwidth(self) -> float:
        return self.expert_bytes / self.expert_load_time if self.expert_load_time > 0 else float("inf")

    def expert_flops(self, tokens: int) -> int:
        return 2 * self.n_matrices * self.d_model * self.d_ff * int(tokens)

    @property
    def gpu_flops(self) -> float:
        """Effective rate at the largest measured point (for reports)."""
        return self.expert_flops(self.token_points[-1]) / max(self.compute_seconds[-1], 1e-30)

    def expert_compute_time(self, tokens: int) -> float:
        n = int(tokens)
        if n <= 0:
            return 0.0
        x, y = self.token_points, self.compute_seconds
        if n >= x[-1]:
            slope = (y[-1] - y[-2]) / (x[-1] - x[-2])
            return float(y[-1] + max(slope, 0.0) * (n - x[-1]))
        if n <= x[0]:
            return float(y[0])
        return float(np.interp(n, x, y))

    # ---- persistence ----
    def to_json(self, path=None) -> str:
        text = json.dumps(asdict(self), indent=1, sort_keys=True)
        if path is not None:
            with open(path, "w", encoding="utf-8") as fh:
                fh.write(text + "\n")
        return text

    @classmethod
    def from_json(cls, path_or_text) -> "MeasuredCostModel":
        text = path_or_text
        if not str(path_or_text).lstrip().startswith("{"):
            with open(path_or_text, "r", encoding="utf-8") as fh:
                text = fh.read()
        return cls(**json.loads(text))


def _time_ms(fn, reps: int, warmup: int = 3) -> float:
    import torch

    for _ in range(warmup):
        fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


def measure_cost_model(cfg, token_points=DEFAULT_POINTS, probe_experts: int | None = None,
                       load_source: str = "host", reps: int = 20, device="cuda", seed: int = 0) -> MeasuredCostModel:
    """Measure K5 / K6 / K2-K3 for ``cfg`` (a block.MoEConfig) on the current B200."""
    import torch

    from . import ops

    dev = torch.device(device)
    d, f, E = cfg.d_model, cfg.d_ff, cfg.num_experts
    swiglu = cfg.activation == "swiglu"
    n_in = 2 * f if swiglu else f
    epi = ops.HM_EPI_SWIGLU if swiglu else ops.HM_EPI_RELU
    P = int(probe_experts or min(E, 32))
    g = torch.Generator(device=dev).manual_seed(seed)
    bf = torch.bfloat16
    w_in = (torch.randn((P * n_in, d), generator=g, device=dev) * 0.02).to(bf)
    w_out = (torch.randn((P * d, f), generator=g, device=dev) * 0.02).to(bf)
    secs = []
    tm = ops.TILE_M
    # the first point is measured twice: the first pass absorbs module load and clock ramp-up
    for i, n in enumerate((token_points[0],) + tuple(token_points)):
        rows = P * n
        sg = torch.tensor([[i * n, n, i, i] for i in range(P)], dtype=torch.int32, device=dev)
        mt = torch.tensor([0] + [(i + 1) * ((n + tm - 1) // tm) for i in range(P)], dtype=torch.int32, device=dev)
        lay = (sg, torch.tensor([P], dtype=torch.int32, device=dev), mt)
        A = torch.randn((rows, d), generator=g, device=dev).to(bf)
        H = torch.empty((rows, f), dtype=bf, device=dev)
        Y = torch.empty((rows, d), dtype=bf, device=dev)

        def step():
            ops.grouped_gemm(A, w_in, n_in, lay, epi, out=H)
            ops.grouped_gemm(H, w_out, d, lay, ops.HM_EPI_STORE, out=Y)

        t = _time_ms(step, reps) / 1e3 / P
        if i > 0:
            secs.append(t)

    # expert fetch (K6): one expert's packed weights
    nbytes = (n_in * d + d * f) * 2
    dst = torch.empty(nbytes // 2, dtype=bf, device=dev)
    if load_source == "host":
        src = torch.empty(nbytes // 2, dtype=bf, pin_memory=True)
    elif load_source == "device":
        src = torch.empty(nbytes // 2, dtype=bf, device=dev)
    else:
        raise ValueError("load_source must be 'host' or 'device'")
    load = _time_ms(lambda: ops.fetch_expert(dst, src), max(3, reps // 2)) / 1e3

    # metadata: plan kernel (+ all-gather of hist when distributed)
    G = cfg.num_ranks
    home = torch.tensor([e % G for e in range(E)], dtype=torch.int32, device=dev)
    m_all = torch.randint(0, 64, (G, E), dtype=torch.int32, device=dev, generator=g)
    meta = _time_ms(lambda: ops.plan(home, G, E, cfg.eq_tokens, cfg.policy_code, ops.HM_LAYOUT_LOCAL, m_all=m_all),
                    reps) / 1e3
    try:
        import torch.distributed as dist

        if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
            h = torch.zeros(E, dtype=torch.int32, device=dev)
            out = torch.empty((dist.get_world_size(), E), dtype=torch.int32, device=dev)
            meta += _time_ms(lambda: dist.all_gather_into_tensor(out, h), reps) / 1e3
    except Exception:  # noqa: BLE001 - a missing process group just means no exchange term
        pass
    return MeasuredCostModel(d_model=d, d_ff=f, dtype_bytes=2, n_matrices=3 if swiglu else 2, metadata_time=meta,
                             expert_load_time=load, token_points=tuple(token_points), compute_seconds=tuple(secs),
                             device_name=torch.cuda.get_device_name(dev), load_source=load_source)
