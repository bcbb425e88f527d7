"""Routing traces in the reference's on-disk format, recorded on and replayed by the B200 path.

SURVEY.md §8(f) row 2.  The reference stores a run's routing as line-delimited JSON
(workload.py:213-321): one header line ``{"version": 1, "kind": "trace", "num_gpus",
"num_experts", "num_layers", "rng", "seed"}`` and one line per batch ``{"batch_id",
"alpha_used", "layers": [[G][E] ints per layer]}``, keys sorted.  This module reads and
writes exactly that format (a file written here is byte-identical to the reference's
``write_trace`` for the same trace, and ``read_trace`` rejects the same malformed files
with the same 1-based line numbers), so routing is exchanged with moesim losslessly
across hosts and numpy versions (the sampler itself is not stable).

Two B200 additions:

* :class:`TraceRecorder` appends the REAL routing of a :class:`HarMoEnyBlock` /
  :class:`MoEStack` / EP block forward (the per-layer m_all the plan kernel already
  produced on the device) as one trace batch — one device→host copy per batch.
* :func:`replay_schedules` schedules every (batch, layer) routing matrix of a trace in
  ONE launch of the batched scheduler (hm_schedule_batched, one CTA per instance), the
  GPU counterpart of the reference's per-layer ``build_schedule`` loop inside
  ``simulate_run`` (engine.py:393-477 → 287-299).
"""

from __future__ import annotations

import json
from dataclasses import dataclass, field

import numpy as np

from .core import Placement, RoutingMatrix

TRACE_VERSION = 1  # workload.py:25
RNG_NAME = "numpy-pcg64"  # workload.py:24 (synthetic traces); recorded traces name their source
RECORDED_RNG = "b200-router"


class TraceParseError(ValueError):
    """Malformed trace file; ``line_no`` is the 1-based offending line (workload.py:31-37)."""

    def __init__(self, line_no: int, message: str):
        super().__init__(f"line {line_no}: {message}")
        self.line_no = line_no


@dataclass
class TraceBatch:
    batch_id: int
    alpha: float
    layers: list  # [RoutingMatrix] * num_layers


@dataclass
class Trace:
    """A replayable sequence of routing matrices: ``batches[b].layers[l]`` is m_all [G,E].

    Same fields and equality as the reference Trace (workload.py:95-135); :meth:`counts`
    gives the dense int64 [B, L, G, E] view the GPU replay consumes."""

    num_gpus: int
    num_experts: int
    num_layers: int
    rng_name: str = RNG_NAME
    seed: int = 0
    batches: list = field(default_factory=list)

    @property
    def num_batches(self) -> int:
        return len(self.batches)

    def tokens_per_batch(self) -> int:
        # row sums count assignments (T*k for top-k), as the reference does (engine.py:442)
        if not self.batches:
            return 0
        return int(self.batches[0].layers[0].counts.sum())

    def counts(self) -> np.ndarray:
        out = np.zeros((self.num_batches, self.num_layers, self.num_gpus, self.num_experts), np.int64)
        for b, batch in enumerate(self.batches):
            for l, m in enumerate(batch.layers):
                out[b, l] = m.counts
        return out

    def append(self, layers, alpha: float = 0.0, batch_id: int | None = None) -> TraceBatch:
        """Append one batch from ``layers`` ([L,G,E] array-like or a list of RoutingMatrix)."""
        mats = [m if isinstance(m, RoutingMatrix) else RoutingMatrix(np.asarray(m)) for m in layers]
        if len(mats) != self.num_layers:
            raise ValueError(f"expected {self.num_layers} layers, got {len(mats)}")
        rows = None
        for m in mats:
            if m.counts.shape != (self.num_gpus, self.num_experts):
                raise ValueError(f"layer shape {m.counts.shape} != {(self.num_gpus, self.num_experts)}")
            if rows is None:
                rows = m.row_sums()
            elif not np.array_equal(rows, m.row_sums()):
                raise ValueError("row sums differ between layers of one batch")
        batch = TraceBatch(batch_id=self.num_batches if batch_id is None else int(batch_id), alpha=float(alpha),
                           layers=mats)
        self.batches.append(batch)
        return batch

    def __eq__(self, other) -> bool:
        if not isinstance(other, Trace):
            return NotImplemented
        head = (self.num_gpus, self.num_experts, self.num_layers, self.rng_name, self.seed)
        if head != (other.num_gpus, other.num_experts, other.num_layers, other.rng_name, other.seed):
            return False
        if self.num_batches != other.num_batches:
            return False
        return all(a.batch_id == b.batch_id and a.alpha == b.alpha and a.layers == b.layers
                   for a, b in zip(self.batches, other.batches))

    # ---- interop with the reference package (optional; moesim need not be installed) ----
    @classmethod
    def from_moesim(cls, t) -> "Trace":
        out = cls(t.num_gpus, t.num_experts, t.num_layers, t.rng_name, t.seed)
        for b in t.batches:
            out.append([np.asarray(m.counts) for m in b.layers], alpha=b.alpha, batch_id=b.batch_id)
        return out

    def to_moesim(self):
        import moesim
        from moesim.workload import TraceBatch as RefBatch

        return moesim.Trace(num_gpus=self.num_gpus, num_experts=self.num_experts, num_layers=self.num_layers,
                            rng_name=self.rng_name, seed=self.seed,
                            batches=[RefBatch(batch_id=b.batch_id, alpha=b.alpha,
                                              layers=[moesim.RoutingMatrix(m.counts) for m in b.layers])
                                     for b in self.batches])


def _dumps(obj) -> str:
    return json.dumps(obj, sort_keys=True)


def write_trace(trace: Trace, path) -> None:
    """Header line + one line per batch, keys sorted (workload.py:213-232)."""
    lines = [_dumps({"version": TRACE_VERSION, "kind": "trace", "num_gpus": trace.num_gpus,
                     "num_experts": trace.num_experts, "num_layers": trace.num_layers, "rng": trace.rng_name,
                     "seed": trace.seed})]
    for b in trace.batches:
        lines.append(_dumps({"batch_id": b.batch_id, "alpha_used": b.alpha,
                             "layers": [m.counts.tolist() for m in b.layers]}))
    with open(path, "w", encoding="utf-8") as fh:
        fh.write("\n".join(lines) + "\n")


def _fail(line_no: int, message: str):
    raise TraceParseError(line_no, message)


def _parse_json(line_no: int, text: str):
    try:
        return json.loads(text)
    except json.JSONDecodeError as exc:
        raise TraceParseError(line_no, f"invalid JSON ({exc.msg})") from exc


def _diagnose_layers(idx: int, layers_raw, L: int, G: int, E: int):
    """Slow path: name the first structural problem of a batch record (workload.py:275-305)."""
    if not isinstance(layers_raw, list) or len(layers_raw) != L:
        got = len(layers_raw) if isinstance(layers_raw, list) else "non-list"
        _fail(idx, f"expected {L} layers, got {got}")
    for li, matrix in enumerate(layers_raw):
        if not isinstance(matrix, list) or len(matrix) != G:
            _fail(idx, f"layer {li}: expected {G} rows")
        for row in matrix:
            if not isinstance(row, list) or len(row) != E:
                _fail(idx, f"layer {li}: expected {E} columns per row")
            for v in row:
                if not isinstance(v, int) or isinstance(v, bool):
                    _fail(idx, f"layer {li}: counts must be integers")
                if v < 0:
                    _fail(idx, f"layer {li}: negative token count {v}")
    _fail(idx, "malformed layers")  # unreachable for well-formed input


def read_trace(path) -> Trace:
    """Parse a trace file (workload.py:240-321): same checks, same line numbers.

    Well-formed records take a vectorised path (one numpy conversion per batch); anything
    numpy cannot take as a dense non-negative int [L,G,E] block falls to a per-element
    diagnosis that names the problem."""
    with open(path, "r", encoding="utf-8") as fh:
        lines = fh.read().splitlines()
    if not lines:
        _fail(1, "empty file, expected a trace header")
    header = _parse_json(1, lines[0])
    if not isinstance(header, dict):
        _fail(1, "header must be a JSON object")
    for key in ("version", "num_gpus", "num_experts", "num_layers", "rng", "seed"):
        if key not in header:
            _fail(1, f"header missing {key!r}")
    if header["version"] != TRACE_VERSION:
        _fail(1, f"unsupported trace version {header['version']}")
    G, E, L = int(header["num_gpus"]), int(header["num_experts"]), int(header["num_layers"])
    if G < 1 or E < 1 or L < 1:
        _fail(1, "header dimensions must be positive")
    trace = Trace(G, E, L, rng_name=str(header["rng"]), seed=int(header["seed"]))
    for idx, text in enumerate(lines[1:], start=2):
        if not text.strip():
            continue
        rec = _parse_json(idx, text)
        if not isinstance(rec, dict):
            _fail(idx, "batch record must be a JSON object")
        for key in ("batch_id", "alpha_used", "layers"):
            if key not in rec:
                _fail(idx, f"batch record missing {key!r}")
        raw = rec["layers"]
        arr = None
        try:
            cand = np.asarray(raw)
            if cand.shape == (L, G, E) and cand.dtype.kind in "iu" and (cand.size == 0 or cand.min() >= 0):
                arr = cand.astype(np.int64)
        except (ValueError, TypeError, OverflowError):
            arr = None
        if arr is None:
            _diagnose_layers(idx, raw, L, G, E)
        sums = arr.sum(axis=2)  # [L, G]
        for li in range(1, L):
            if not np.array_equal(sums[li], sums[0]):
                _fail(idx, f"layer {li}: row sums differ from earlier layers in this batch")
        trace.batches.append(TraceBatch(batch_id=int(rec["batch_id"]), alpha=float(rec["alpha_used"]),
                                        layers=[RoutingMatrix(arr[li]) for li in range(L)]))
    return trace


# ----------------------------------------------------------------------------------------
# B200 side: record real routing, replay through the batched GPU scheduler
# ----------------------------------------------------------------------------------------


class TraceRecorder:
    """Append each forward's per-layer m_all (already on the device, BlockStats.m_all) to a
    trace.  ``model`` is a HarMoEnyBlock, EPHarMoEnyBlock or MoEStack; call :meth:`record`
    after each forward (it synchronises on one small D2H copy: L*G*E int32)."""

    def __init__(self, model, seed: int = 0, rng_name: str = RECORDED_RNG):
        self.model = model
        layers = getattr(model, "layers", [model])
        cfg = layers[0].cfg
        G = cfg.num_ranks
        self.trace = Trace(num_gpus=G, num_experts=cfg.num_experts, num_layers=len(layers), rng_name=rng_name,
                           seed=seed)

    def _layers(self):
        return getattr(self.model, "layers", [self.model])

    def record(self, alpha: float = 0.0) -> TraceBatch:
        import torch

        mats = [blk.stats.m_all for blk in self._layers()]
        if any(m is None for m in mats):
            raise RuntimeError("TraceRecorder.record: run a forward first")
        host = torch.stack([m.reshape(self.trace.num_gpus, self.trace.num_experts) for m in mats]).cpu().numpy()
        return self.trace.append(host.astype(np.int64), alpha=alpha)


@dataclass
class ReplayResult:
    """Schedules of every (batch, layer) instance of a trace."""

    S: np.ndarray  # int64 [B, L, G, E, G]
    iters: np.ndarray  # int64 [B, L]
    loads: np.ndarray  # int64 [B, L, G]
    device_ms: float  # scheduler kernel time for the whole trace

    def max_over_mean(self) -> np.ndarray:
        """max_g t_g / mean_g t_g per (batch, layer) (core.py:197-203); 1.0 for empty layers."""
        loads = self.loads.astype(np.float64)
        mean = loads.mean(axis=2)
        return np.where(mean > 0, loads.max(axis=2) / np.where(mean > 0, mean, 1.0), 1.0)


def replay_schedules(trace: Trace, placement, q: int, rebalance: bool = True, device="cuda") -> ReplayResult:
    """Schedule every routing matrix of ``trace`` in one hm_schedule_batched launch.

    ``placement`` is a Placement (core.py:157-194) or a home[E] array.  Bit-identical to
    running the reference's build_schedule (engine.py:287-299: initial_assign, then
    rebalance when ``rebalance``) per (batch, layer)."""
    import torch

    from . import ops

    if int(q) < 1:
        raise ValueError("token threshold q must be >= 1")
    home = np.asarray(placement.home if isinstance(placement, Placement) else placement, np.int64)
    if home.shape != (trace.num_experts,) or (home.size and (home.min() < 0 or home.max() >= trace.num_gpus)):
        raise ValueError("placement dimensions do not match the trace")
    B, L, G, E = trace.num_batches, trace.num_layers, trace.num_gpus, trace.num_experts
    counts = trace.counts()
    if counts.size and counts.max() > np.iinfo(np.int32).max // max(G, 1):
        raise ValueError("trace counts exceed the int32 scheduler range")
    dev = torch.device(device)
    m_dev = torch.from_numpy(counts.reshape(B * L, G, E).astype(np.int32)).to(dev)
    h_dev = torch.from_numpy(home.astype(np.int32)).to(dev)
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    start.record()
    S, iters, loads = ops.schedule_batched(m_dev, h_dev, int(q), rebalance)
    end.record()
    torch.cuda.synchronize(dev)
    return ReplayResult(S=S.cpu().numpy().astype(np.int64).reshape(B, L, G, E, G),
                        iters=iters.cpu().numpy().astype(np.int64).reshape(B, L),
                        loads=loads.cpu().numpy().astype(np.int64).reshape(B, L, G),
                        device_ms=float(start.elapsed_time(end)))
