"""Synthetic routing workloads (router stand-in inputs for tests and the bench).

The reference's router stand-in is ``skew_probabilities`` + per-source
multinomial counts (moesim/workload.py:138-180).  That encodes top-k only as
larger row sums (pkg/README.md:160-163).  The B200 block routes real tokens, so
this module adds what SURVEY.md §8(d) specifies for measurement:

* Zipf expert popularity p_i ∝ (i+1)^-s (hot experts are the low ids, so a
  blocked placement piles them on GPU 0, mirroring PAPER.md:450-454);
* top-k *without replacement* via Gumbel-top-k on log p (count matrices for
  scheduler-only runs);
* router-bias construction (bias_e = log p_e) so the real router kernel
  produces Zipf-skewed routing from x ~ N(0,1), Wg ~ N(0, 1/d).

All draws use ``numpy.random.Generator(PCG64(seed))``; generated inputs are
serialised into fixtures where cross-version stability matters.
"""

from __future__ import annotations

import functools

import numpy as np


def skew_probabilities(alpha: float, skewed, num_experts: int) -> np.ndarray:
    """Same contract as moesim/workload.py:138-164 (hot-set mass alpha)."""
    if not 0.0 <= alpha <= 1.0:
        raise ValueError(f"alpha must be in [0, 1], got {alpha}")
    skewed = [int(e) for e in skewed]
    if len(set(skewed)) != len(skewed):
        raise ValueError("skewed expert indices must be distinct")
    if any(not 0 <= e < num_experts for e in skewed):
        raise ValueError("skewed expert index out of range")
    if not skewed and alpha > 0:
        raise ValueError("skewed experts required when alpha > 0")
    probs = np.empty(num_experts, dtype=np.float64)
    if alpha == 0.0 or len(skewed) == num_experts:
        probs.fill(1.0 / num_experts)
        return probs
    probs.fill((1.0 - alpha) / (num_experts - len(skewed)))
    probs[skewed] = alpha / len(skewed)
    return probs


def zipf_probabilities(num_experts: int, s: float) -> np.ndarray:
    """p_i ∝ (i+1)^-s; s = 0 is uniform."""
    if num_experts < 1:
        raise ValueError("num_experts must be >= 1")
    if s < 0:
        raise ValueError("zipf exponent must be >= 0")
    w = np.arange(1, num_experts + 1, dtype=np.float64) ** (-float(s))
    return w / w.sum()


def gumbel_topk_assignments(probs, num_tokens: int, k: int, rng: np.random.Generator) -> np.ndarray:
    """[T, k] expert ids, top-k without replacement by Gumbel-top-k on log p."""
    probs = np.asarray(probs, dtype=np.float64)
    E = probs.size
    if not 1 <= k <= E:
        raise ValueError("k must be in [1, E]")
    logp = np.log(np.maximum(probs, 1e-300))
    out = np.empty((num_tokens, k), dtype=np.int32)
    chunk = 4096
    for s in range(0, num_tokens, chunk):
        n = min(chunk, num_tokens - s)
        keys = logp[None, :] + rng.gumbel(size=(n, E))
        part = np.argpartition(-keys, k - 1, axis=1)[:, :k]
        out[s : s + n] = part
    return out


def zipf_routing_matrix(num_gpus: int, tokens_per_gpu: int, num_experts: int, k: int, s: float,
                        seed: int, permute_experts: bool = False) -> np.ndarray:
    """m_all[G, E]: per-source-GPU histogram of Zipf top-k-without-replacement
    routing.  ``permute_experts`` applies a seeded random
    id permutation so the hot experts are spread over homes."""
    rng = np.random.Generator(np.random.PCG64(seed))
    p = zipf_probabilities(num_experts, s)
    if permute_experts:
        p = p[rng.permutation(num_experts)]
    m = np.zeros((num_gpus, num_experts), dtype=np.int64)
    for g in range(num_gpus):
        a = gumbel_topk_assignments(p, tokens_per_gpu, k, rng)
        m[g] = np.bincount(a.reshape(-1), minlength=num_experts)
    return m


def router_bias(num_experts: int, s: float, seed: int | None = None) -> np.ndarray:
    """bias_e = log p_e (Zipf), optionally id-permuted with ``seed``."""
    p = zipf_probabilities(num_experts, s)
    if seed is not None:
        p = p[np.random.Generator(np.random.PCG64(seed)).permutation(num_experts)]
    return np.log(p).astype(np.float32)


def zipf_topk_frequencies(num_experts: int, s: float, k: int, samples: int = 20000, seed: int = 0) -> np.ndarray:
    """Per-expert share of assignments under Gumbel-top-k on log p_zipf (top-k without
    replacement); shares sum to 1."""
    rng = np.random.Generator(np.random.PCG64(seed))
    a = gumbel_topk_assignments(zipf_probabilities(num_experts, s), samples, k, rng)
    return np.bincount(a.reshape(-1), minlength=num_experts) / (samples * k)


def calibrated_router_bias(num_experts: int, s: float, k: int, noise_std: float = 1.0, iters: int = 200,
                           samples: int = 8192, seed: int = 0) -> np.ndarray:
    """See _calibrated_router_bias (deterministic, memoised: stacks reuse it per layer)."""
    return _calibrated_router_bias(int(num_experts), float(s), int(k), float(noise_std), int(iters), int(samples),
                                   int(seed)).copy()


@functools.lru_cache(maxsize=64)
def _calibrated_router_bias(num_experts: int, s: float, k: int, noise_std: float, iters: int, samples: int,
                            seed: int) -> np.ndarray:
    """Bias b such that top-k of (N(0, noise_std^2) logits + b) routes with the Zipf
    Gumbel-top-k shares.  The synthetic router's logits x.Wg are Gaussian (x ~ N(0,1),
    Wg ~ N(0, 1/d) -> std 1), whose light tails concentrate top-k far more than the
    Gumbel noise of the Zipf definition (top-1 at s=1 would leave ~45% of experts idle);
    the bias is fitted by fixed-point iteration on a fixed noise sample."""
    if s == 0.0:
        return np.zeros(num_experts, np.float32)
    target = zipf_topk_frequencies(num_experts, s, k, seed=seed + 1)
    rng = np.random.Generator(np.random.PCG64(seed))
    noise = rng.standard_normal((samples, num_experts)).astype(np.float32) * np.float32(noise_std)
    b = np.log(np.maximum(target, 1e-9)).astype(np.float64)
    lt = np.log(np.maximum(target, 1e-6))
    best, best_err = b.copy(), np.inf
    for it in range(iters):
        logits = noise + b[None, :].astype(np.float32)
        top = np.argpartition(-logits, k - 1, axis=1)[:, :k]
        f = np.bincount(top.reshape(-1), minlength=num_experts) / (samples * k)
        err = np.abs(f - target).sum()
        if err < best_err:
            best, best_err = b.copy(), err
        step = 0.25 if it < iters // 2 else 0.1  # damped: top-1 shares react steeply
        b += step * (lt - np.log(np.maximum(f, 1e-6)))
        b -= b.max()
    return best.astype(np.float32)


# ------------------------------------------------------------------------------------------
# The reference's workload API (moesim/workload.py:40-210): skew specs, the per-source
# multinomial sampler and trace generation.  Same validation, same RNG call sequence
# (PCG64, one uniform per batch when resampling, one multinomial per layer), so for one
# numpy build the traces are identical to the reference's (pinned in tests/test_trace.py
# against tests/golden/trace_g4_e16.jsonl, which the reference itself wrote).  These
# produce count matrices for scheduler-only runs and trace replay; the MoE block's own
# routing comes from the router kernel.
# ------------------------------------------------------------------------------------------
MODE_FIXED = "fixed"
MODE_RESAMPLE_UNIFORM = "resample_uniform"


from dataclasses import dataclass  # noqa: E402


@dataclass(frozen=True)
class SkewSpec:
    """Expert-popularity skew (workload.py:40-67): mass ``alpha`` on ``skewed_experts``,
    constant or redrawn per batch from U[resample_lo, resample_hi]."""

    alpha: float
    skewed_experts: tuple = (0,)
    mode: str = MODE_FIXED
    resample_lo: float = 0.0
    resample_hi: float = 0.0

    def __post_init__(self):
        object.__setattr__(self, "skewed_experts", tuple(int(e) for e in self.skewed_experts))
        if not 0.0 <= self.alpha <= 1.0:
            raise ValueError(f"alpha must be in [0, 1], got {self.alpha}")
        if self.mode not in (MODE_FIXED, MODE_RESAMPLE_UNIFORM):
            raise ValueError(f"unknown per-batch mode {self.mode!r}")
        if not 0.0 <= self.resample_lo <= self.resample_hi <= 1.0:
            raise ValueError("resample bounds must satisfy 0 <= lo <= hi <= 1")
        if len(set(self.skewed_experts)) != len(self.skewed_experts):
            raise ValueError("skewed expert indices must be distinct")
        if any(e < 0 for e in self.skewed_experts):
            raise ValueError("skewed expert indices must be non-negative")
        max_alpha = self.resample_hi if self.mode == MODE_RESAMPLE_UNIFORM else self.alpha
        if max_alpha > 0 and not self.skewed_experts:
            raise ValueError("skewed_experts must be non-empty when alpha can exceed 0")


@dataclass(frozen=True)
class WorkloadSpec:
    """One synthetic experiment (workload.py:70-82)."""

    num_batches: int
    tokens_per_gpu_per_batch: int
    skew: SkewSpec
    seed: int

    def __post_init__(self):
        if self.num_batches < 1:
            raise ValueError("num_batches must be >= 1")
        if self.tokens_per_gpu_per_batch < 1:
            raise ValueError("tokens_per_gpu_per_batch must be >= 1")


def sample_routing(probs, tokens_per_gpu: int, num_gpus: int, rng: np.random.Generator):
    """One routing matrix, each source row an independent multinomial (workload.py:167-180)."""
    from .core import RoutingMatrix

    probs = np.asarray(probs, dtype=np.float64)
    total = probs.sum()
    if abs(total - 1.0) > 1e-9:
        raise ValueError(f"probabilities must sum to 1, got {total}")
    return RoutingMatrix(rng.multinomial(tokens_per_gpu, probs / total, size=num_gpus))


def generate_trace(spec: WorkloadSpec, model, num_gpus: int):
    """num_batches x num_layers routing matrices (workload.py:183-210), layers independent."""
    from .trace import Trace, TraceBatch

    rng = np.random.Generator(np.random.PCG64(spec.seed))
    batches = []
    for b in range(spec.num_batches):
        if spec.skew.mode == MODE_RESAMPLE_UNIFORM:
            alpha = float(rng.uniform(spec.skew.resample_lo, spec.skew.resample_hi))
        else:
            alpha = spec.skew.alpha
        probs = skew_probabilities(alpha, spec.skew.skewed_experts, model.num_experts)
        layers = [sample_routing(probs, spec.tokens_per_gpu_per_batch, num_gpus, rng) for _ in range(model.num_layers)]
        batches.append(TraceBatch(batch_id=b, alpha=alpha, layers=layers))
    return Trace(num_gpus=num_gpus, num_experts=model.num_experts, num_layers=model.num_layers, seed=spec.seed,
                 batches=batches)
