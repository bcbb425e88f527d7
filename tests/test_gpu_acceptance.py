"""The reference's scheduler acceptance criteria, run against the GPU scheduler kernel.

* Criterion 2 (test_acceptance.py:115-150): all 10,000 instances of the acceptance generator
  (seed 20250811, G <= 8, E <= 32, up to 10^4 tokens, uniform / Dirichlet / one-hot-heavy
  routing, random homes, q in {1,2,5,17,100,1000}).  Every GPU schedule must equal the C
  oracle's bit for bit (the oracle is pinned to the reference's own output on the first 2,000,
  tests/test_oracle_golden.py) and satisfy the invariants: conservation, the maximum load never
  rises, receivers end at or below the floor average, the iteration bound, and the fixpoint.
* Criterion 7 (test_acceptance.py:235-257): post-rebalance load spread <= max(q, total % G + q)
  on the reference's skewed traces (seeds 3/17/99, alpha 0.5/0.7/0.9, round-robin, q = 64).
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import moe_oracle as orc  # noqa: E402

pytestmark = pytest.mark.gpu


def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda")


def _instances(n=10_000):
    """test_acceptance.py:117-135, verbatim generator order."""
    rng = np.random.default_rng(20250811)
    for i in range(n):
        g = int(rng.integers(1, 9))
        e = int(rng.integers(1, 33))
        tokens = int(rng.integers(0, 10_001))
        cells = g * e
        kind = i % 3
        if kind == 0:
            probs = np.full(cells, 1.0 / cells)
        elif kind == 1:
            probs = rng.dirichlet(np.full(cells, 0.2))
        else:
            probs = np.full(cells, 1.0 / cells)
            probs[int(rng.integers(0, cells))] = 9.0 * cells
            probs /= probs.sum()
        m = rng.multinomial(tokens, probs).reshape(g, e)
        home = rng.integers(0, g, size=e)
        q = int(rng.choice([1, 1, 2, 5, 17, 100, 1000]))
        yield i, m, home, q


def test_criterion_2_all_instances_bit_exact_and_invariant():
    from paper_2506_12417_b200 import ops

    dev = _cuda()
    n = 0
    for i, m, home, q in _instances():
        g, e = m.shape
        m_d = torch.from_numpy(m.astype(np.int32)).to(dev)
        h_d = torch.from_numpy(home.astype(np.int32)).to(dev)
        S0, _, _ = ops.schedule(m_d, h_d, q, rebalance=False)
        S1, it, loads = ops.schedule(m_d, h_d, q, rebalance=True)
        S2 = S1.clone()
        it2, _ = ops.rebalance_(S2, q)  # fixpoint: rebalancing a rebalanced schedule moves nothing
        S0, S1, S2 = (t.cpu().numpy().astype(np.int64) for t in (S0, S1, S2))
        iters = int(it.item())
        S_ref, it_ref = orc.schedule(m, home, q, True)
        assert np.array_equal(S1, S_ref) and iters == it_ref, f"instance {i}: differs from the oracle"
        loads0, loads1 = S0.sum(axis=(0, 1)), S1.sum(axis=(0, 1))
        t_avg = int(m.sum()) // g
        assert np.array_equal(S1.sum(axis=2), m), f"instance {i}: conservation violated"
        assert loads1.max(initial=0) <= loads0.max(initial=0), f"instance {i}: max load increased"
        grew = loads1 > loads0
        assert np.all(loads1[grew] <= t_avg), f"instance {i}: receiver exceeded floor average"
        assert iters <= int(np.maximum(loads0 - t_avg, 0).sum()), f"instance {i}: iteration bound exceeded"
        assert np.array_equal(S2, S1) and int(it2.item()) == 0, f"instance {i}: not a fixpoint"
        assert np.array_equal(loads.cpu().numpy(), loads1)
        n += 1
    assert n == 10_000


def test_criterion_7_spread_bound():
    from paper_2506_12417_b200 import (ModelSpec, SkewSpec, WorkloadSpec, generate_trace, initial_assign,
                                       load_per_gpu, rebalance, round_robin_placement, total_tokens)

    _cuda()
    model = ModelSpec(num_layers=4, num_experts=16, d_model=64, d_ff=128, dtype_bytes=2)
    G, q = 4, 64
    placement = round_robin_placement(model.num_experts, G)
    checked = 0
    for seed in (3, 17, 99):
        for alpha in (0.5, 0.7, 0.9):
            wl = WorkloadSpec(num_batches=5, tokens_per_gpu_per_batch=2048,
                              skew=SkewSpec(alpha=alpha, skewed_experts=(0,)), seed=seed)
            for batch in generate_trace(wl, model, G).batches:
                for m_all in batch.layers:
                    s = rebalance(initial_assign(m_all, placement), q)
                    loads = load_per_gpu(s)
                    bound = max(q, total_tokens(s) % G + q)
                    assert int(loads.max() - loads.min()) <= bound
                    checked += 1
    assert checked == 3 * 3 * 5 * 4
