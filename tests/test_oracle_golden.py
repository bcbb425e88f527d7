"""Pin the CPU oracle (oracle/sched_oracle.c) to the reference's own outputs.

Fixtures come from tests/golden/make_golden.py, which ran moesim itself; the
known answers mirror reference tests test_policies.py:42-146 and
test_acceptance.py:86-150.
"""

import numpy as np
import pytest

from conftest import iter_packed
from oracle import moe_oracle as orc


def test_fig4_exact(golden):
    (inst,) = list(iter_packed(golden("fig4")))
    S0 = orc.initial_assign(inst["m"], inst["home"])
    assert S0.sum(axis=(0, 1)).tolist() == [2, 4, 9]  # test_core.py:29-30
    S1, it = orc.rebalance_with_stats(S0, 1)
    assert np.array_equal(S1, inst["S"])
    assert it == inst["iters"]
    assert S1.sum(axis=(0, 1)).tolist() == [5, 5, 5]


@pytest.mark.parametrize("pack", ["acceptance_c2", "baseline_shapes", "wide_schedules"])
def test_schedule_matches_reference(golden, pack):
    n = 0
    for inst in iter_packed(golden(pack)):
        S, it = orc.schedule(inst["m"], inst["home"], inst["q"], rebalance=True)
        assert np.array_equal(S, inst["S"]), f"instance {inst['i']}"
        assert it == inst["iters"], f"instance {inst['i']}"
        n += 1
    assert n > 30


def test_placements_match_reference():
    # test_policies.py:42-67
    assert orc.round_robin_home(3, 3).tolist() == [0, 1, 2]
    assert orc.round_robin_home(2, 4).tolist() == [0, 1]
    assert orc.blocked_home(4, 2).tolist() == [0, 0, 1, 1]
    assert orc.blocked_home(5, 3).tolist() == [0, 0, 1, 1, 2]
    assert orc.blocked_home(128, 8)[:16].tolist() == [0] * 16


def test_edge_cases():
    # q < 1 rejected (policies.py:168-169)
    with pytest.raises(ValueError):
        orc.rebalance_with_stats(np.zeros((2, 2, 2), np.int64), 0)
    # zeros and G=1: no iterations
    S, it = orc.rebalance_with_stats(np.zeros((3, 4, 3), np.int64), 1)
    assert it == 0 and not S.any()
    S, it = orc.schedule(np.array([[5, 7, 9]]), [0, 0, 0], 1)
    assert it == 0 and S.sum() == 21
    # huge q is a no-op (test_policies.py:112-114)
    m = np.array([[1, 1, 3], [1, 1, 3], [0, 2, 3]])
    S0 = orc.initial_assign(m, [0, 1, 2])
    S1, it = orc.rebalance_with_stats(S0, int(S0.sum()) + 1)
    assert it == 0 and np.array_equal(S0, S1)


def test_plan_order_matches_reference(golden):
    d = golden("plan_order")
    ow = orr = oo = 0
    for i in range(len(d["E"])):
        E = int(d["E"][i])
        work = d["work"][ow : ow + E]
        res = d["resident"][orr : orr + E]
        L = int(d["order_len"][i])
        expect = d["order"][oo : oo + L]
        ow += E
        orr += E
        oo += L
        assert orc.plan_order(work, res).tolist() == expect.tolist()


def test_dispatch_contract_small():
    # source 0 of Fig. 4 after rebalance: expert 2's 3 tokens all go to GPU 0
    m = np.array([[1, 1, 3], [1, 1, 3], [0, 2, 3]])
    S, _ = orc.schedule(m, [0, 1, 2], 1)
    idx = np.array([[2], [0], [2], [1], [2]], np.int32)  # 5 tokens of source 0, top-1
    dest, rank = orc.dispatch_ranks(idx, S, 0)
    assert rank.tolist() == [0, 0, 1, 0, 2]
    assert dest.tolist() == [0, 0, 0, 1, 0]
    # source 1: expert 2 split 1 -> GPU1, 2 -> GPU2, in (token, slot) order
    idx = np.array([[2], [2], [0], [2], [1]], np.int32)
    dest, rank = orc.dispatch_ranks(idx, S, 1)
    assert dest.tolist() == [1, 2, 0, 2, 1]


def test_bf16_roundtrip():
    x = np.array([1.0, 1.00390625, 1.005859375, -3.5, 65504.0, 1e-30], np.float32)
    b = orc.f32_to_bf16(x)
    assert orc.bf16_to_f32(b)[0] == 1.0
    assert orc.bf16_to_f32(b)[1] == 1.0  # tie to even
    assert orc.bf16_to_f32(b)[2] == 1.0078125
    assert orc.bf16_to_f32(b)[3] == -3.5


def test_even_split_oracle_matches_reference(golden):
    """even_split_assign (policies.py:174-203) restated in C == the reference's own output."""
    n = 0
    for inst in iter_packed(golden("baseline_policies")):
        S = orc.even_split(inst["m"])
        assert np.array_equal(S, inst["S"]), f"instance {inst['i']}"
        assert np.array_equal(S.sum(axis=2), inst["m"])  # conservation per (source, expert)
        n += 1
    assert n > 500


def _affinity_cases(d):
    oc = 0
    for E, G, slots in zip(d["aff_E"], d["aff_G"], d["aff_slots"]):
        E = int(E)
        yield d["aff_counts"][oc:oc + E], int(G), int(slots), d["aff_home"][oc:oc + E]
        oc += E


def test_affinity_matches_reference(golden):
    """affinity_placement (policies.py:206-229): C oracle and the package's host placement."""
    from paper_2506_12417_b200 import PopularityProfile, affinity_placement

    d = golden("baseline_policies")
    n = 0
    for counts, G, slots, home in _affinity_cases(d):
        assert np.array_equal(orc.affinity_home(counts, G, slots), home)
        p = affinity_placement(PopularityProfile(counts=counts, window_batches=1), G, slots)
        assert list(p.home) == home.tolist()
        n += 1
    assert n == 300
    with pytest.raises(ValueError, match="infeasible placement"):
        affinity_placement(PopularityProfile(counts=np.ones(5, np.int64), window_batches=1), 2, 2)
    with pytest.raises(ValueError):
        orc.affinity_home(np.ones(5, np.int64), 2, 2)
    with pytest.raises(ValueError, match="non-negative"):
        PopularityProfile(counts=np.array([1, -1]), window_batches=1)
