"""Generate golden scheduler fixtures from the reference implementation itself.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_golden.py

It imports ``moesim`` read-only from /root/reference/pkg/src and records the
reference's own outputs, so the CPU oracle (oracle/sched_oracle.c) and the CUDA
scheduler kernel are pinned to the reference, not to a restatement:

* fig4.npz            - the paper's Fig. 4 example (test_policies.py:89-103)
* acceptance_c2.npz   - the first N instances of acceptance criterion 2's
                        generator, seed 20250811 (test_acceptance.py:115-150)
* baseline_shapes.npz - BASELINE shapes (E=128 k=1 / E=128 k=8 / E=8 k=2) x
                        Zipf s x G x placement x q, Zipf top-k routing
* plan_order.npz      - plan_gpu_execution (engine.py:204-275) order/timing on
                        random work lists with the unit cost model
                        (test_engine.py:30-43)
* trace_g4_e16.jsonl  - a trace written by the reference's write_trace
                        (workload.py:183-232), resampled alpha, 5 batches x 3 layers
* trace_g4_e16_schedules.npz - the reference build_schedule (engine.py:287-299)
                        of every (batch, layer) of that trace, per placement and q
* wide_schedules.npz  - totals >= 2^21 tokens and G*E*G beyond shared memory (the
                        64-bit rebalance loop of the CUDA scheduler)
* baseline_policies.npz - even_split_assign (policies.py:174-203) on the
                        baseline-shape + acceptance matrices; affinity_placement
                        (policies.py:206-229) on random popularity profiles

The inputs are stored alongside the outputs, so the fixtures do not depend on
numpy RNG stream stability.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

import moesim  # noqa: E402
from moesim import (  # noqa: E402
    CostModel,
    Placement,
    RoutingMatrix,
    SimFlags,
    blocked_placement,
    initial_assign,
    plan_gpu_execution,
    rebalance_with_stats,
    round_robin_placement,
)
from moesim.engine import EventCategory  # noqa: E402

from paper_2506_12417_b200.workload import zipf_routing_matrix  # noqa: E402


def _pack(instances):
    """instances: list of dicts with m (G,E), home (E,), q, S (G,E,G), iters."""
    G = np.array([i["m"].shape[0] for i in instances], np.int32)
    E = np.array([i["m"].shape[1] for i in instances], np.int32)
    q = np.array([i["q"] for i in instances], np.int64)
    iters = np.array([i["iters"] for i in instances], np.int64)
    m = np.concatenate([i["m"].reshape(-1) for i in instances]).astype(np.int64)
    home = np.concatenate([np.asarray(i["home"]).reshape(-1) for i in instances]).astype(np.int64)
    S = np.concatenate([i["S"].reshape(-1) for i in instances]).astype(np.int64)
    return dict(G=G, E=E, q=q, iters=iters, m=m, home=home, S=S)


def _run(m, home, q):
    G, E = m.shape
    s0 = initial_assign(RoutingMatrix(m), Placement(home=tuple(int(h) for h in home), num_gpus=G))
    s1, it = rebalance_with_stats(s0, int(q))
    return dict(m=np.asarray(m), home=np.asarray(home), q=int(q), S=s1.counts.copy(), iters=it)


def fig4():
    m = np.array([[1, 1, 3], [1, 1, 3], [0, 2, 3]], np.int64)
    return _pack([_run(m, [0, 1, 2], 1)])


def acceptance_c2(n=2000):
    # exact generator of test_acceptance.py:117-135 (first n of its 10,000)
    rng = np.random.default_rng(20250811)
    out = []
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
        home = [int(x) for x in rng.integers(0, g, size=e)]
        q = int(rng.choice([1, 1, 2, 5, 17, 100, 1000]))
        out.append(_run(m, home, q))
    return _pack(out)


SHAPES = {
    # name: (E, k, T_total)  -- SURVEY.md §8 C1/C2/C3 (C3 with T=16384)
    "switch128": (128, 1, 4096),
    "qwen128": (128, 8, 16384),
    "mixtral8": (8, 2, 16384),
}


def baseline_shapes():
    out, names = [], []
    seed = 11
    for name, (E, k, T) in SHAPES.items():
        for s in (0.0, 0.5, 1.0, 1.5):
            for G in (1, 2, 4, 8):
                m = zipf_routing_matrix(G, T // G, E, k, s, seed)
                for pl in ("round_robin", "blocked"):
                    home = (round_robin_placement if pl == "round_robin" else blocked_placement)(E, G).home
                    for q in (1, 32, 256, 1499):
                        out.append(_run(m, home, q))
                        names.append(f"{name}|s={s}|G={G}|{pl}|q={q}")
    d = _pack(out)
    d["names"] = np.array(names)
    return d


def wide_schedules():
    """Instances that leave the CUDA scheduler's packed 32-bit fast loop: totals >= 2^21
    tokens (the (value, index) keys no longer fit 32 bits) and G*E*G too large for the
    shared-memory copy (2*G*E*G*4 B > 200 KB, S scanned in global memory).  Both take the
    64-bit loop of hm_sched.cu; the reference answers come from moesim itself."""
    out, names = [], []
    rng = np.random.default_rng(2021)
    # BASELINE shapes at 2^21+ assignments (Zipf top-k, blocked = hot experts on GPU 0)
    for (E, k, G, Tg, s) in ((128, 8, 8, 40000, 1.0), (128, 1, 4, 600000, 1.5), (8, 2, 8, 140000, 0.5),
                             (128, 8, 2, 140000, 0.0)):
        m = zipf_routing_matrix(G, Tg, E, k, s, 11)
        assert m.sum() >= 1 << 21
        for pl in ("round_robin", "blocked"):
            home = (round_robin_placement if pl == "round_robin" else blocked_placement)(E, G).home
            for q in (1, 32, 1499):
                out.append(_run(m, home, q))
                names.append(f"E={E}|k={k}|G={G}|Tg={Tg}|s={s}|{pl}|q={q}")
    # S too large for shared memory: G=16/E=256, G=32/E=64, G=12/E=512 (random skew, small and
    # large totals)
    for (G, E) in ((16, 256), (32, 64), (12, 512)):
        for tokens in (50_000, 3_000_000):
            probs = rng.dirichlet(np.full(G * E, 0.3))
            m = rng.multinomial(tokens, probs).reshape(G, E)
            home = [int(x) for x in rng.integers(0, G, size=E)]
            for q in (1, 17):
                out.append(_run(m, home, q))
                names.append(f"G={G}|E={E}|tokens={tokens}|q={q}")
    d = _pack(out)
    d["names"] = np.array(names)
    return d


def plan_order(n=400):
    rng = np.random.default_rng(4242)
    cost = CostModel(d_model=4, d_ff=4, dtype_bytes=2, gpu_flops=56.0, pcie_bandwidth=64.0 / 1.5,
                     metadata_time=0.0)
    works, residents, slots, orders, spans, fetch_starts, wait_total, flags_async = [], [], [], [], [], [], [], []
    E_list = []
    for i in range(n):
        E = int(rng.integers(1, 17))
        work = rng.integers(0, 12, size=E) * (rng.random(E) < 0.7)
        nres = int(rng.integers(0, E + 1))
        res = np.zeros(E, np.int32)
        res[rng.permutation(E)[:nres]] = 1
        sl = max(2, nres + int(rng.integers(0, 3)))
        async_on = bool(i % 2 == 0)
        plan = plan_gpu_execution([(e, int(work[e])) for e in range(E)], set(np.nonzero(res)[0].tolist()), sl,
                                  SimFlags(async_loading_enabled=async_on), cost)
        comp = [ev.expert for ev in plan.events if ev.category is EventCategory.COMPUTE]
        fs = [ev.start for ev in plan.events
              if ev.category in (EventCategory.EXPERT_LOAD_ASYNC, EventCategory.EXPERT_LOAD_SYNC)]
        wt = sum(ev.duration for ev in plan.events if ev.category is EventCategory.WAIT)
        E_list.append(E)
        works.append(work.astype(np.int64))
        residents.append(res)
        slots.append(sl)
        orders.append(np.array(comp, np.int32))
        spans.append(plan.span)
        fetch_starts.append(np.array(fs, np.float64))
        wait_total.append(wt)
        flags_async.append(async_on)
    return dict(
        E=np.array(E_list, np.int32), work=np.concatenate(works), resident=np.concatenate(residents),
        slots=np.array(slots, np.int32), order_len=np.array([len(o) for o in orders], np.int32),
        order=np.concatenate(orders) if orders else np.zeros(0, np.int32), span=np.array(spans),
        fetch_len=np.array([len(f) for f in fetch_starts], np.int32),
        fetch_start=np.concatenate(fetch_starts), wait=np.array(wait_total),
        async_on=np.array(flags_async), load_time=np.array(1.5),
    )


def trace_files():
    """A reference-written trace (workload.py:183-232) plus the reference's schedule of every
    (batch, layer) instance (engine.py:287-299, rebalance on, round-robin and blocked)."""
    from moesim import ModelSpec, SchedulerConfig, SkewSpec, WorkloadSpec, generate_trace, write_trace
    from moesim.engine import build_schedule
    from moesim.policies import PlacementKind, SchedulingPolicy

    model = ModelSpec(num_layers=3, num_experts=16, d_model=64, d_ff=128, dtype_bytes=2)
    spec = WorkloadSpec(num_batches=5, tokens_per_gpu_per_batch=700,
                        skew=SkewSpec(alpha=0.0, skewed_experts=(0, 5), mode="resample_uniform",
                                      resample_lo=0.3, resample_hi=0.95), seed=7)
    G = 4
    trace = generate_trace(spec, model, num_gpus=G)
    path = os.path.join(HERE, "trace_g4_e16.jsonl")
    write_trace(trace, path)
    print(f"wrote {path} ({os.path.getsize(path)} bytes)")
    out = {}
    for pl in ("round_robin", "blocked"):
        for q in (1, 17):
            kind = PlacementKind.ROUND_ROBIN if pl == "round_robin" else PlacementKind.BLOCKED
            cfg = SchedulerConfig(token_threshold_q=q, policy=SchedulingPolicy.REBALANCE, placement=kind)
            home = (round_robin_placement if pl == "round_robin" else blocked_placement)(16, G)
            S = [build_schedule(m, home, cfg, SimFlags()).counts for b in trace.batches for m in b.layers]
            out[f"S_{pl}_q{q}"] = np.stack(S).astype(np.int64)
            out[f"home_{pl}"] = np.asarray(home.home, np.int64)
    return out


def baseline_policies():
    """The paper's ablation baselines on the same seam: the reference's
    even_split_assign (policies.py:174-203) on every baseline-shape and acceptance routing
    matrix, and affinity_placement (policies.py:206-229) on random popularity profiles."""
    from moesim import PopularityProfile, affinity_placement, even_split_assign

    out = []
    for pack in (baseline_shapes(), acceptance_c2(400)):
        off = 0
        for G, E in zip(pack["G"], pack["E"]):
            m = pack["m"][off:off + G * E].reshape(G, E)
            off += G * E
            S = even_split_assign(RoutingMatrix(m), int(G)).counts
            out.append(dict(m=m, home=np.zeros(E, np.int64), q=1, S=S, iters=0))
    d = _pack(out)
    rng = np.random.default_rng(777)
    E_l, G_l, slots_l, counts_l, home_l = [], [], [], [], []
    for i in range(300):
        E = int(rng.integers(1, 160))
        G = int(rng.integers(1, 9))
        slots = -(-E // G) + int(rng.integers(0, 4))
        if i % 4 == 0:
            counts = rng.integers(0, 5, size=E)  # many ties
        else:
            counts = (rng.zipf(1.3, size=E) * rng.integers(1, 100)).clip(max=10**9)
        home = affinity_placement(PopularityProfile(counts=counts, window_batches=1), G, slots).home
        E_l.append(E)
        G_l.append(G)
        slots_l.append(slots)
        counts_l.append(np.asarray(counts, np.int64))
        home_l.append(np.asarray(home, np.int64))
    d.update(aff_E=np.array(E_l, np.int32), aff_G=np.array(G_l, np.int32), aff_slots=np.array(slots_l, np.int32),
             aff_counts=np.concatenate(counts_l), aff_home=np.concatenate(home_l))
    return d


def main():
    print("moesim", moesim.__version__, "numpy", np.__version__)
    for name, fn in [("fig4", fig4), ("acceptance_c2", acceptance_c2), ("baseline_shapes", baseline_shapes),
                     ("plan_order", plan_order), ("trace_g4_e16_schedules", trace_files),
                     ("baseline_policies", baseline_policies), ("wide_schedules", wide_schedules)]:
        if len(sys.argv) > 1 and name not in sys.argv[1:]:  # regenerate only the named fixtures
            continue
        d = fn()
        path = os.path.join(HERE, name + ".npz")
        np.savez_compressed(path, **d)
        print(f"wrote {path} ({os.path.getsize(path)} bytes)")


if __name__ == "__main__":
    main()
