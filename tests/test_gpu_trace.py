"""Batched GPU scheduler + trace record/replay on the B200."""

import os

import numpy as np
import pytest
import torch

from conftest import GOLDEN, iter_packed
from oracle import moe_oracle as orc

pytestmark = pytest.mark.gpu


def test_replay_reference_trace_bit_exact(golden):
    from paper_2506_12417_b200.trace import read_trace, replay_schedules

    t = read_trace(os.path.join(GOLDEN, "trace_g4_e16.jsonl"))
    ref = golden("trace_g4_e16_schedules")
    for pl in ("round_robin", "blocked"):
        for q in (1, 17):
            r = replay_schedules(t, ref[f"home_{pl}"], q)
            assert np.array_equal(r.S.reshape(-1, 4, 16, 4), ref[f"S_{pl}_q{q}"]), (pl, q)
            assert np.array_equal(r.loads, r.S.sum(axis=(2, 3)))
            assert (r.max_over_mean() >= 1.0).all()


def test_schedule_batched_matches_golden_instances(golden):
    """Every baseline_shapes instance with the same (G, E, q, home) batched into one launch."""
    from paper_2506_12417_b200 import ops

    groups = {}
    for inst in iter_packed(golden("baseline_shapes")):
        key = (inst["m"].shape, inst["q"], inst["home"].tobytes())
        groups.setdefault(key, []).append(inst)
    n = 0
    for (shape, q, _), insts in groups.items():
        m = torch.tensor(np.stack([i["m"] for i in insts]), dtype=torch.int32, device="cuda")
        home = torch.tensor(insts[0]["home"], dtype=torch.int32, device="cuda")
        S, iters, loads = ops.schedule_batched(m, home, q)
        S = S.cpu().numpy()
        for b, inst in enumerate(insts):
            assert np.array_equal(S[b], inst["S"]), inst["i"]
            assert int(iters[b]) == inst["iters"], inst["i"]
            n += 1
    assert n == 384


def test_schedule_batched_random_vs_oracle():
    from paper_2506_12417_b200 import ops

    rng = np.random.default_rng(5)
    for G, E, q in [(8, 128, 1), (8, 128, 32), (4, 64, 5), (2, 8, 1), (1, 16, 1)]:
        B = 37
        m = rng.integers(0, 300, size=(B, G, E)) * (rng.random((B, G, E)) < 0.6)
        m[:, :, 0] += rng.integers(0, 5000, size=(B, G))  # a hot expert
        home = orc.blocked_home(E, G)
        S, iters, loads = ops.schedule_batched(torch.tensor(m, dtype=torch.int32, device="cuda"),
                                               torch.tensor(home, dtype=torch.int32, device="cuda"), q)
        S = S.cpu().numpy()
        for b in range(B):
            want, it = orc.schedule(m[b], home, q)
            assert np.array_equal(S[b], want), (G, E, q, b)
            assert int(iters[b]) == it
    # empty batch is a no-op, bad q raises
    S, _, _ = ops.schedule_batched(torch.zeros((0, 2, 4), dtype=torch.int32, device="cuda"),
                                   torch.zeros(4, dtype=torch.int32, device="cuda"), 1)
    assert S.shape == (0, 2, 4, 2)
    with pytest.raises(ValueError):
        ops.schedule_batched(torch.zeros((1, 2, 4), dtype=torch.int32, device="cuda"),
                             torch.zeros(4, dtype=torch.int32, device="cuda"), 0)


def test_record_stack_then_replay_matches_live_schedules(tmp_path):
    """Record the real routing of a 3-layer stack, write/read the file, replay it: the
    replayed schedules are bit-identical to the ones the live forward used."""
    from paper_2506_12417_b200.block import MoEConfig
    from paper_2506_12417_b200.stack import MoEStack
    from paper_2506_12417_b200.trace import TraceRecorder, read_trace, replay_schedules, write_trace

    cfg = MoEConfig(d_model=256, d_ff=256, num_experts=16, top_k=2, logical_ranks=4, eq_tokens=8,
                    placement="blocked")
    stack = MoEStack.random(cfg, num_layers=3, seed=3, zipf_s=1.2)
    rec = TraceRecorder(stack, seed=3)
    live = []
    g = torch.Generator(device="cpu").manual_seed(0)
    for b in range(3):
        x = torch.randn((512, 256), generator=g).to(device="cuda", dtype=torch.bfloat16)
        stack(x)
        torch.cuda.synchronize()
        rec.record(alpha=0.0)
        live.append(np.stack([s.schedule.cpu().numpy() for s in stack.stats]))
    p = tmp_path / "rec.jsonl"
    write_trace(rec.trace, p)
    t = read_trace(p)
    assert t == rec.trace and t.num_gpus == 4 and t.num_layers == 3 and t.rng_name == "b200-router"
    assert (t.counts().sum(axis=(2, 3)) == 512 * 2).all()
    assert np.array_equal(stack.layers[0].home_np, orc.blocked_home(16, 4))
    r = replay_schedules(t, stack.layers[0].home_np, cfg.eq_tokens)
    assert np.array_equal(r.S, np.stack(live).reshape(r.S.shape))


def test_measure_cost_model_on_b200(tmp_path):
    from paper_2506_12417_b200.block import MoEConfig
    from paper_2506_12417_b200.costmodel import MeasuredCostModel, measure_cost_model

    cfg = MoEConfig(d_model=2048, d_ff=768, num_experts=128, top_k=8, logical_ranks=8)
    c = measure_cost_model(cfg, token_points=(1, 128, 512, 2048), reps=5)
    assert c.n_matrices == 3 and c.expert_bytes == 3 * 2048 * 768 * 2
    assert all(s > 0 for s in c.compute_seconds)
    assert c.compute_seconds[-1] > c.compute_seconds[0]  # more tokens cost more
    # 2048 tokens/expert at >= 30% of the measured bf16 peak (loose: this is a sanity bound)
    assert c.gpu_flops > 0.3 * 1.3e15, c.gpu_flops
    assert 0 < c.expert_load_time < 5e-3 and 0 < c.metadata_time < 1e-3
    p = tmp_path / "cost.json"
    c.to_json(p)
    assert MeasuredCostModel.from_json(p) == c
