"""MeasuredCostModel through the reference simulator's cost seam."""

import os
import sys

import numpy as np
import pytest

from conftest import GOLDEN, REPO
from paper_2506_12417_b200.costmodel import MeasuredCostModel


def _model(**kw):
    base = dict(d_model=768, d_ff=3072, dtype_bytes=2, n_matrices=2, metadata_time=2e-6, expert_load_time=1e-4,
                token_points=(1, 128, 256, 1024), compute_seconds=(2e-6, 2e-6, 3e-6, 9e-6))
    base.update(kw)
    return MeasuredCostModel(**base)


def _moesim():
    ref = os.path.join(REPO, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "moesim")):
        pytest.skip("reference not installed in baseline/_ref")
    if ref not in sys.path:
        sys.path.insert(0, ref)
    import moesim

    return moesim


def test_interpolation_and_derived_fields():
    c = _model()
    assert c.expert_compute_time(0) == 0.0
    assert c.expert_compute_time(1) == 2e-6
    assert c.expert_compute_time(64) == 2e-6  # flat between 1 and 128
    assert c.expert_compute_time(192) == pytest.approx(2.5e-6)
    assert c.expert_compute_time(2048) == pytest.approx(9e-6 + 6e-6 / 768 * 1024)  # extrapolated
    assert c.expert_bytes == 2 * 768 * 3072 * 2 and c.token_bytes == 768 * 2
    assert c.pcie_bandwidth == pytest.approx(c.expert_bytes / 1e-4)
    assert c.gpu_flops == pytest.approx(c.expert_flops(1024) / 9e-6)


def test_json_round_trip(tmp_path):
    c = _model(device_name="NVIDIA B200", load_source="host")
    p = tmp_path / "cost.json"
    c.to_json(p)
    assert MeasuredCostModel.from_json(p) == c
    assert MeasuredCostModel.from_json(c.to_json()) == c


@pytest.mark.parametrize("bad", [dict(token_points=(1,), compute_seconds=(1.0,)),
                                 dict(token_points=(4, 2, 8, 9)),
                                 dict(compute_seconds=(1, -1, 1, 1)),
                                 dict(expert_load_time=-1.0)])
def test_validation(bad):
    with pytest.raises(ValueError):
        _model(**bad)


def test_reference_simulate_run_accepts_measured_cost():
    """moesim.simulate_run(..., cost=MeasuredCostModel) replays a reference-written trace; the
    schedule-derived outputs are unchanged and latencies follow the injected costs."""
    moesim = _moesim()
    trace = moesim.read_trace(os.path.join(GOLDEN, "trace_g4_e16.jsonl"))
    model = moesim.ModelSpec(num_layers=3, num_experts=16, d_model=64, d_ff=128, dtype_bytes=2)
    cluster = moesim.ClusterSpec(num_gpus=4, expert_slots_per_gpu=8, link_bandwidth=9e11, link_latency=1e-6,
                                 pcie_bandwidth=5.5e10, gpu_flops=1.6e15)
    cfg = moesim.SchedulerConfig(token_threshold_q=17, placement=moesim.PlacementKind.BLOCKED)
    flags = moesim.SimFlags()
    cost = MeasuredCostModel(d_model=64, d_ff=128, dtype_bytes=2, n_matrices=2, metadata_time=3e-6,
                             expert_load_time=5e-6, token_points=(1, 128, 1024),
                             compute_seconds=(1e-6, 1e-6, 4e-6))
    base = moesim.simulate_run(trace, model, cluster, cfg, flags)
    got = moesim.simulate_run(trace, model, cluster, cfg, flags, cost=cost)
    for a, b in zip(base.per_gpu_token_loads, got.per_gpu_token_loads):
        assert np.array_equal(a, b)
    assert len(got.per_batch_latency) == trace.num_batches
    assert all(lat > 3 * 3e-6 for lat in got.per_batch_latency)  # >= metadata per layer
    assert got.per_batch_latency != base.per_batch_latency
