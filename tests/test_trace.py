"""Trace JSONL format against a file the reference itself wrote.

Mirrors the reference's trace tests (test_workload.py:136-183): round trip, empty trace,
malformed files named by line; plus byte-identity with the reference writer and the
oracle's schedules of every (batch, layer) against the reference's build_schedule.
"""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import moe_oracle as orc
from paper_2506_12417_b200.trace import Trace, TraceParseError, read_trace, write_trace

REF_TRACE = os.path.join(GOLDEN, "trace_g4_e16.jsonl")


def test_reference_file_parses():
    t = read_trace(REF_TRACE)
    assert (t.num_gpus, t.num_experts, t.num_layers, t.num_batches) == (4, 16, 3, 5)
    assert t.rng_name == "numpy-pcg64" and t.seed == 7
    c = t.counts()
    assert c.shape == (5, 3, 4, 16) and c.dtype == np.int64
    assert (c.sum(axis=3) == 700).all()  # tokens_per_gpu_per_batch
    assert t.tokens_per_batch() == 4 * 700
    assert [b.batch_id for b in t.batches] == list(range(5))
    assert all(0.3 <= b.alpha <= 0.95 for b in t.batches)


def test_write_is_byte_identical_to_reference(tmp_path):
    t = read_trace(REF_TRACE)
    out = tmp_path / "t.jsonl"
    write_trace(t, out)
    assert out.read_bytes() == open(REF_TRACE, "rb").read()
    assert read_trace(out) == t


def test_empty_trace_round_trip(tmp_path):
    t = Trace(num_gpus=2, num_experts=4, num_layers=2, seed=1)
    p = tmp_path / "empty.jsonl"
    write_trace(t, p)
    back = read_trace(p)
    assert back == t and back.num_batches == 0 and back.tokens_per_batch() == 0


def test_append_validates():
    t = Trace(num_gpus=2, num_experts=3, num_layers=2)
    t.append(np.array([[[1, 2, 3], [0, 0, 4]], [[3, 3, 0], [2, 1, 1]]]), alpha=0.5)
    assert t.num_batches == 1 and t.batches[0].batch_id == 0
    with pytest.raises(ValueError):
        t.append(np.ones((1, 2, 3), np.int64))  # wrong layer count
    with pytest.raises(ValueError):
        t.append(np.array([[[1, 2, 3], [0, 0, 4]], [[3, 3, 1], [2, 1, 1]]]))  # row sums differ
    with pytest.raises(ValueError):
        t.append(-np.ones((2, 2, 3), np.int64))


def _corrupt(tmp_path, fn, name="bad.jsonl"):
    lines = open(REF_TRACE).read().splitlines()
    fn(lines)
    p = tmp_path / name
    p.write_text("\n".join(lines) + "\n")
    return p


def test_negative_count_names_line(tmp_path):
    # test_workload.py:153-161
    def neg(lines):
        lines[2] = lines[2].replace("[[[", "[[[-", 1)

    with pytest.raises(TraceParseError, match="line 3") as ei:
        read_trace(_corrupt(tmp_path, neg))
    assert ei.value.line_no == 3 and "negative" in str(ei.value)


def test_truncated_layer_names_line(tmp_path):
    # test_workload.py:164-176
    def trunc(lines):
        rec = json.loads(lines[1])
        rec["layers"] = rec["layers"][:-1]
        lines[1] = json.dumps(rec)

    with pytest.raises(TraceParseError, match="line 2"):
        read_trace(_corrupt(tmp_path, trunc))


def test_invalid_json_names_line(tmp_path):
    # test_workload.py:179-183
    p = tmp_path / "garbled.jsonl"
    p.write_text('{"version": 1, "num_gpus": 2, "num_experts": 4, "num_layers": 1, "rng": "numpy-pcg64", '
                 '"seed": 0}\nnot json\n')
    with pytest.raises(TraceParseError, match="line 2"):
        read_trace(p)


@pytest.mark.parametrize("case", ["short_row", "float", "row_sums", "missing_key", "not_object"])
def test_structural_errors_name_line(tmp_path, case):
    def mutate(lines):
        rec = json.loads(lines[4])  # batch 3 -> line 5
        if case == "short_row":
            rec["layers"][1][2] = rec["layers"][1][2][:-1]
        elif case == "float":
            rec["layers"][0][0][0] = 1.5
        elif case == "row_sums":
            rec["layers"][2][0][0] += 1
        elif case == "missing_key":
            del rec["alpha_used"]
        elif case == "not_object":
            rec = [1, 2]
        lines[4] = json.dumps(rec)

    with pytest.raises(TraceParseError, match="line 5"):
        read_trace(_corrupt(tmp_path, mutate))


@pytest.mark.parametrize("header", ["", '{"version": 2, "num_gpus": 1, "num_experts": 1, "num_layers": 1, '
                                        '"rng": "x", "seed": 0}',
                                    '{"version": 1, "num_gpus": 1, "num_experts": 1, "rng": "x", "seed": 0}',
                                    '{"version": 1, "num_gpus": 0, "num_experts": 1, "num_layers": 1, '
                                    '"rng": "x", "seed": 0}'])
def test_bad_header_is_line_1(tmp_path, header):
    p = tmp_path / "h.jsonl"
    p.write_text(header)
    with pytest.raises(TraceParseError, match="line 1"):
        read_trace(p)


def test_oracle_schedules_trace_like_reference(golden):
    """The oracle's per-(batch, layer) schedule == the reference's build_schedule of the same file."""
    t = read_trace(REF_TRACE)
    ref = golden("trace_g4_e16_schedules")
    m = t.counts().reshape(-1, 4, 16)
    for pl in ("round_robin", "blocked"):
        for q in (1, 17):
            want = ref[f"S_{pl}_q{q}"]
            assert want.shape == (15, 4, 16, 4)
            for i in range(m.shape[0]):
                S, _ = orc.schedule(m[i], ref[f"home_{pl}"], q, rebalance=True)
                assert np.array_equal(S, want[i]), (pl, q, i)


def test_generate_trace_reproduces_reference_file(tmp_path):
    """generate_trace / sample_routing / SkewSpec / WorkloadSpec (workload.py:40-210): the spec
    make_golden.py handed the reference reproduces the reference-written file byte for byte
    (same numpy build; cross-version RNG stability is not promised)."""
    from paper_2506_12417_b200 import ModelSpec, SkewSpec, WorkloadSpec, generate_trace

    model = ModelSpec(num_layers=3, num_experts=16, d_model=64, d_ff=128, dtype_bytes=2)
    spec = WorkloadSpec(num_batches=5, tokens_per_gpu_per_batch=700,
                        skew=SkewSpec(alpha=0.0, skewed_experts=(0, 5), mode="resample_uniform",
                                      resample_lo=0.3, resample_hi=0.95), seed=7)
    t = generate_trace(spec, model, num_gpus=4)
    ref = read_trace(REF_TRACE)
    if t != ref:
        pytest.skip(f"numpy {np.__version__} draws a different PCG64 multinomial stream than the fixture's build")
    out = tmp_path / "g.jsonl"
    write_trace(t, out)
    assert out.read_bytes() == open(REF_TRACE, "rb").read()


def test_workload_spec_validation():
    from paper_2506_12417_b200 import RoutingMatrix, SkewSpec, WorkloadSpec, sample_routing

    with pytest.raises(ValueError, match="alpha"):
        SkewSpec(alpha=1.5)
    with pytest.raises(ValueError, match="unknown per-batch mode"):
        SkewSpec(alpha=0.5, mode="nope")
    with pytest.raises(ValueError, match="resample bounds"):
        SkewSpec(alpha=0.0, mode="resample_uniform", resample_lo=0.9, resample_hi=0.1)
    with pytest.raises(ValueError, match="distinct"):
        SkewSpec(alpha=0.5, skewed_experts=(1, 1))
    with pytest.raises(ValueError, match="non-empty"):
        SkewSpec(alpha=0.5, skewed_experts=())
    with pytest.raises(ValueError, match="num_batches"):
        WorkloadSpec(num_batches=0, tokens_per_gpu_per_batch=1, skew=SkewSpec(alpha=0.0), seed=0)
    with pytest.raises(ValueError, match="sum to 1"):
        sample_routing(np.array([0.5, 0.6]), 10, 2, np.random.default_rng(0))
    m = sample_routing(np.array([0.25, 0.75]), 10, 3, np.random.default_rng(0))
    assert isinstance(m, RoutingMatrix) and m.counts.shape == (3, 2) and (m.counts.sum(axis=1) == 10).all()
