"""bench.py's reference arm (CPU) prints the contract's JSON line: one line, the same metric /
unit / direction as the GPU arm, a cpu_baseline describing the run and a zero-copy e2e."""

import json
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--impl", "reference", "--steps", "2",
                          "--warmup", "1", "--workload", "switch128"],
                         capture_output=True, text=True, timeout=600, cwd=REPO)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference"
    assert d["metric"] == "moe_block_tokens_per_sec" and d["unit"] == "tokens/s" and d["higher_is_better"] is True
    assert d["value"] > 0 and d["steps"] == 2 and d["warmup"] == 1 and d["n_gpus"] == 1
    cb = d["cpu_baseline"]
    assert cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    assert cb["host"]["os_cpu_count"] >= 1 and cb["host"]["sched_getaffinity"] >= 1
    if os.path.isdir(os.path.join(REPO, "baseline", "_ref", "moesim")):
        # the reference itself schedules the batch (moesim.build_schedule on its m_all)
        assert cb["kind"] == "reference" and "moesim" in cb["sample"]
        ms = cb["moesim"]
        assert ms["build_schedule_us"] > 0 and ms["rebalance_with_stats_us"] > 0 and ms["simulate_layer_us"] > 0
        assert ms["build_schedule_reps"] >= 20 and ms["G"] == 8 and ms["iterations"] > 0
        assert ms["load_max_over_mean"] <= 1.1
        assert cb["port"]["kind"] == "port" and cb["port"]["value"] > 0
    else:
        assert cb["kind"] == "port"
    assert d["e2e"] == {"value": d["value"], "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


def test_reference_arm_other_ranks_exit_quietly():
    env = dict(os.environ, RANK="1", WORLD_SIZE="2", LOCAL_RANK="1")
    out = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--impl", "reference", "--gpus", "2"],
                         capture_output=True, text=True, timeout=120, cwd=REPO, env=env)
    assert out.returncode == 0 and not out.stdout.strip()


def test_launch_mismatch_exits_nonzero():
    """A launch whose WORLD_SIZE disagrees with --gpus never prints a line (exit 2)."""
    env = dict(os.environ, RANK="0", WORLD_SIZE="2", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--impl", "reference", "--gpus", "1"],
                         capture_output=True, text=True, timeout=120, cwd=REPO, env=env)
    assert out.returncode == 2 and not out.stdout.strip()
    assert "WORLD_SIZE=2" in out.stderr


def test_gpus_n_self_launches_n_ranks():
    """--gpus 2 without a launcher starts 2 ranks itself (torch.distributed.run); here each
    rank then stops at the GPU check (no CUDA device), which must fail loudly, not print a
    1-GPU line."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--gpus", "2", "--steps", "1",
                          "--warmup", "1"], capture_output=True, text=True, timeout=300, cwd=REPO, env=env)
    assert "launching 2 ranks" in out.stderr
    assert '"n_gpus": 1' not in out.stdout
    import torch

    if not torch.cuda.is_available():
        assert out.returncode != 0
