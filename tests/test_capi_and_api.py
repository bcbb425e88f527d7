"""CPU-side checks of the boundary: the C-ABI library loads and exports every
symbol include/harmoe.h declares; the Python layer mirrors the reference API
(value types, placements, threshold, error behaviour) and fails loudly (no
CPU fallback) when no GPU is present."""

import os
import re
import subprocess

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(REPO, "include", "harmoe.h")
LIB = os.path.join(REPO, "paper_2506_12417_b200", "libharmoe.so")


def header_symbols():
    src = open(HEADER).read()
    return re.findall(r"^HM_API\s+[\w\s\*]+?\b(hm_\w+)\s*\(", src, flags=re.M)


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(LIB):
        subprocess.run(["make", "-s", "-j8", "-C", os.path.join(REPO, "paper_2506_12417_b200", "csrc")], check=True)
    from paper_2506_12417_b200 import _lib

    return _lib.load()


def test_library_exports_every_header_symbol(lib):
    syms = header_symbols()
    assert len(syms) >= 14
    for s in syms:
        assert hasattr(lib, s), f"{s} declared in harmoe.h but not exported"
    from paper_2506_12417_b200 import _lib

    assert set(syms) == set(_lib.SIGNATURES), "ctypes signature table out of sync with harmoe.h"
    assert lib.hm_version() == 1
    assert lib.hm_gemm_tile_m() == 128


def test_exported_symbols_are_only_the_abi():
    out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True).stdout
    exported = {ln.split()[-1] for ln in out.splitlines() if " T " in ln}
    assert {s for s in exported if s.startswith("hm_")} == set(header_symbols())


def test_sass_has_tcgen05_and_tma():
    out = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    assert "UTCHMMA" in out, "grouped GEMM / router must issue tcgen05.mma"
    assert "UTMALDG" in out, "operands must be staged by TMA"
    assert "LDTM" in out, "epilogues must read TMEM with tcgen05.ld"
    assert "HMMA" not in out.replace("UTCHMMA", ""), "no legacy mma.sync path"


def test_value_types_mirror_reference():
    from paper_2506_12417_b200 import (Placement, RoutingMatrix, ScheduleTensor, blocked_placement,
                                        load_per_gpu, round_robin_placement, total_tokens, validate_against)

    m = RoutingMatrix([[1, 1, 3], [1, 1, 3], [0, 2, 3]])
    assert m.counts.flags.writeable is False and m.counts.dtype == np.int64
    with pytest.raises(ValueError):
        RoutingMatrix([1, 2, 3])
    with pytest.raises(ValueError):
        RoutingMatrix([[1, -1]])
    with pytest.raises(ValueError):
        ScheduleTensor(np.zeros((2, 3, 4)))
    S = np.zeros((3, 3, 3), np.int64)
    for g in range(3):
        for e in range(3):
            S[g, e, e] = m.counts[g, e]
    s = ScheduleTensor(S)
    assert load_per_gpu(s).tolist() == [2, 4, 9] and total_tokens(s) == 15
    assert validate_against(s, m)
    assert round_robin_placement(128, 8).homes_on(0) == tuple(range(0, 128, 8))
    assert blocked_placement(5, 3).home == (0, 0, 1, 1, 2)
    with pytest.raises(ValueError):
        Placement(home=(0, 3), num_gpus=2)
    assert Placement(home=(0, 0, 1), num_gpus=2).fits(2) and not Placement(home=(0, 0, 0), num_gpus=2).fits(2)


def test_threshold_matches_reference_known_values():
    # test_policies.py:206-224 known answers (876 / 2 / 64) and the B200 Eq. 4 value
    from paper_2506_12417_b200 import estimate_token_threshold

    assert estimate_token_threshold(14e12, 2, 16e9) == 876
    assert estimate_token_threshold(1.0, 2.0, 1.0) == 2
    assert estimate_token_threshold(1e12, 1, 8e9) == 64
    assert estimate_token_threshold(1.3474e15, 2, 900e9) == 1499
    with pytest.raises(ValueError):
        estimate_token_threshold(0, 2, 1)


def test_no_cpu_fallback_without_gpu():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2506_12417_b200 import Placement, RoutingMatrix, initial_assign, rebalance

    m = RoutingMatrix([[1, 2], [3, 4]])
    with pytest.raises(RuntimeError):
        initial_assign(m, Placement(home=(0, 1), num_gpus=2))
    with pytest.raises(ValueError):  # argument errors precede the device check, like the reference
        rebalance(None, 0)
    from paper_2506_12417_b200 import ops

    with pytest.raises(ValueError):
        ops.combine(torch.zeros(4, 8), None, torch.zeros(2, 2))


def test_extract_expert_weights_hf_layouts():
    torch = pytest.importorskip("torch")
    from torch import nn

    from paper_2506_12417_b200.integration import extract_expert_weights

    class Ex(nn.Module):
        def __init__(self):
            super().__init__()
            self.gate_proj, self.up_proj, self.down_proj = nn.Linear(8, 16), nn.Linear(8, 16), nn.Linear(16, 8)

    ex = nn.ModuleList([Ex() for _ in range(3)])
    w1, w2, w3 = extract_expert_weights(ex, "swiglu")
    assert w1.shape == (3, 16, 8) and w2.shape == (3, 8, 16) and w3.shape == (3, 16, 8)
    assert torch.equal(w1[1], ex[1].gate_proj.weight)

    class Fused(nn.Module):
        def __init__(self):
            super().__init__()
            self.gate_up_proj = nn.Parameter(torch.randn(3, 8, 32))
            self.down_proj = nn.Parameter(torch.randn(3, 16, 8))

    fz = Fused()
    w1, w2, w3 = extract_expert_weights(fz, "swiglu", d_model=8)
    assert torch.equal(w1[2], fz.gate_up_proj[2, :, :16].T) and torch.equal(w2[0], fz.down_proj[0].T)
    assert torch.equal(w3[1], fz.gate_up_proj[1, :, 16:].T)

    # transformers 5 fused experts (Qwen3MoeExperts / MixtralExperts): [E, 2f, d] gate rows first,
    # down [E, d, f]; hidden_dim disambiguates 2f == d
    from transformers.models.qwen3_moe.configuration_qwen3_moe import Qwen3MoeConfig
    from transformers.models.qwen3_moe.modeling_qwen3_moe import Qwen3MoeExperts

    hf = Qwen3MoeExperts(Qwen3MoeConfig(hidden_size=16, moe_intermediate_size=8, num_experts=3))
    nn.init.normal_(hf.gate_up_proj)
    nn.init.normal_(hf.down_proj)
    w1, w2, w3 = extract_expert_weights(hf, "swiglu")
    assert w1.shape == (3, 8, 16) and w3.shape == (3, 8, 16) and w2.shape == (3, 16, 8)
    assert torch.equal(w1[1], hf.gate_up_proj[1, :8]) and torch.equal(w3[1], hf.gate_up_proj[1, 8:])
    assert torch.equal(w2[2], hf.down_proj[2])
    with pytest.raises(ValueError):
        extract_expert_weights(Fused(), "swiglu", d_model=5)


def test_patch_moesim_rejects_mismatched_placement():
    """The patched build_schedule keeps the reference's dimension check (policies.py:111-112)
    instead of handing the kernel an out-of-range home vector (checked before any GPU call)."""
    import sys

    ref = os.path.join(REPO, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "moesim")):
        pytest.skip("reference not installed in baseline/_ref")
    sys.path.insert(0, ref)
    import moesim

    from paper_2506_12417_b200.integration import patch_moesim

    restore = patch_moesim(moesim)
    try:
        m = moesim.RoutingMatrix(np.ones((2, 4), np.int64))
        cfg = moesim.SchedulerConfig(token_threshold_q=1)
        for pl in (moesim.round_robin_placement(4, 3), moesim.round_robin_placement(5, 2)):
            with pytest.raises(ValueError, match="placement dimensions"):
                moesim.engine.build_schedule(m, pl, cfg, moesim.SimFlags())
    finally:
        restore()


def test_replace_moe_layer_takes_routing_semantics_from_the_module():
    """norm_topk_prob of the replaced HF router sets MoEConfig.renormalize (shipped Qwen2-MoE
    checkpoints use False); a top_k that disagrees with the module is an error."""
    import torch
    from torch import nn

    from paper_2506_12417_b200 import MoEConfig
    from paper_2506_12417_b200.integration import _routing_config

    class Router(nn.Module):
        def __init__(self, k, ntp):
            super().__init__()
            self.top_k, self.norm_topk_prob = k, ntp
            self.weight = nn.Parameter(torch.zeros(16, 256))

    cfg = MoEConfig(d_model=256, num_experts=16, d_ff=256, top_k=4)
    assert cfg.renormalize is True
    assert _routing_config(nn.Module(), Router(4, False), cfg).renormalize is False
    assert _routing_config(nn.Module(), Router(4, True), cfg).renormalize is True
    assert _routing_config(nn.Module(), nn.Linear(256, 16), cfg).renormalize is True  # no attribute: keep
    with pytest.raises(ValueError, match="top-2"):
        _routing_config(nn.Module(), Router(2, True), cfg)


def test_bounded_cache_needs_async_fetch():
    """Synchronous loading (fetches in stream order ahead of FFN1) cannot wait for cache slots
    that only FFN1 / FFN2 free, so a bounded expert cache with async_fetch=False is rejected."""
    from paper_2506_12417_b200 import MoEConfig

    kw = dict(d_model=256, num_experts=16, d_ff=256, top_k=2, world_size=2, rank=0)
    MoEConfig(expert_cache_size=2, **kw)  # async: fine
    MoEConfig(expert_cache_size=8, async_fetch=False, **kw)  # every fetchable expert has a slot
    with pytest.raises(ValueError, match="async_fetch"):
        MoEConfig(expert_cache_size=2, async_fetch=False, **kw)
    with pytest.raises(ValueError, match="expert_cache_size"):
        MoEConfig(expert_cache_size=-1, **kw)


def test_new_entry_points_validate_before_touching_the_device(lib):
    """Round-2 entry points reject bad arguments with HM_EINVAL before any CUDA call (so this
    runs without a GPU): the swap-AB GEMM's epilogues, the ordered push's power-of-two G, the
    push work list's required outputs."""
    import ctypes

    from paper_2506_12417_b200 import _lib

    L = _lib.load()
    vp = ctypes.c_void_p
    # SwiGLU is not a swap-AB epilogue
    assert L.hm_grouped_gemm_swap(None, 0, None, 256, 256, 64, None, None, _lib.HM_EPI_SWIGLU, vp(16), None,
                                  None, None, None, None) == _lib.HM_EINVAL
    # N must be a multiple of 256
    assert L.hm_grouped_gemm_swap(None, 0, None, 100, 100, 64, None, None, _lib.HM_EPI_STORE, vp(16), None,
                                  None, None, None, None) == _lib.HM_EINVAL
    # G = 3 is not a power of two
    assert L.hm_dispatch_push_ordered(None, None, None, None, None, None, vp(16), vp(16), vp(16), 8, 0, 3, 16, 2, 256,
                                      vp(16), vp(16), vp(16), vp(16), None, vp(16), None) == _lib.HM_EINVAL
    # the push work list is required
    assert L.hm_plan_dispatch(None, None, 4, 16, 4, 1, 0, *([None] * 9), 0, None, None, None, None) == _lib.HM_EINVAL
    assert b"push_items" in L.hm_last_error()
