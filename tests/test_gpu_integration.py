"""Drop-in seams on the GPU:

* patch_moesim(): the reference simulator (baseline/_ref, installed from
  /root/reference/pkg) runs with its build_schedule/rebalance rebound to the
  B200 scheduler kernel and produces identical layer results and run metrics;
* replace_moe_layer(): a PyTorch MoE model (HF-style expert names) keeps its
  outputs (vs the original fp32 torch forward) after its MoE modules are
  swapped for HarMoEnyLayer.
"""

import os
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
from torch import nn  # noqa: E402

pytestmark = pytest.mark.gpu
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda")


def _moesim():
    ref = os.path.join(REPO, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "moesim")):
        pytest.skip("reference not installed in baseline/_ref")
    if ref not in sys.path:
        sys.path.insert(0, ref)
    import moesim

    return moesim


def _assert_hf_parity(got, ref, x, gate_w, k, what):
    """The stated bar (|y - y_ref| <= 1e-2 + 2e-2 |y_ref| elementwise, relative
    Frobenius <= 5e-3) against the module's own fp32 forward, on every token except those whose
    top-k, computed in fp64 from the module's gate weights, is decided by a near tie (there the
    fp32 HF router and the bf16-input tcgen05 router may legitimately pick different experts;
    the near-tie count is printed)."""
    from oracle import moe_oracle as orc

    d = x.shape[-1]
    logits = x.reshape(-1, d).double().cpu().numpy() @ gate_w.detach().double().cpu().numpy().T
    near = orc.topk_min_gap(logits, k) < orc.NEAR_TIE_REL * np.maximum(1.0, np.abs(logits).max(axis=1))
    g = got.reshape(-1, d).double().cpu().numpy()[~near]
    r = ref.reshape(-1, d).double().cpu().numpy()[~near]
    err = np.abs(g - r)
    bar = 1e-2 + 2e-2 * np.abs(r)
    frob = float(np.linalg.norm(g - r) / np.linalg.norm(r))
    print(f"[hf parity] {what}: {int(near.sum())} near-tie tokens of {len(near)}, worst ratio "
          f"{float((err / bar).max()):.3f}, Frobenius {frob:.2e}")
    assert np.all(err <= bar), f"{what}: {(err > bar).sum()} elements out of the stated bar"
    assert frob <= 5e-3, f"{what}: relative Frobenius error {frob}"


def test_patch_moesim_simulate_run_identical():
    _cuda()
    moesim = _moesim()
    from paper_2506_12417_b200.integration import patch_moesim

    model = moesim.model_preset("switch128")
    cluster = moesim.ClusterSpec(num_gpus=8, expert_slots_per_gpu=16, link_bandwidth=2e11, link_latency=1e-6,
                                 pcie_bandwidth=8e9, gpu_flops=1e12)
    wl = moesim.WorkloadSpec(num_batches=2, tokens_per_gpu_per_batch=8192,
                             skew=moesim.SkewSpec(alpha=0.9, skewed_experts=tuple(range(10))), seed=7)
    trace = moesim.generate_trace(wl, model, cluster.num_gpus)
    cfg = moesim.SchedulerConfig(token_threshold_q=64, policy=moesim.SchedulingPolicy.REBALANCE,
                                 placement=moesim.PlacementKind.BLOCKED)
    ref = moesim.simulate_run(trace, model, cluster, cfg, moesim.SimFlags())
    restore = patch_moesim(moesim)
    try:
        got = moesim.simulate_run(trace, model, cluster, cfg, moesim.SimFlags())
        for a, b in zip(ref.per_gpu_token_loads, got.per_gpu_token_loads):
            assert np.array_equal(a, b)
        assert ref.per_batch_latency == got.per_batch_latency
        # Fig. 4 layer through the patched seam
        m = moesim.RoutingMatrix([[1, 1, 3], [1, 1, 3], [0, 2, 3]])
        s = moesim.engine.build_schedule(m, moesim.Placement(home=(0, 1, 2), num_gpus=3),
                                         moesim.SchedulerConfig(token_threshold_q=1), moesim.SimFlags())
        assert moesim.load_per_gpu(s).tolist() == [5, 5, 5]
    finally:
        restore()


@pytest.mark.parametrize("policy", ["EVEN_SPLIT", "AFFINITY"])
def test_patch_moesim_baseline_policies_identical(policy):
    """The ablation baselines through the patched seam (GPU even split, affinity placement)
    reproduce the reference simulator's loads and latencies exactly (engine.py:292-293,435-440)."""
    _cuda()
    moesim = _moesim()
    from paper_2506_12417_b200.integration import patch_moesim

    model = moesim.model_preset("switch128")
    cluster = moesim.ClusterSpec(num_gpus=4, expert_slots_per_gpu=40, link_bandwidth=2e11, link_latency=1e-6,
                                 pcie_bandwidth=8e9, gpu_flops=1e12)
    wl = moesim.WorkloadSpec(num_batches=4, tokens_per_gpu_per_batch=4096,
                             skew=moesim.SkewSpec(alpha=0.8, skewed_experts=tuple(range(6))), seed=11)
    trace = moesim.generate_trace(wl, model, cluster.num_gpus)
    cfg = moesim.SchedulerConfig(token_threshold_q=32, policy=getattr(moesim.SchedulingPolicy, policy),
                                 placement=moesim.PlacementKind.ROUND_ROBIN,
                                 affinity_refresh_batches=2 if policy == "AFFINITY" else None)
    ref = moesim.simulate_run(trace, model, cluster, cfg, moesim.SimFlags())
    restore = patch_moesim(moesim)
    try:
        got = moesim.simulate_run(trace, model, cluster, cfg, moesim.SimFlags())
    finally:
        restore()
    for a, b in zip(ref.per_gpu_token_loads, got.per_gpu_token_loads):
        assert np.array_equal(a, b)
    assert ref.per_batch_latency == got.per_batch_latency


class _Expert(nn.Module):
    def __init__(self, d, f):
        super().__init__()
        self.gate_proj = nn.Linear(d, f, bias=False)
        self.up_proj = nn.Linear(d, f, bias=False)
        self.down_proj = nn.Linear(f, d, bias=False)

    def forward(self, x):
        return self.down_proj(nn.functional.silu(self.gate_proj(x)) * self.up_proj(x))


class _MoE(nn.Module):
    def __init__(self, d, f, E, k):
        super().__init__()
        self.gate = nn.Linear(d, E, bias=False)
        self.experts = nn.ModuleList([_Expert(d, f) for _ in range(E)])
        self.k = k

    def forward(self, x):
        shape = x.shape
        x = x.reshape(-1, shape[-1])
        p = torch.softmax(self.gate(x).float(), dim=-1)
        w, idx = torch.topk(p, self.k, dim=-1)
        w = w / w.sum(-1, keepdim=True)
        y = torch.zeros_like(x)
        for e in range(len(self.experts)):
            t, j = torch.nonzero(idx == e, as_tuple=True)
            if t.numel():
                y[t] += w[t, j, None] * self.experts[e](x[t])
        return y.reshape(shape)


class _Layer(nn.Module):
    def __init__(self, d, f, E, k):
        super().__init__()
        self.mlp = _MoE(d, f, E, k)

    def forward(self, x):
        return x + self.mlp(x)


def test_replace_moe_layer_matches_torch_reference():
    dev = _cuda()
    from paper_2506_12417_b200 import MoEConfig, replace_moe_layer

    torch.manual_seed(0)
    d, f, E, k = 256, 256, 16, 2
    model = nn.Sequential(_Layer(d, f, E, k), _Layer(d, f, E, k)).to(dev)
    for p in model.parameters():
        p.data = p.data.to(torch.bfloat16).float() * 0.5  # bf16-representable weights
    x = torch.randn((4, 64, d), device=dev).to(torch.bfloat16).float()
    with torch.no_grad():
        ref = model[0](x)
    gate_w = model[0].mlp.gate.weight.detach().clone()
    cfg = MoEConfig(d_model=d, num_experts=E, d_ff=f, top_k=k, activation="swiglu", eq_tokens=8)
    n = replace_moe_layer(model, _Layer, _MoE, "experts", "gate", cfg, device=dev)
    assert n == 2
    with torch.no_grad():
        got = model[0](x)
    _assert_hf_parity(got - x, ref - x, x, gate_w, k, "torch MoE layer")


def _hf_reference_block(block_cls, config, dev):
    torch.manual_seed(3)
    blk = block_cls(config).to(dev)
    for p in blk.parameters():
        nn.init.normal_(p, std=0.05)
        p.data = p.data.to(torch.bfloat16).float()  # bf16-representable weights, fp32 HF math
    return blk


@pytest.mark.parametrize("arch", ["qwen3_moe", "mixtral", "qwen2_moe", "qwen2_moe_hf_default"])
def test_replace_moe_layer_on_transformers_blocks(arch):
    """The paper's drop-in API on the real transformers 5 MoE blocks (fused [E, 2f, d] experts,
    TopK routers): the B200 block reproduces the HF block's own forward within the bf16 bar."""
    dev = _cuda()
    from paper_2506_12417_b200 import MoEConfig, replace_moe_layer

    d, f, E, k = 256, 256, 16, 2 if arch == "mixtral" else 4
    if arch.startswith("qwen2_moe"):  # the paper's Qwen family: routed experts + a gated shared expert
        from transformers.models.qwen2_moe.configuration_qwen2_moe import Qwen2MoeConfig as C
        from transformers.models.qwen2_moe.modeling_qwen2_moe import Qwen2MoeSparseMoeBlock as B

        # "qwen2_moe_hf_default": the config's own default norm_topk_prob (False, as shipped
        # Qwen1.5/2-MoE checkpoints) - the replaced layer must not renormalise the top-k weights
        extra = {} if arch == "qwen2_moe_hf_default" else dict(norm_topk_prob=True)
        conf = C(hidden_size=d, moe_intermediate_size=f, shared_expert_intermediate_size=512, num_experts=E,
                 num_experts_per_tok=k, **extra)
        assert arch != "qwen2_moe_hf_default" or conf.norm_topk_prob is False
    elif arch == "qwen3_moe":
        from transformers.models.qwen3_moe.configuration_qwen3_moe import Qwen3MoeConfig as C
        from transformers.models.qwen3_moe.modeling_qwen3_moe import Qwen3MoeSparseMoeBlock as B

        conf = C(hidden_size=d, moe_intermediate_size=f, num_experts=E, num_experts_per_tok=k, norm_topk_prob=True)
    else:
        from transformers.models.mixtral.configuration_mixtral import MixtralConfig as C
        from transformers.models.mixtral.modeling_mixtral import MixtralSparseMoeBlock as B

        conf = C(hidden_size=d, intermediate_size=f, num_local_experts=E, num_experts_per_tok=k)

    class Parent(nn.Module):
        def __init__(self):
            super().__init__()
            self.mlp = _hf_reference_block(B, conf, dev)

        def forward(self, x):
            return self.mlp(x)

    model = Parent()
    x = torch.randn((2, 96, d), device=dev).to(torch.bfloat16).float()
    with torch.no_grad():
        ref = model(x)
    gate_w = model.mlp.gate.weight.detach().clone()
    # renormalize is taken from the module's norm_topk_prob where it has one (Qwen2/3-MoE)
    cfg = MoEConfig(d_model=d, num_experts=E, d_ff=f, top_k=k, activation="swiglu", eq_tokens=4)
    assert replace_moe_layer(model, Parent, B, "experts", "gate", cfg, device=dev) == 1
    assert model.mlp.block.cfg.renormalize is (arch != "qwen2_moe_hf_default")
    with torch.no_grad():
        got = model(x)
    assert got.shape == ref.shape
    _assert_hf_parity(got, ref, x, gate_w, k, arch)


def test_replace_moe_layer_in_a_transformers_model():
    """replace_moe_layer(model, Qwen3MoeDecoderLayer, Qwen3MoeSparseMoeBlock, "experts", "gate", cfg)
    on a randomly initialised 2-layer Qwen3-MoE causal LM: every MoE layer is
    swapped and the logits stay within the bf16 bar of the original model's."""
    dev = _cuda()
    from transformers.models.qwen3_moe.configuration_qwen3_moe import Qwen3MoeConfig
    from transformers.models.qwen3_moe.modeling_qwen3_moe import (Qwen3MoeDecoderLayer, Qwen3MoeForCausalLM,
                                                                  Qwen3MoeSparseMoeBlock)

    from paper_2506_12417_b200 import MoEConfig, replace_moe_layer

    torch.manual_seed(0)
    conf = Qwen3MoeConfig(vocab_size=512, hidden_size=256, intermediate_size=512, moe_intermediate_size=256,
                          num_hidden_layers=2, num_attention_heads=4, num_key_value_heads=2, head_dim=64,
                          num_experts=16, num_experts_per_tok=4, norm_topk_prob=True, max_position_embeddings=256)
    conf._attn_implementation = "eager"
    model = Qwen3MoeForCausalLM(conf).to(dev).eval()
    for p in model.parameters():
        p.data = p.data.to(torch.bfloat16).float()
    ids = torch.randint(0, 512, (2, 64), device=dev)
    with torch.no_grad():
        ref = model(ids).logits
    cfg = MoEConfig(d_model=256, num_experts=16, d_ff=256, top_k=4, activation="swiglu", eq_tokens=4, renormalize=True)
    assert replace_moe_layer(model, Qwen3MoeDecoderLayer, Qwen3MoeSparseMoeBlock, "experts", "gate", cfg,
                             device=dev) == 2
    with torch.no_grad():
        got = model(ids).logits
    frob = float(torch.linalg.norm(got - ref) / torch.linalg.norm(ref))
    assert frob < 2e-2, f"relative Frobenius error of the logits {frob}"
    assert (got.argmax(-1) == ref.argmax(-1)).float().mean() > 0.95


def test_replace_moe_layer_on_switch_transformers():
    """Switch-128's own module family (SwitchTransformersSparseMLP: top-1 router classifier,
    ModuleDict of ReLU wi/wo experts, weight = the top-1 softmax probability) with the expert
    capacity above the token count (HarMoEny never drops tokens)."""
    dev = _cuda()
    from transformers.models.switch_transformers.configuration_switch_transformers import SwitchTransformersConfig
    from transformers.models.switch_transformers.modeling_switch_transformers import SwitchTransformersSparseMLP

    from paper_2506_12417_b200 import MoEConfig, replace_moe_layer

    d, f, E, T = 256, 512, 16, 192
    conf = SwitchTransformersConfig(d_model=d, d_ff=f, num_experts=E, expert_capacity=T, dropout_rate=0.0)

    class Parent(nn.Module):
        def __init__(self):
            super().__init__()
            self.mlp = _hf_reference_block(SwitchTransformersSparseMLP, conf, dev).eval()

        def forward(self, x):
            return self.mlp(x)

    model = Parent()
    x = torch.randn((1, T, d), device=dev).to(torch.bfloat16).float()
    with torch.no_grad():
        ref = model(x)
    gate_w = model.mlp.router.classifier.weight.detach().clone()
    cfg = MoEConfig(d_model=d, num_experts=E, d_ff=f, top_k=1, activation="relu", eq_tokens=4)
    assert replace_moe_layer(model, Parent, SwitchTransformersSparseMLP, "experts", "router.classifier", cfg,
                             device=dev) == 1
    with torch.no_grad():
        got = model(x)
    _assert_hf_parity(got, ref, x, gate_w, 1, "switch_transformers")
