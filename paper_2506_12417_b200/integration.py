"""Integration seams: the paper's model-level API and the reference simulator's
scheduler seam.

* ``replace_moe_layer(model, moe_parent_type, moe_type, path_to_experts,
  path_to_router_linear_layer, config)`` - the listing of PAPER.md:231-258:
  walks a PyTorch model, and every ``moe_type`` submodule found under a
  ``moe_parent_type`` module is replaced by a :class:`HarMoEnyLayer` that runs
  the B200 block with the original router and expert weights.
* ``patch_moesim(moesim_module)`` - drops the GPU scheduler into the reference
  simulator by rebinding ``moesim.engine.build_schedule`` and
  ``moesim.engine.rebalance`` (the names engine.py:40-51 imports; patching
  ``moesim.policies`` alone is not seen by the engine).

Inference only, like HarMoEny (§3: expert-parallel MoE inference).
"""

from __future__ import annotations

import torch
from torch import nn

from .block import HarMoEnyBlock, MoEConfig


def _get_path(module: nn.Module, path: str):
    obj = module
    for part in path.split("."):
        obj = obj[int(part)] if part.isdigit() else getattr(obj, part)
    return obj


_GATE_NAMES = ("gate_proj", "w1", "wi_0", "fc1", "wi")
_UP_NAMES = ("up_proj", "w3", "wi_1")
_DOWN_NAMES = ("down_proj", "w2", "wo", "fc2")


def _linear_weight(expert: nn.Module, names) -> torch.Tensor | None:
    for n in names:
        if hasattr(expert, n):
            lin = getattr(expert, n)
            return lin.weight if isinstance(lin, nn.Module) else lin
    return None


def extract_expert_weights(experts, activation: str, d_model: int | None = None):
    """Stack per-expert weights as [E, out, in] (nn.Linear layout).
    Accepts an nn.ModuleList of expert MLPs with HF names (gate_proj/up_proj/down_proj,
    w1/w3/w2, wi/wo) or a module holding fused 3-D parameters ``gate_up_proj`` /
    ``down_proj``, either in the per-expert nn.Linear layout ([E, 2f, d] / [E, d, f]:
    transformers 5 ``Qwen3MoeExperts``, ``MixtralExperts``, ``OlmoeExperts``; gate rows first)
    or transposed ([E, d, 2f] / [E, f, d]).  ``d_model`` (the router's input width, or the
    module's ``hidden_dim``) tells the two apart when 2f == d would make the shapes ambiguous."""
    if hasattr(experts, "gate_up_proj") and hasattr(experts, "down_proj") and not isinstance(experts, nn.ModuleList):
        gu = experts.gate_up_proj.detach()
        dn = experts.down_proj.detach()
        d = getattr(experts, "hidden_dim", None) or d_model
        if d is None:
            raise ValueError("fused expert weights: pass d_model to tell [E, 2f, d] from [E, d, 2f]")
        if gu.shape[-1] == d and dn.shape[-2] == d:  # [E, 2f, d] and [E, d, f]: nn.Linear layout
            f = gu.shape[-2] // 2
            return gu[:, :f].contiguous(), dn.contiguous(), gu[:, f:].contiguous()
        if gu.shape[-2] == d and dn.shape[-1] == d:  # [E, d, 2f] and [E, f, d]: transposed
            f = gu.shape[-1] // 2
            w1 = gu[..., :f].transpose(1, 2).contiguous()
            w3 = gu[..., f:].transpose(1, 2).contiguous()
            return w1, dn.transpose(1, 2).contiguous(), w3
        raise ValueError(f"fused expert weights {tuple(gu.shape)} / {tuple(dn.shape)} do not match d_model={d}")
    mods = list(experts.values()) if isinstance(experts, nn.ModuleDict) else list(experts)  # expert_0, expert_1, ...
    w1 = torch.stack([_linear_weight(e, _GATE_NAMES).detach() for e in mods])
    w2 = torch.stack([_linear_weight(e, _DOWN_NAMES).detach() for e in mods])
    w3 = None
    if activation == "swiglu":
        w3 = torch.stack([_linear_weight(e, _UP_NAMES).detach() for e in mods])
    return w1, w2, w3


class HarMoEnyLayer(nn.Module):
    """nn.Module wrapper: hidden [..., d] -> MoE(hidden) through the B200 block.

    ``shared_expert`` / ``shared_expert_gate`` (the always-on dense expert of Qwen1.5/2-MoE,
    the paper's Qwen model): y += sigmoid(gate(x)) * shared(x), a plain dense MLP outside the
    routed path, run by the original module (cuBLAS) beside the routed experts."""

    def __init__(self, block, returns_router_logits: bool = False, shared_expert: nn.Module | None = None,
                 shared_expert_gate: nn.Module | None = None):
        super().__init__()
        self.block = block
        self.returns_router_logits = returns_router_logits
        self.shared_expert = shared_expert
        self.shared_expert_gate = shared_expert_gate

    @torch.no_grad()
    def forward(self, hidden_states: torch.Tensor, *args, **kwargs):
        shape = hidden_states.shape
        x = hidden_states.reshape(-1, shape[-1]).to(torch.bfloat16).contiguous()
        y = self.block(x).reshape(shape).to(hidden_states.dtype)
        if self.shared_expert is not None:
            s = self.shared_expert(hidden_states)
            if self.shared_expert_gate is not None:
                s = torch.sigmoid(self.shared_expert_gate(hidden_states)) * s
            y = y + s
        if self.returns_router_logits:
            return y, None
        return y


def _routing_config(moe_module: nn.Module, router, config: MoEConfig) -> MoEConfig:
    """Take the routing semantics from the module being replaced: ``norm_topk_prob`` (HF
    Qwen2/Qwen3-MoE routers; shipped Qwen1.5/2-MoE checkpoints use False) sets
    ``renormalize``, and a module ``top_k`` / ``num_experts_per_tok`` that disagrees with the
    config is an error rather than a silent change of the routing."""
    import dataclasses

    for obj in (router, moe_module):
        k = getattr(obj, "top_k", None) or getattr(obj, "num_experts_per_tok", None)
        if isinstance(k, int) and k != config.top_k:
            raise ValueError(f"MoEConfig.top_k={config.top_k} but the replaced module routes top-{k}")
    for obj in (router, moe_module):
        ntp = getattr(obj, "norm_topk_prob", None)
        if isinstance(ntp, bool):
            if ntp != config.renormalize:
                config = dataclasses.replace(config, renormalize=ntp)
            break
    return config


def build_block(moe_module: nn.Module, path_to_experts: str, path_to_router_linear_layer: str, config: MoEConfig,
                device=None):
    experts = _get_path(moe_module, path_to_experts)
    router = _get_path(moe_module, path_to_router_linear_layer)
    config = _routing_config(moe_module, router, config)
    wg = router.weight.detach() if isinstance(router, nn.Module) else router.detach()
    w1, w2, w3 = extract_expert_weights(experts, config.activation, d_model=wg.shape[-1])
    if config.world_size > 1:
        from .ep import EPHarMoEnyBlock

        return EPHarMoEnyBlock(config, wg, w1, w2, w3, device=device)
    return HarMoEnyBlock(config, wg, w1, w2, w3, device=device)


def replace_moe_layer(model: nn.Module, moe_parent_type, moe_type, path_to_experts: str,
                      path_to_router_linear_layer: str, config: MoEConfig, device=None,
                      returns_router_logits: bool = False) -> int:
    """PAPER.md:249-256.  Returns the number of layers replaced."""
    replaced = 0
    for parent in list(model.modules()):
        if not isinstance(parent, moe_parent_type):
            continue
        for name, child in list(parent.named_children()):
            if isinstance(child, moe_type):
                blk = build_block(child, path_to_experts, path_to_router_linear_layer, config, device=device)
                setattr(parent, name, HarMoEnyLayer(blk, returns_router_logits,
                                                    shared_expert=getattr(child, "shared_expert", None),
                                                    shared_expert_gate=getattr(child, "shared_expert_gate", None)))
                replaced += 1
    return replaced


def patch_moesim(moesim_module=None):
    """Rebind the reference simulator's scheduler seam to the GPU kernels.

    ``moesim.engine.simulate_layer`` calls ``build_schedule`` (engine.py:334),
    which calls ``rebalance`` (engine.py:298); both names are module globals of
    ``moesim.engine``.  Returns a callable that restores the originals."""
    import numpy as np

    if moesim_module is None:
        import moesim as moesim_module  # noqa: F811
    eng = moesim_module.engine
    ref_core = moesim_module.core
    from . import policies

    orig = (eng.build_schedule, eng.rebalance, eng.even_split_assign, eng.affinity_placement)

    def rebalance(s_initial, q):
        s, _ = policies.rebalance_with_stats(s_initial, q)
        return ref_core.ScheduleTensor(np.asarray(s.counts))

    def even_split_assign(m_all, num_gpus):
        return ref_core.ScheduleTensor(np.asarray(policies.even_split_assign(m_all, num_gpus).counts))

    def affinity_placement(profile, num_gpus, slots):
        p = policies.affinity_placement(policies.PopularityProfile(counts=profile.counts,
                                                                   window_batches=profile.window_batches),
                                        num_gpus, slots)
        return ref_core.Placement(home=p.home, num_gpus=p.num_gpus)

    def build_schedule(m_all, placement, config, flags):
        from . import ops
        from .policies import _to_i32

        if config.policy is moesim_module.SchedulingPolicy.EVEN_SPLIT:  # engine.py:292-293 (placement unused)
            policy, home = ops.HM_POLICY_EVEN_SPLIT, np.zeros(m_all.num_experts, np.int64)
        else:
            # the reference's initial_assign check (policies.py:111-112): never hand the kernel
            # a home vector of the wrong length or with ranks outside the routing matrix
            if placement.num_experts != m_all.num_experts or placement.num_gpus != m_all.num_gpus:
                raise ValueError("placement dimensions do not match routing matrix")
            home = np.asarray(placement.home, np.int64)
            do_rb = config.policy is moesim_module.SchedulingPolicy.REBALANCE and flags.rebalancing_enabled
            policy = ops.HM_POLICY_REBALANCE if do_rb else ops.HM_POLICY_NONE
        S, _, _ = ops.schedule(_to_i32(m_all.counts, "build_schedule"), _to_i32(home, "home"),
                               config.token_threshold_q, rebalance=policy)
        return ref_core.ScheduleTensor(S.cpu().numpy().astype(np.int64))

    eng.build_schedule, eng.rebalance = build_schedule, rebalance
    eng.even_split_assign, eng.affinity_placement = even_split_assign, affinity_placement

    def restore():
        eng.build_schedule, eng.rebalance, eng.even_split_assign, eng.affinity_placement = orig

    return restore
