"""Context for the headline number: the same Qwen-128 MoE layer (d 2048, expert d_ff 768, 128
experts, top-8, 16,384 tokens, bf16) through (a) this repo's block, (b) transformers 5's
Qwen3MoeSparseMoeBlock (eager per-expert loop) and (c) vLLM's Triton fused_experts with a torch
router.  Diagnostics only (not a bench value); CUDA-event device time per forward.

    python tools/compare_libs.py [qwen128|mixtral8] [tokens]
"""

import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_12417_b200.block import HarMoEnyBlock, MoEConfig  # noqa: E402


def timed(fn, it=10, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(it):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / it


def main():
    shape = sys.argv[1] if len(sys.argv) > 1 else "qwen128"
    d, f, E, k, T = {"qwen128": (2048, 768, 128, 8, 16384), "mixtral8": (4096, 14336, 8, 2, 16384)}[shape]
    if len(sys.argv) > 2:  # token count override (e.g. small decode-like batches)
        T = int(sys.argv[2])
    dev = torch.device("cuda")
    cfg = MoEConfig(d_model=d, d_ff=f, num_experts=E, top_k=k, eq_tokens=32, renormalize=True)
    print(f"{shape}: d {d}, d_ff {f}, {E} experts, top-{k}, {T} tokens")
    blk = HarMoEnyBlock.random(cfg, seed=0, zipf_s=1.0)
    x = torch.randn((T, d), device=dev).to(torch.bfloat16)
    cap = blk.capture(T, groups=(("router", "schedule", "permute", "gemm1", "gemm2", "combine"),))  # one graph
    cap.x.copy_(x)
    ours = timed(lambda: cap.replay())
    print(f"this repo (graph replay)         : {ours:8.3f} ms  {T / ours / 1e3:8.2f} M tok/s", flush=True)

    # the same weights in the HF / vLLM layouts: gate_up [E, 2f, d] (gate rows first), down [E, d, f]
    E_, f2 = E, 2 * f
    w13 = blk.w_in.view(E_, f // 128, 2, 128, d)
    gate = w13[:, :, 0].reshape(E_, f, d)
    up = w13[:, :, 1].reshape(E_, f, d)
    gate_up = torch.cat([gate, up], dim=1).contiguous()  # [E, 2f, d]
    down = blk.w_out.view(E_, d, f).contiguous()
    wg = blk.wg[:E]
    bias = blk.bias.float()

    try:
        from vllm.model_executor.layers.fused_moe.fused_moe import fused_experts

        def vllm_fwd():
            logits = torch.matmul(x, wg.t()).float() + bias
            p = torch.softmax(logits, dim=-1)
            w, ids = torch.topk(p, k, dim=-1)
            w = w / w.sum(-1, keepdim=True)
            return fused_experts(x, gate_up, down, w, ids.to(torch.int32))

        t = timed(vllm_fwd)
        print(f"vLLM fused_experts (Triton)      : {t:8.3f} ms  {T / t / 1e3:8.2f} M tok/s", flush=True)
    except Exception as e:  # noqa: BLE001
        print(f"vLLM fused_experts unavailable: {type(e).__name__}: {e}"[:300], flush=True)

    try:  # FlashInfer's ahead-of-time built CUTLASS fused MoE for SM100 (the TensorRT-LLM kernels)
        from flashinfer.fused_moe import cutlass_fused_moe

        def fi_fwd():
            logits = torch.matmul(x, wg.t()).float() + bias
            p = torch.softmax(logits, dim=-1)
            w, ids = torch.topk(p, k, dim=-1)
            w = w / w.sum(-1, keepdim=True)
            # timing only: the gate/up half order follows TensorRT-LLM's convention, not checked here
            return cutlass_fused_moe(x, ids.to(torch.int32), w, gate_up, down, torch.bfloat16, quant_scales=[])

        t = timed(fi_fwd)
        print(f"FlashInfer cutlass_fused_moe (SM100 AOT): {t:8.3f} ms  {T / t / 1e3:8.2f} M tok/s", flush=True)
    except Exception as e:  # noqa: BLE001
        print(f"FlashInfer cutlass_fused_moe unavailable: {type(e).__name__}: {e}"[:300], flush=True)

    if shape != "qwen128" or T != 16384:
        return
    try:
        from transformers.models.qwen3_moe.configuration_qwen3_moe import Qwen3MoeConfig
        from transformers.models.qwen3_moe.modeling_qwen3_moe import Qwen3MoeSparseMoeBlock

        hf = Qwen3MoeSparseMoeBlock(Qwen3MoeConfig(hidden_size=d, moe_intermediate_size=f, num_experts=E,
                                                   num_experts_per_tok=k, norm_topk_prob=True)).to(dev)
        hf = hf.to(torch.bfloat16)
        with torch.no_grad():
            hf.gate.weight.copy_(wg)
            hf.experts.gate_up_proj.copy_(gate_up)
            hf.experts.down_proj.copy_(down)
        xh = x.view(1, T, d)
        with torch.no_grad():
            t = timed(lambda: hf(xh), it=3, warm=1)
        print(f"transformers Qwen3MoeSparseMoeBlock: {t:8.3f} ms  {T / t / 1e3:8.2f} M tok/s", flush=True)
    except Exception as e:  # noqa: BLE001
        print(f"transformers block unavailable: {type(e).__name__}: {e}"[:300], flush=True)


if __name__ == "__main__":
    main()
