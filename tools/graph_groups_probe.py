"""Diagnostics: step time of the captured forward as 4 stage graphs (bench default) vs one graph."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_12417_b200.block import HarMoEnyBlock, MoEConfig  # noqa: E402


def t(fn, flush, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for i in range(n):
        flush.fill_(i)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return float(np.median(ts)), float(np.mean(ts))


def main():
    for wl, kw, T in (("qwen128", dict(d_model=2048, d_ff=768, num_experts=128, top_k=8), 16384),
                      ("switch128", dict(d_model=768, d_ff=3072, num_experts=128, top_k=1, activation="relu",
                                         logical_ranks=4, eq_tokens=4), 4096)):
        cfg = MoEConfig(**kw)
        blk = HarMoEnyBlock.random(cfg, seed=0, zipf_s=1.0)
        x = torch.randn((T, cfg.d_model), device="cuda").to(torch.bfloat16)
        flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device="cuda")
        grouped = blk.capture(T)
        grouped.x.copy_(x)
        one = blk.capture(T, groups=(("router", "schedule", "permute", "gemm1", "gemm2", "combine"),))
        one.x.copy_(x)
        print(wl, "grouped (median, mean us)", t(lambda: grouped.replay(), flush), "one graph", t(lambda: one.replay(), flush),
              flush=True)


if __name__ == "__main__":
    main()
