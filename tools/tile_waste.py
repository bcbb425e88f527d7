"""Diagnostics: expert row counts of the bench workload and grouped-GEMM tile padding."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_12417_b200.block import HarMoEnyBlock, MoEConfig  # noqa: E402

for s in (0.0, 0.5, 1.0, 1.5):
    cfg = MoEConfig(d_model=2048, d_ff=768, num_experts=128, top_k=8, eq_tokens=32)
    blk = HarMoEnyBlock.random(cfg, seed=0, zipf_s=s)
    g = torch.Generator(device="cuda").manual_seed(1234)
    x = torch.randn((16384, 2048), device="cuda", generator=g).to(torch.bfloat16)
    blk(x)
    n = blk.stats.m_all.cpu().numpy().sum(axis=0)
    for tm in (128, 256):
        pad = int((np.ceil(n / tm) * tm).sum())
        print(f"s={s}: rows {n.sum()} max {n.max()} min {n.min()} | tile {tm}: padded {pad} (+{100 * (pad / n.sum() - 1):.1f}%)")
