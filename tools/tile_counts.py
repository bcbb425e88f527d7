"""Pair-tile totals of the bench workloads' grouped GEMMs vs the resident pair count (diagnostics:
does the last wave run half empty?)."""
import sys, torch
sys.path.insert(0, '.')
from paper_2506_12417_b200 import ops
from paper_2506_12417_b200.block import HarMoEnyBlock, MoEConfig
from paper_2506_12417_b200 import _lib
P = _lib.load().hm_gemm_resident_pairs(0, 0)
for (name, d, f, E, k, act, T, G, q) in (("switch128", 768, 3072, 128, 1, "relu", 4096, 4, 4),
                                          ("qwen128", 2048, 768, 128, 8, "swiglu", 16384, 1, 32),
                                          ("mixtral8", 4096, 14336, 8, 2, "swiglu", 16384, 1, 32),
                                          ("mixtral8_4k", 4096, 14336, 8, 2, "swiglu", 4096, 1, 32)):
    cfg = MoEConfig(d_model=d, d_ff=f, num_experts=E, top_k=k, activation=act, logical_ranks=G, eq_tokens=q)
    blk = HarMoEnyBlock.random(cfg, seed=0, zipf_s=1.0)
    x = torch.randn((T, d), device="cuda").to(torch.bfloat16)
    blk(x); torch.cuda.synchronize()
    lay = blk.stats.extras["layout"]
    ns = int(lay.n_seg.item()); mp = lay.mtile_prefix[:ns + 1].cpu()
    pt = int((((mp[1:] - mp[:-1]) + 1) // 2).sum())
    n_in = 2 * f if act == "swiglu" else f
    for g, N in (("ffn1", n_in), ("ffn2", d)):
        tot = pt * (N // 256)
        print(f"{name} {g}: {tot} pair tiles on {P} pairs = {tot / P:.2f} waves, last wave {tot % P}", flush=True)
    del blk
