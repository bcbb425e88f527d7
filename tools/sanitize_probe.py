"""Small eager forwards of every hot-path kernel for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck):  bash tools/sanitize.sh  (diagnostics, run on the GPU box)."""

import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_12417_b200.block import HarMoEnyBlock, MoEConfig  # noqa: E402


def main():
    dev = torch.device("cuda")
    for kw in (dict(top_k=4, activation="swiglu", logical_ranks=2),  # fused gather FFN1
               dict(top_k=2, activation="swiglu", logical_ranks=1),  # copy-permute + TMA FFN1
               dict(top_k=1, activation="relu", logical_ranks=4)):
        cfg = MoEConfig(d_model=256, num_experts=16, d_ff=256, eq_tokens=2, placement="blocked", **kw)
        blk = HarMoEnyBlock.random(cfg, seed=1, device=dev, zipf_s=1.2, std=0.05)
        x = torch.randn((400, 256), device=dev).to(torch.bfloat16)
        y = blk(x)
        torch.cuda.synchronize()
        print(kw, "ok", float(y.float().abs().sum()))


if __name__ == "__main__":
    main()
