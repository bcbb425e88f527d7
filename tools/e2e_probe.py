"""Diagnostics for the end-to-end path: compute alone, PCIe alone, and the pipeline (per step)."""

import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_12417_b200.block import HarMoEnyBlock, MoEConfig  # noqa: E402


def timed(fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


def main():
    T = 16384
    cfg = MoEConfig(d_model=2048, d_ff=768, num_experts=128, top_k=8, eq_tokens=32)
    blk = HarMoEnyBlock.random(cfg, seed=0, zipf_s=1.0)
    x = torch.randn((T, 2048), device="cuda").to(torch.bfloat16)
    xh = x.cpu().pin_memory()
    yh = torch.empty_like(xh).pin_memory()
    cap = blk.capture(T)
    cap.x.copy_(x)
    print(f"compute (graph replay): {timed(lambda: cap.replay()):.3f} ms")
    xd = torch.empty_like(x)
    yd = torch.empty_like(x)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def pcie():
        with torch.cuda.stream(s1):
            xd.copy_(xh, non_blocking=True)
        with torch.cuda.stream(s2):
            yh.copy_(yd, non_blocking=True)
        torch.cuda.current_stream().wait_stream(s1)
        torch.cuda.current_stream().wait_stream(s2)

    print(f"H2D 64 MB || D2H 64 MB: {timed(pcie):.3f} ms")
    for chunks in (1, 2, 4):
        for sets in (2, 3):
            from paper_2506_12417_b200.block import HostPipeline

            pipe = HostPipeline(blk, T, chunks, n_sets=sets)
            print(f"pipeline chunks={chunks} sets={sets}: {timed(lambda: pipe.run(xh, yh)):.3f} ms/step")
            del pipe
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
