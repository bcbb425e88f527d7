"""Microbenchmark of the router kernel over token counts / widths (diagnostics)."""

import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_12417_b200 import ops  # noqa: E402


def t_us(fn, it=20):
    """Device time per call: the calls are captured into one CUDA graph (no host overhead)."""
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(3):
            fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(it):
            fn()
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / it * 1e3


def main():
    for (T, d, E, k) in [(16384, 2048, 128, 8), (8192, 2048, 128, 8), (4096, 2048, 128, 8), (2048, 2048, 128, 8),
                         (16384, 2048, 128, 1), (16384, 2048, 16, 1), (16384, 2048, 16, 8), (16384, 512, 128, 8),
                         (4096, 768, 128, 1), (16384, 4096, 8, 2)]:
        x = torch.randn((T, d), device="cuda").to(torch.bfloat16)
        wg = (torch.randn((ops.e_pad(E), d), device="cuda") * 0.02).to(torch.bfloat16)
        us = t_us(lambda: ops.router_topk(x, wg, None, 1, T, k, k > 1, E=E))
        print(f"T={T:6d} d={d} E={E} k={k}: {us:7.1f} us  ({T * d * 2 / us / 1e3:7.1f} GB/s of x)")


if __name__ == "__main__":
    main()
