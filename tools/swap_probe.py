"""Diagnostics: row-major vs swap-AB grouped GEMM on the Switch-128 shapes (Zipf-like ~32-row
experts), each launch alone after an L2 flush, CUDA events (median of 20)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_12417_b200 import ops  # noqa: E402


def main():
    dev = torch.device("cuda")
    E, T = 128, 4096
    p = 1.0 / np.arange(1, E + 1)
    p /= p.sum()
    counts = np.random.default_rng(0).multinomial(T, p)
    sg, rows = [], 0
    mt = [0]
    for e, n in enumerate(counts):
        if n:
            sg.append([rows, int(n), e, e])
            rows += int(n)
            mt.append(mt[-1] + (int(n) + 127) // 128)
    lay = (torch.tensor(sg, dtype=torch.int32, device=dev), torch.tensor([len(sg)], dtype=torch.int32, device=dev),
           torch.tensor(mt, dtype=torch.int32, device=dev))
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device=dev)
    for (N, K, epi) in ((3072, 768, ops.HM_EPI_RELU), (768, 3072, ops.HM_EPI_STORE)):
        A = torch.randn((rows, K), device=dev).to(torch.bfloat16)
        W = (torch.randn((E * N, K), device=dev) * 0.02).to(torch.bfloat16)
        out = torch.empty((rows, N), dtype=torch.bfloat16, device=dev)
        for name, fn in (("row-major", lambda: ops.grouped_gemm(A, W, N, lay, epi, out=out)),
                         ("swap-AB", lambda: ops.grouped_gemm_swap(A, W, N, lay, epi, out=out))):
            ts = []
            for i in range(23):
                flush.fill_(i)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                fn()
                b.record()
                torch.cuda.synchronize()
                if i >= 3:
                    ts.append(a.elapsed_time(b) * 1e3)
            print(f"N={N} K={K} {name}: {np.median(ts):7.1f} us  ({E * N * K * 2 / np.median(ts) / 1e6:5.2f} TB/s of W)")


if __name__ == "__main__":
    main()
