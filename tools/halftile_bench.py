"""Microbenchmark: cost of an M=128 cta_group::2 "half" pair tile vs a full M=256 one.

Same total rows (131,072) and FFN1 shape (N 1536, K 2048, SwiGLU), cut into 256-row
segments (full tiles only) or 128-row segments (every tile a half tile).  Run with and
without HM_GEMM_NO_HALF=1 to see what the half-tile MMA saves over padding.

    python tools/halftile_bench.py
"""

import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_12417_b200 import ops  # noqa: E402
from tools.gemm_bench import timeit  # noqa: E402


def main():
    dev = torch.device("cuda")
    N, K, E = 1536, 2048, 128
    W = (torch.randn((E * N, K), device=dev) * 0.02).to(torch.bfloat16)
    total = 131072
    A = torch.randn((total, K), device=dev).to(torch.bfloat16)
    for seg_rows in (256, 128, 64):
        n = total // seg_rows
        sg = [[i * seg_rows, seg_rows, i % E, i % E] for i in range(n)]
        mt = [0]
        for _ in range(n):
            mt.append(mt[-1] + (seg_rows + 127) // 128)
        lay = (torch.tensor(sg, dtype=torch.int32, device=dev), torch.tensor([n], dtype=torch.int32, device=dev),
               torch.tensor(mt, dtype=torch.int32, device=dev))
        out = ops.grouped_gemm(A, W, N, lay, ops.HM_EPI_SWIGLU)
        t = timeit(lambda: ops.grouped_gemm(A, W, N, lay, ops.HM_EPI_SWIGLU, out=out), iters=20)
        fl = 2.0 * total * N * K
        print(f"half={os.environ.get('HM_GEMM_NO_HALF', '0') != '1'} seg_rows={seg_rows}: {t:8.1f} us "
              f"{fl / t / 1e6:7.1f} TF/s (algorithmic)", flush=True)


if __name__ == "__main__":
    main()
