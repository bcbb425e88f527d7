"""Microbenchmark: FFN2-shaped grouped GEMM variants (diagnosis of the FFN2 efficiency gap).

    python tools/ffn2_bench.py
"""

import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_12417_b200 import ops  # noqa: E402
from tools.gemm_bench import segs, timeit  # noqa: E402


def run(rows_total, N, K, E, epi, row_map=False, label=""):
    dev = torch.device("cuda")
    lay, rows = segs([rows_total // E] * E, dev)
    A = torch.randn((rows, K), device=dev).to(torch.bfloat16)
    W = (torch.randn((E * N, K), device=dev) * 0.02).to(torch.bfloat16)
    rm = torch.randperm(rows, device=dev).to(torch.int32) if row_map else None
    out = ops.grouped_gemm(A, W, N, lay, epi, row_map=rm)
    t = timeit(lambda: ops.grouped_gemm(A, W, N, lay, epi, out=out, row_map=rm), iters=30)
    fl = 2.0 * rows * N * K
    print(f"{label:28s} rows={rows} N={N} K={K} E={E}: {t:8.1f} us {fl / t / 1e6:7.1f} TF/s", flush=True)


def main():
    run(131072, 2048, 768, 128, ops.HM_EPI_STORE, label="ffn2 uniform")
    run(131072, 2048, 768, 128, ops.HM_EPI_STORE, row_map=True, label="ffn2 uniform + row_map")
    run(131072, 2048, 768, 8, ops.HM_EPI_STORE, label="ffn2 8 experts")
    run(131072, 2048, 1536, 128, ops.HM_EPI_STORE, label="ffn2 K x2")
    run(131072, 1024, 768, 128, ops.HM_EPI_STORE, label="ffn2 N/2")
    run(131072, 1536, 2048, 128, ops.HM_EPI_SWIGLU, label="ffn1 uniform")
    run(131072, 1536, 2048, 128, ops.HM_EPI_STORE, label="ffn1 store epi")


if __name__ == "__main__":
    main()
