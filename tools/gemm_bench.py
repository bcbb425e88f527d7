"""Microbenchmark: hm_grouped_gemm vs cuBLAS (torch.matmul) on dense and grouped shapes.

    python tools/gemm_bench.py
"""

import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_12417_b200 import ops  # noqa: E402


def timeit(fn, iters=20, warm=5):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters * 1e3  # us


def segs(counts, dev):
    rows, mt, sg = 0, [0], []
    for e, n in enumerate(counts):
        if n:
            sg.append([rows, n, e, e])
            rows += n
            mt.append(mt[-1] + (n + 127) // 128)
    return (torch.tensor(sg, dtype=torch.int32, device=dev), torch.tensor([len(sg)], dtype=torch.int32, device=dev),
            torch.tensor(mt, dtype=torch.int32, device=dev)), rows


def main():
    dev = torch.device("cuda")
    for (M, N, K, E, epi) in [(16384, 1536, 2048, 1, "store"), (131072, 1536, 2048, 128, "swiglu"),
                              (131072, 2048, 768, 128, "store"), (8192, 8192, 8192, 1, "store")]:
        counts = [M // E] * E
        lay, rows = segs(counts, dev)
        A = torch.randn((rows, K), device=dev).to(torch.bfloat16)
        W = (torch.randn((E * N, K), device=dev) * 0.02).to(torch.bfloat16)
        code = ops.HM_EPI_SWIGLU if epi == "swiglu" else ops.HM_EPI_STORE
        out = ops.grouped_gemm(A, W, N, lay, code)
        t_hm = timeit(lambda: ops.grouped_gemm(A, W, N, lay, code, out=out))
        flops = 2.0 * rows * N * K
        Wd = W[:N]
        t_cb = timeit(lambda: torch.matmul(A[: rows // E], Wd.T)) * E if E <= 8 else float("nan")
        print(f"M={M} N={N} K={K} E={E} {epi}: hm {t_hm:8.1f} us {flops / t_hm / 1e6:7.1f} TF/s"
              f" | cuBLAS(per-expert x E) {t_cb:8.1f} us {flops / t_cb / 1e6:7.1f} TF/s")


if __name__ == "__main__":
    main()
