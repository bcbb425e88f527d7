"""Co-residency probe (diagnostics): can the HBM-bound combine run beside the persistent,
tensor-bound FFN2 GEMM?  Times FFN2 alone, the combine alone, and both launched together on two
streams (the combine reads a second block's buffers, so there is no data dependence).  If the pair
takes ~max(FFN2, combine), a token-chunked FFN2 (rows of the first half of the tokens first) could
hide the first half's combine under the second half's GEMM."""

import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_12417_b200.block import HarMoEnyBlock, MoEConfig  # noqa: E402


def main():
    T = 16384
    cfg = MoEConfig(d_model=2048, d_ff=768, num_experts=128, top_k=8, activation="swiglu", eq_tokens=32)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    blocks, stages = [], []
    for i, s in enumerate((s1, s2)):
        blk = HarMoEnyBlock.random(cfg, seed=i, device="cuda", zipf_s=1.0)
        st = {"x": torch.randn((T, 2048), device="cuda").to(torch.bfloat16)}
        with torch.cuda.stream(s):
            sg = dict(blk._stages(st, 1, T, s))
            for name in ("router", "schedule", "permute", "gemm1", "gemm2", "combine"):
                if name in sg:
                    sg[name]()
        torch.cuda.synchronize()
        blocks.append(blk)
        stages.append(sg)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device="cuda")

    def timed(fn, n=10):
        ts = []
        for i in range(n):
            flush.fill_(i)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s1)
            s2.wait_stream(s1)
            fn()
            s1.wait_stream(s2)
            b.record(s1)
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) * 1e3)
        return float(np.median(ts[2:]))

    g2 = lambda: stages[0]["gemm2"]()  # noqa: E731  (on s1)
    cb = lambda: stages[1]["combine"]()  # noqa: E731  (on s2)
    for _ in range(2):
        a = timed(g2)
        b = timed(cb)
        c = timed(lambda: (g2(), cb()))
        print(f"FFN2 alone {a:.1f} us, combine alone {b:.1f} us, both on two streams {c:.1f} us "
              f"(serial would be {a + b:.1f}, perfect overlap {max(a, b):.1f})", flush=True)


if __name__ == "__main__":
    main()
