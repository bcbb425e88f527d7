"""Router kernel device time (graph replay) with the L2 flushed before every call (CUDA events),
for the default one-CTA-per-tile kernel and the split-K cluster experiment (HM_ROUTER_V2=1,
HM_ROUTER_C / HM_ROUTER_STAGES to sweep it)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_12417_b200 import ops  # noqa: E402


def main():
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device="cuda")
    clean = torch.ones(256 * 1024 * 1024 // 4, dtype=torch.int32, device="cuda")
    mode = os.environ.get("FLUSH", "write+read")
    for (T, d, E, k) in [(16384, 2048, 128, 8), (2048, 2048, 128, 8), (4096, 768, 128, 1), (1024, 768, 128, 1),
                         (16384, 4096, 8, 2), (2048, 4096, 8, 2)]:
        x = torch.randn((T, d), device="cuda").to(torch.bfloat16)
        wg = (torch.randn((ops.e_pad(E), d), device="cuda") * 0.02).to(torch.bfloat16)
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            for _ in range(3):
                ops.router_topk(x, wg, None, 1, T, k, k > 1, E=E)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()  # graph replay: no host launch work inside the timed region
        with torch.cuda.graph(g):
            ops.router_topk(x, wg, None, 1, T, k, k > 1, E=E)
        ts = []
        for i in range(20):
            flush.fill_(i)
            if mode == "write+read":  # write back the fill's dirty lines before the timed call
                clean.sum()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            g.replay()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) * 1e3)
        ts.sort()
        med = ts[len(ts) // 2]
        print(f"{'v2' if os.environ.get('HM_ROUTER_V2', '0') == '1' else 'v1'} T={T:6d} d={d} E={E} k={k}: "
              f"{med:7.1f} us cold ({mode})  ({T * d * 2 / med / 1e3:7.1f} GB/s of x)", flush=True)


if __name__ == "__main__":
    main()
