"""Per-tile phase timeline of the router kernel (diagnostics build with -DHM_ROUTER_STAMPS:
bash tools/build_variant.sh stamps -DHM_ROUTER_STAMPS; HM_LIB_PATH=.../libharmoe_stamps.so).
Phases (ns from the earliest CTA start): 0 start, 1 first stage landed, 7 last MMA issued,
2 accumulator ready, 3 per-part top-k done, 4 merge + outputs done, 5 rank pass done, 6 end."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_12417_b200 import _lib, ops  # noqa: E402


def main():
    lib = _lib.load()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device="cuda")
    for (T, d, E, k) in [(16384, 2048, 128, 8), (2048, 2048, 128, 8), (4096, 768, 128, 1), (16384, 4096, 8, 2)]:
        x = torch.randn((T, d), device="cuda").to(torch.bfloat16)
        wg = (torch.randn((ops.e_pad(E), d), device="cuda") * 0.02).to(torch.bfloat16)
        nt = (T + 127) // 128
        for cold in (True, False):
            stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
            for _ in range(3):
                if cold:
                    flush.fill_(1)
                lib.hm_debug_stamp(0, stream)
                ops.router_topk(x, wg, None, 1, T, k, k > 1, E=E)
                lib.hm_debug_stamp(1, stream)
            torch.cuda.synchronize()
            gap = np.zeros((4096, 8), dtype=np.uint64)
            assert lib.hm_debug_router_stamps(gap.ctypes.data_as(ctypes.c_void_p), 4096) == 0
            pre, post = int(gap[4095, 0]), int(gap[4095, 1])
            st = np.zeros((nt, 8), dtype=np.uint64)
            assert lib.hm_debug_router_stamps(st.ctypes.data_as(ctypes.c_void_p), nt) == 0
            st = st.astype(np.int64)
            t0 = st[:, 0].min()
            rel = (st - t0) / 1000.0
            names = ["start", "stage0", "lastmma", "acc", "part", "merge", "rank", "end"]
            order = [0, 1, 7, 2, 3, 4, 5, 6]
            med = np.median(rel[:, order], axis=0)
            mx = rel[:, order].max(axis=0)
            print(f"   stamp kernel before -> first CTA start {(t0 - pre) / 1e3:.1f} us; last epilogue stamp -> "
                  f"stamp kernel after {(post - st[:, 5].max()) / 1e3:.1f} us; whole {(post - pre) / 1e3:.1f} us")
            print(f"T={T} d={d} E={E} k={k} {'cold' if cold else 'warm'}: span {rel[:, 6].max():.1f} us; "
                  "median/max per phase (us): " + ", ".join(f"{names[i]} {a:.1f}/{b:.1f}" for i, a, b in
                                                             zip(range(8), med, mx)), flush=True)


if __name__ == "__main__":
    main()
