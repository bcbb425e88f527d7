# needs a diagnostics build: bash tools/build_variant.sh phases -DHM_PLAN_PHASES; HM_LIB_PATH=paper_2506_12417_b200/libharmoe_phases.so
"""Diagnostics: phase timing inside the fused planner (hm_debug_plan_phases)."""

import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_12417_b200 import _lib  # noqa: E402
from paper_2506_12417_b200.block import HarMoEnyBlock, MoEConfig  # noqa: E402


def main():
    for G in (1, 8):
        cfg = MoEConfig(d_model=2048, d_ff=768, num_experts=128, top_k=8, logical_ranks=G, eq_tokens=32,
                        placement="blocked")
        blk = HarMoEnyBlock.random(cfg, seed=0, zipf_s=1.0)
        x = torch.randn((16384, 2048), device="cuda").to(torch.bfloat16)
        for _ in range(3):
            blk(x)
        torch.cuda.synchronize()
        buf = (ctypes.c_longlong * 8)()
        _lib.check(_lib.load().hm_debug_plan_phases(buf), "phases")
        t = list(buf)
        sub = (f" [head {(t[4] - t[2]) / 1e3:.1f}, slots+segs {(t[5] - t[4]) / 1e3:.1f}, "
               f"scan {(t[6] - t[5]) / 1e3:.1f}]") if G > 1 else " (single-GPU planner)"
        print(f"G={G}: hist {(t[1] - t[0]) / 1e3:.1f} us, schedule {(t[2] - t[1]) / 1e3:.1f} us, "
              f"layout {(t[3] - t[2]) / 1e3:.1f} us{sub}, iters {int(blk.stats.iters.item())}")


if __name__ == "__main__":
    main()
