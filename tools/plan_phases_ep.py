# needs a diagnostics build: bash tools/build_variant.sh phases -DHM_PLAN_PHASES; HM_LIB_PATH=paper_2506_12417_b200/libharmoe_phases.so
"""Diagnostics: phase timing inside the fused planner for one EP rank (HM_LAYOUT_EP_EXPERT,
the p2p transport's layout) at G=8 on the C2 shape, round-robin and blocked placement."""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_12417_b200 import _lib, ops  # noqa: E402
from paper_2506_12417_b200.block import MoEConfig, placement_home, random_weights  # noqa: E402


def main():
    d, E, k, T, G = 2048, 128, 8, 16384, 8
    for placement in ("round_robin", "blocked"):
        cfg = MoEConfig(d_model=d, d_ff=768, num_experts=E, top_k=k, eq_tokens=32, placement=placement,
                        logical_ranks=G)
        wg, _, _, _, bias = random_weights(cfg, 0, torch.device("cuda"), 1.0)
        wgp = torch.zeros((ops.e_pad(E), d), dtype=torch.bfloat16, device="cuda")
        wgp[:E] = wg
        x = torch.randn((T, d), device="cuda").to(torch.bfloat16)
        Tg = T // G
        _, _, tile_hist, _ = ops.router_topk(x, wgp, bias, G, Tg, k, True, E=E)
        m_all, _ = ops.hist_scan(tile_hist, G, (Tg + 127) // 128)
        home = torch.from_numpy(placement_home(cfg)).to("cuda")
        for me in (0, 3, 6):
            for _ in range(3):
                p = ops.plan(home, G, E, 32, ops.HM_POLICY_REBALANCE, ops.HM_LAYOUT_EP_EXPERT, me, m_all=m_all)
            torch.cuda.synchronize()
            buf = (ctypes.c_longlong * 8)()
            _lib.check(_lib.load().hm_debug_plan_phases(buf), "phases")
            t = list(buf)
            print(f"{placement} me={me}: hist {(t[1] - t[0]) / 1e3:.1f} us, schedule {(t[2] - t[1]) / 1e3:.1f} us, "
                  f"layout {(t[3] - t[2]) / 1e3:.1f} us [head {(t[4] - t[2]) / 1e3:.1f}, slots+segs "
                  f"{(t[5] - t[4]) / 1e3:.1f}, scan {(t[6] - t[5]) / 1e3:.1f}], iters {int(p.iters.item())}, "
                  f"clock {t[7] / max(1, t[3] - t[0]) * 1e3:.0f} MHz", flush=True)


if __name__ == "__main__":
    main()
