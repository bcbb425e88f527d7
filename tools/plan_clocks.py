"""Planner phase cycles (diagnostics build: bash tools/build_variant.sh pst -DHM_PLAN_STAMPS;
HM_LIB_PATH=paper_2506_12417_b200/libharmoe_pst.so python tools/plan_clocks.py).
Stamps: 0 start, 1 m_all loaded, 2 schedule init done, 3 rebalance done, 4 S written,
5.. layout sub-phases (LOCAL: 5 counts+scans, 6 slot_base+keys, 7 ranks+segs, 8 tile scan;
EP_EXPERT: 5 counts, 6 scans+slot_base+keys, 7 ranks+segs, 8 tile scan)."""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_12417_b200 import _lib, ops  # noqa: E402
from paper_2506_12417_b200.block import HarMoEnyBlock, MoEConfig, placement_home, random_weights  # noqa: E402


def clocks(lib):
    buf = (ctypes.c_longlong * 16)()
    assert lib.hm_debug_plan_clocks(buf) == 0
    t = list(buf)
    return " ".join(f"{i}:{(t[i] - t[i - 1]) / 1e3:.1f}k" for i in range(1, 9) if t[i] >= t[i - 1] > 0)


def main():
    lib = _lib.load()
    for (d, f, k, act, T, G, q, pl) in ((768, 3072, 1, "relu", 4096, 4, 4, "round_robin"),
                                         (2048, 768, 8, "swiglu", 16384, 8, 32, "round_robin"),
                                         (2048, 768, 8, "swiglu", 16384, 8, 32, "blocked")):
        cfg = MoEConfig(d_model=d, d_ff=f, num_experts=128, top_k=k, activation=act, logical_ranks=G, eq_tokens=q,
                        placement=pl)
        blk = HarMoEnyBlock.random(cfg, seed=0, zipf_s=1.0)
        x = torch.randn((T, d), device="cuda").to(torch.bfloat16)
        for _ in range(3):
            blk(x)
        torch.cuda.synchronize()
        print(f"LOCAL d={d} G={G} {pl} iters {int(blk.stats.iters.item())}: kcycles {clocks(lib)}", flush=True)
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
        for _ in range(3):
            p = ops.plan(home, G, E, 32, ops.HM_POLICY_REBALANCE, ops.HM_LAYOUT_EP_EXPERT, 3, m_all=m_all)
        torch.cuda.synchronize()
        print(f"EP_EXPERT G={G} {placement} iters {int(p.iters.item())}: kcycles {clocks(lib)}", flush=True)


if __name__ == "__main__":
    main()
