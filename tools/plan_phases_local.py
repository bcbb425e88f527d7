# needs a diagnostics build: bash tools/build_variant.sh phases -DHM_PLAN_PHASES; HM_LIB_PATH=paper_2506_12417_b200/libharmoe_phases.so
import ctypes, sys, torch
sys.path.insert(0, '.')
from paper_2506_12417_b200 import _lib
from paper_2506_12417_b200.block import HarMoEnyBlock, MoEConfig
for (d, f, k, act, T, G, q) in ((768, 3072, 1, "relu", 4096, 4, 4), (2048, 768, 8, "swiglu", 16384, 8, 32), (2048, 768, 8, "swiglu", 16384, 4, 32)):
    cfg = MoEConfig(d_model=d, d_ff=f, num_experts=128, top_k=k, activation=act, logical_ranks=G, eq_tokens=q, placement="round_robin")
    blk = HarMoEnyBlock.random(cfg, seed=0, zipf_s=1.0)
    x = torch.randn((T, d), device="cuda").to(torch.bfloat16)
    for _ in range(3):
        blk(x)
    torch.cuda.synchronize()
    buf = (ctypes.c_longlong * 8)()
    _lib.check(_lib.load().hm_debug_plan_phases(buf), "phases")
    t = list(buf)
    print(f"d={d} G={G}: hist {(t[1]-t[0])/1e3:.1f} us, schedule {(t[2]-t[1])/1e3:.1f} us, layout {(t[3]-t[2])/1e3:.1f} us "
          f"[head {(t[4]-t[2])/1e3:.1f}, slots+segs {(t[5]-t[4])/1e3:.1f}, scan {(t[6]-t[5])/1e3:.1f}], iters {int(blk.stats.iters.item())}")
    print(f"   SM clock during the planner: {t[7] / ((t[3] - t[0])) * 1e3:.0f} MHz ({t[7]} cycles)")
