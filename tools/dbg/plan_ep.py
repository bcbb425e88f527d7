import ctypes, os, sys, torch, numpy as np
sys.path.insert(0, '.')
from paper_2506_12417_b200 import _lib, ops
from paper_2506_12417_b200.workload import zipf_routing_matrix
from oracle import moe_oracle as orc
for pl in ("round_robin", "blocked"):
    G, E = 8, 128
    m = zipf_routing_matrix(G, 2048, E, 8, 1.0, 11)
    home = orc.blocked_home(E, G) if pl == "blocked" else orc.round_robin_home(E, G)
    mt = torch.from_numpy(m.astype(np.int32)).cuda(); ht = torch.from_numpy(home.astype(np.int32)).cuda()
    for mode in (ops.HM_LAYOUT_EP, ops.HM_LAYOUT_EP_EXPERT):
        for _ in range(5):
            p = ops.plan(ht, G, E, 32, True, mode, 3, m_all=mt)
        torch.cuda.synchronize()
        buf = (ctypes.c_longlong * 8)()
        _lib.check(_lib.load().hm_debug_plan_phases(buf), "phases")
        t = list(buf)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(20):
            ops.plan(ht, G, E, 32, True, mode, 3, m_all=mt)
        b.record(); torch.cuda.synchronize()
        print(f"{pl} mode {mode}: load {(t[1]-t[0])/1e3:.1f} us, schedule {(t[2]-t[1])/1e3:.1f} us, layout {(t[3]-t[2])/1e3:.1f} us, iters {int(p.iters.item())}; back-to-back {a.elapsed_time(b)/20*1e3:.1f} us/launch")
