# Graph grouping without stage marks: 4 groups (default) vs 3 (gemm2+combine merged) vs 1, and
# the gemm1-only bracket on each.
python - <<'PY'
import torch, numpy as np
from paper_2506_12417_b200.block import HarMoEnyBlock, MoEConfig
import bench
G4 = (("router", "schedule", "permute"), ("gemm1",), ("gemm2",), ("combine",))
G3 = (("router", "schedule", "permute"), ("gemm1",), ("gemm2", "combine"))
G1 = (("router", "schedule", "permute", "gemm1", "gemm2", "combine"),)
for wl, T, G, q in (("switch128", 4096, 4, 4), ("qwen128", 16384, 1, 32)):
    d, f, E, k, act, _ = bench.WORKLOADS[wl]
    cfg = MoEConfig(d_model=d, d_ff=f, num_experts=E, top_k=k, activation=act, eq_tokens=q, logical_ranks=G)
    blk = HarMoEnyBlock.random(cfg, seed=0, device="cuda", zipf_s=1.0)
    x = torch.randn((T, d), device="cuda", generator=torch.Generator(device="cuda").manual_seed(1234)).to(torch.bfloat16)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device="cuda")
    s = torch.cuda.current_stream()
    caps = {}
    for name, grp in (("G4", G4), ("G3", G3), ("G1", G1)):
        caps[name] = blk.capture(T, groups=grp); caps[name].x.copy_(x)
    for r in range(3):
        for name, cap in caps.items():
            a = np.mean(bench._timed_steps(cap.replay, 20, 5, flush, s)) * 1e3
            b = np.mean(bench._timed_steps(lambda: cap.replay([], only={"gemm1"}), 20, 5, flush, s)) * 1e3
            print(wl, name, "no marks %.1f us" % a, "gemm1 bracket %.1f us" % b, flush=True)
PY
