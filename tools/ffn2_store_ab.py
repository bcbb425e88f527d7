"""FFN2 store-path experiment: token-major scatter (row_map) + dense combine vs expert-major
contiguous store + pos-gather combine, on the bench's Qwen-128 block."""
import sys, torch, numpy as np
sys.path.insert(0, '.')
from paper_2506_12417_b200 import ops
from paper_2506_12417_b200.block import HarMoEnyBlock, MoEConfig
cfg = MoEConfig(d_model=2048, d_ff=768, num_experts=128, top_k=8)
blk = HarMoEnyBlock.random(cfg, seed=0, zipf_s=1.0)
x = torch.randn((16384, 2048), device="cuda").to(torch.bfloat16)
y = blk(x); torch.cuda.synchronize()
st = blk.stats.extras
lay = st["layout"]; pos = st["pos"]; w = st["topk_w"]
T, k = 16384, 8
h = torch.randn((T * k, 768), device="cuda").to(torch.bfloat16) * 0.1
inv = torch.empty(T * k, dtype=torch.int32, device="cuda")
inv[pos.reshape(-1).long()] = torch.arange(T * k, dtype=torch.int32, device="cuda")
flush = torch.empty(64 * 1024 * 1024, dtype=torch.int32, device="cuda")
def timeit(fn, n=20):
    for _ in range(3): fn()
    ts = []
    for i in range(n):
        flush.fill_(i)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b) * 1e3)
    return float(np.median(ts))
Ytm = torch.empty((T * k, 2048), dtype=torch.bfloat16, device="cuda")
Yem = torch.empty((T * k, 2048), dtype=torch.bfloat16, device="cuda")
t1 = timeit(lambda: ops.grouped_gemm(h, blk.w_out, 2048, lay, ops.HM_EPI_STORE, out=Ytm, row_map=inv))
t2 = timeit(lambda: ops.grouped_gemm(h, blk.w_out, 2048, lay, ops.HM_EPI_STORE, out=Yem))
c1 = timeit(lambda: ops.combine(Ytm, None, w))
c2 = timeit(lambda: ops.combine(Yem, pos, w))
ya = ops.combine(Ytm, None, w); yb = ops.combine(Yem, pos, w); torch.cuda.synchronize()
print(f"token-major scatter FFN2 {t1:.1f} us + dense combine {c1:.1f} us = {t1 + c1:.1f}")
print(f"expert-major FFN2 {t2:.1f} us + pos-gather combine {c2:.1f} us = {t2 + c2:.1f}   identical: {torch.equal(ya, yb)}")
