"""Bandwidth of the in-GEMM K6 fetch pairs: a GEMM over tiny segments of n fetched experts
(qwen128 expert sizes), so the launch time is the copy time."""
import sys, time, torch
sys.path.insert(0, '.')
from paper_2506_12417_b200 import ops
dev = torch.device('cuda')
d, f = 2048, 768
n_in = 2 * f
for nf in (2, 8, 16):
    E = nf + 1
    i32 = dict(dtype=torch.int32, device=dev)
    segs = [[0, 8, 0, 0]] + [[8 * (i + 1), 8, 1 + i, 1 + i] for i in range(nf)]
    mt = [0]
    for s_ in segs: mt.append(mt[-1] + 1)
    segs_t, nseg_t, mt_t = torch.tensor(segs, **i32), torch.tensor([len(segs)], **i32), torch.tensor(mt, **i32)
    fetch_t = torch.tensor(list(range(1, E)), **i32); nf_t = torch.tensor([nf], **i32)
    lay = ops.Layout(None, segs_t, nseg_t, mt_t, fetch_t, nf_t)
    Win = (torch.randn((E, n_in, d), device=dev) * 0.05).to(torch.bfloat16)
    Wout = (torch.randn((E, d, f), device=dev) * 0.05).to(torch.bfloat16)
    src_in = torch.tensor([Win[e].data_ptr() for e in range(E)], dtype=torch.int64, device=dev)
    src_out = torch.tensor([Wout[e].data_ptr() for e in range(E)], dtype=torch.int64, device=dev)
    W1 = torch.zeros((E * n_in, d), dtype=torch.bfloat16, device=dev); W1[:n_in] = Win[0]
    W2 = torch.zeros((E * d, f), dtype=torch.bfloat16, device=dev)
    A = torch.randn((8 * E, d), device=dev).to(torch.bfloat16)
    ready_in = torch.zeros(E, **i32); ready_out = torch.zeros(E, **i32); done = torch.zeros(E, **i32); cnt = torch.zeros(2 * E, **i32)
    for pairs in (1, 2, 4):
        ts = []
        for ep in range(1, 6):
            done.zero_()
            fp = ops.fetch_plan(fetch_t, nf_t, src_in, src_out, W1, W2, n_in * d * 2, d * f * 2, 1, nf, ready_in, ready_out, cnt, ep, 1, pairs=pairs)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            ops.grouped_gemm(A, W1, n_in, lay, ops.HM_EPI_SWIGLU, slot_ready=ready_in, ready_from_slot=1, epoch=ep, slot_done=done, fetch=fp)
            b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b) * 1e3)
        us = sorted(ts)[2]
        nbytes = nf * (n_in * d + d * f) * 2
        print(f"{nf} experts, {pairs} fetch pairs: {us:.1f} us, {nbytes / us / 1e3:.0f} GB/s (local HBM -> HBM)", flush=True)
