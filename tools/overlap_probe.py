"""Diagnostics: ordered dispatch push alone, FFN1 alone, and push + FFN1 (PDL) on one GPU, eager
and graph-captured (one EP rank's share of C2 at G=8: its tokens pushed into G local stand-ins)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_12417_b200 import ops  # noqa: E402
from paper_2506_12417_b200.block import MoEConfig, pack_w13, placement_home, random_weights  # noqa: E402


def ev_time(fn, n=10):
    """Median device time of fn() replayed from a CUDA graph (no host launch gaps)."""
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(2):
            fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    fn = g.replay
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(n):
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return float(np.median(ts))


def main():
    d, f, E, k, T, G, me = 2048, 768, 128, 8, 16384, 8, 5
    dev = torch.device("cuda")
    cfg = MoEConfig(d_model=d, d_ff=f, num_experts=E, top_k=k, eq_tokens=32, logical_ranks=G)
    wg, w1, w2, w3, bias = random_weights(cfg, 0, dev, 1.0)
    wgp = torch.zeros((ops.e_pad(E), d), dtype=torch.bfloat16, device=dev)
    wgp[:E] = wg
    w_in = pack_w13(w1, w3).reshape(-1, d)
    Tg = T // G
    x = torch.randn((T, d), device=dev).to(torch.bfloat16)
    idx, w, tile_hist, lrank = ops.router_topk(x, wgp, bias, G, Tg, k, True, E=E)
    tiles = Tg // 128
    m_all, tile_off = ops.hist_scan(tile_hist, G, tiles)
    home = torch.from_numpy(placement_home(cfg)).to(dev)
    p, pl = ops.plan_dispatch(home, G, E, 32, True, me, m_all)
    S = p.S.cpu().numpy()
    rows = int(S[:, :, me].sum())
    cap = int(S.sum(axis=(0, 1)).max()) + 1
    bufs = [torch.zeros((cap, d), dtype=torch.bfloat16, device=dev) for _ in range(G)]
    toks = [torch.zeros(cap, dtype=torch.int32, device=dev) for _ in range(G)]
    i64 = dict(dtype=torch.int64, device=dev)
    dst_rows = torch.tensor([b.data_ptr() for b in bufs], **i64)
    dst_tok = torch.tensor([t.data_ptr() for t in toks], **i64)
    arrive = torch.zeros((G, E), dtype=torch.int32, device=dev)
    arrive_ptrs = torch.tensor([arrive[g].data_ptr() for g in range(G)], **i64)
    order = torch.empty(Tg * k, dtype=torch.int32, device=dev)
    sync = torch.zeros(2, dtype=torch.int32, device=dev)
    sl = slice(me * Tg, (me + 1) * Tg)
    xm, im, lm = x[sl].contiguous(), idx[sl].contiguous(), lrank[sl].contiguous()
    tm = tile_off[me * tiles:(me + 1) * tiles].contiguous()
    pre = torch.from_numpy((S[:, :, me].sum(axis=0) - S[me, :, me]).astype(np.int32)).to(dev)
    h = torch.empty((cap, f), dtype=torch.bfloat16, device=dev)
    lay = p.layout

    def push():
        arrive.zero_()
        arrive[me].copy_(pre)
        ops.dispatch_push_ordered(xm, im, lm, tm, p.S, lay.slot_base, pl, me, dst_rows, dst_tok, arrive_ptrs, order,
                                  sync)

    def push_plain():
        ops.dispatch_push(xm, im, lm, tm, p.S, lay.slot_base, None, me, dst_rows, dst_tok)

    def ffn1():
        ops.grouped_gemm(bufs[me], w_in, 2 * f, lay, ops.HM_EPI_SWIGLU, out=h)

    def both(pdl=True):
        push()
        ops.grouped_gemm_arrive(bufs[me], w_in, 2 * f, lay, ops.HM_EPI_SWIGLU, arrive[me], out=h, pdl=pdl)

    print(f"rank {me}: {rows} receive rows")
    print(f"unordered push   {ev_time(push_plain):7.1f} us")
    print(f"ordered push     {ev_time(push):7.1f} us")
    print(f"FFN1             {ev_time(ffn1):7.1f} us")
    print(f"push + FFN1 PDL  {ev_time(both):7.1f} us")
    print(f"push + FFN1 ser. {ev_time(lambda: both(False)):7.1f} us")
    print(f"counters only    {ev_time(lambda: (arrive.zero_(), arrive[me].copy_(pre))):7.1f} us")
    full = torch.from_numpy(S[:, :, me].sum(axis=0).astype(np.int32)).to(dev)
    arr_full = torch.zeros(E, dtype=torch.int32, device=dev)

    def both_nowait(pdl=True):
        push()
        arr_full.copy_(full)
        ops.grouped_gemm_arrive(bufs[me], w_in, 2 * f, lay, ops.HM_EPI_SWIGLU, arr_full, out=h, pdl=pdl)

    def both_nowait2(pdl=True):
        arr_full.copy_(full)
        push()
        ops.grouped_gemm_arrive(bufs[me], w_in, 2 * f, lay, ops.HM_EPI_SWIGLU, arr_full, out=h, pdl=pdl)

    print(f"push + FFN1 (counters full, copy between) PDL {ev_time(both_nowait):7.1f} us")
    print(f"push + FFN1 (counters full) PDL {ev_time(both_nowait2):7.1f} us, serial "
          f"{ev_time(lambda: both_nowait2(False)):7.1f} us")


if __name__ == "__main__":
    main()
