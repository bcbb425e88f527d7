"""Small eager forwards of every hot-path kernel for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck):  bash tools/sanitize.sh  (diagnostics, run on the GPU box)."""

import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_12417_b200.block import HarMoEnyBlock, MoEConfig  # noqa: E402


def main():
    dev = torch.device("cuda")
    for kw in (dict(top_k=4, activation="swiglu", logical_ranks=2),  # fused gather FFN1
               dict(top_k=2, activation="swiglu", logical_ranks=1),  # copy-permute + TMA FFN1
               dict(top_k=1, activation="relu", logical_ranks=4)):
        cfg = MoEConfig(d_model=256, num_experts=16, d_ff=256, eq_tokens=2, placement="blocked", **kw)
        blk = HarMoEnyBlock.random(cfg, seed=1, device=dev, zipf_s=1.2, std=0.05)
        x = torch.randn((400, 256), device=dev).to(torch.bfloat16)
        y = blk(x)
        torch.cuda.synchronize()
        print(kw, "ok", float(y.float().abs().sum()))
    ordered_push_and_fetch(dev)


def ordered_push_and_fetch(dev):
    """The EP kernels that need no second process: plan_dispatch + the ordered push into G local
    stand-in receive buffers + FFN1 gated by the arrival counters (PDL), and the K6 fetch kernel."""
    import numpy as np

    from oracle import moe_oracle as orc
    from paper_2506_12417_b200 import ops

    G, E, k, d, Tg = 2, 16, 2, 256, 200
    wg = torch.zeros((ops.e_pad(E), d), dtype=torch.bfloat16, device=dev)
    wg[:E] = (torch.randn((E, d), device=dev) * 0.05).to(torch.bfloat16)
    bias = torch.linspace(1.0, -1.0, E, device=dev)
    xs, routed, hists = [], [], []
    for _ in range(G):
        x = torch.randn((Tg, d), device=dev).to(torch.bfloat16)
        idx, _, th, lrank = ops.router_topk(x, wg, bias, 1, Tg, k, True, E=E)
        hist, toff = ops.hist_scan(th, 1, (Tg + 127) // 128)
        xs.append(x)
        routed.append((idx, lrank, toff))
        hists.append(hist)
    m_all = torch.cat(hists).contiguous()
    home = torch.from_numpy(orc.blocked_home(E, G).astype(np.int32)).to(dev)
    cap = G * Tg * k
    rows = [torch.zeros((cap, d), dtype=torch.bfloat16, device=dev) for _ in range(G)]
    toks = [torch.zeros(cap, dtype=torch.int32, device=dev) for _ in range(G)]
    arrive = torch.zeros((G, E), dtype=torch.int32, device=dev)
    i64 = dict(dtype=torch.int64, device=dev)
    ptr = lambda ts: torch.tensor([t.data_ptr() for t in ts], **i64)  # noqa: E731
    order = torch.empty(Tg * k, dtype=torch.int32, device=dev)
    sync = torch.zeros(2, dtype=torch.int32, device=dev)
    lay = None
    for me in range(G):
        p, pl = ops.plan_dispatch(home, G, E, 2, True, me, m_all)
        idx, lrank, toff = routed[me]
        ops.dispatch_push_ordered(xs[me], idx, lrank, toff, p.S, p.layout.slot_base, pl, me, ptr(rows), ptr(toks),
                                  torch.tensor([arrive[g].data_ptr() for g in range(G)], **i64), order, sync)
        lay = p.layout
    W = (torch.randn((E * 256, d), device=dev) * 0.05).to(torch.bfloat16)
    h = ops.grouped_gemm_arrive(rows[G - 1], W, 256, lay, ops.HM_EPI_RELU, arrive[G - 1], pdl=True)
    # K6: fetch the layout's fetch list from local "home" copies into cache slots
    w_in = torch.randn((E, 256, d), device=dev).to(torch.bfloat16)
    w_out = torch.randn((E, d, 128), device=dev).to(torch.bfloat16)
    src_in = torch.tensor([w_in[e].data_ptr() for e in range(E)], **i64)
    src_out = torch.tensor([w_out[e].data_ptr() for e in range(E)], **i64)
    dst_in, dst_out = torch.empty_like(w_in), torch.empty_like(w_out)
    r_in = torch.zeros(E, dtype=torch.int32, device=dev)
    r_out = torch.zeros(E, dtype=torch.int32, device=dev)
    ctr = torch.zeros(2 * E, dtype=torch.int32, device=dev)
    ops.fetch_experts(lay.fetch, lay.n_fetch, src_in, src_out, 256 * d * 2, d * 128 * 2, dst_in, dst_out, 0, E,
                      r_in, r_out, ctr, value=1)
    torch.cuda.synchronize()
    n = int(m_all.sum().item()) if G == 1 else int(p.S[:, :, G - 1].sum().item())  # rows written
    print("ordered push + arrive-gated FFN1 + fetch ok", float(h[:n].float().abs().sum()))


if __name__ == "__main__":
    main()
