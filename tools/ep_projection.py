"""One EP rank's share of a G-GPU expert-parallel step, measured on ONE B200.

Every kernel of rank `me`'s critical path runs for real at the per-rank size and is timed
alone (CUDA-graph replay, L2 flushed before each call, CUDA events):

  router      hm_router_topk on the rank's T/G tokens
  plan        hm_plan (EP layout of rank `me`) on the m_all the metadata exchange delivers
  dispatch    hm_dispatch_push of the rank's tokens (the G destination buffers are local here)
  ffn1/ffn2   the grouped GEMMs over rank `me`'s expert-major receive buffer (the p2p transport's
              HM_LAYOUT_EP_EXPERT: one segment per expert) with the EP weight slots (home experts,
              then the fetched experts in plan order)
  combine     hm_combine of the rank's T/G tokens

What one GPU cannot measure is modelled explicitly and reported separately: NVLink transfer
times at `nvlink_gbs` (dispatch rows out / in, FFN2 rows back, fetched expert weights) and a
fixed cost per cross-rank flag handshake (metadata, tokens, outputs).  The fetch channel is
modelled as the reference does (engine.py:204-275): one transfer at a time in plan order, a
fetched expert's FFN1 tiles start when its gate/up block has landed, resident experts first.

    python tools/ep_projection.py [--G 8] [--placement round_robin|blocked] [--q 32]
"""

from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_12417_b200 import ops  # noqa: E402
from paper_2506_12417_b200.block import MoEConfig, pack_w13, placement_home, random_weights  # noqa: E402


def _graph_time_us(fn, flush, reps=10):
    """Median device time of fn() replayed from a CUDA graph with the L2 flushed before each call."""
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        for _ in range(2):
            fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    ts = []
    for i in range(reps):
        flush.fill_(i)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return float(np.median(ts))


def _plan_orders(S, home_np):
    """Every destination's plan order (engine.py:233-234): residents with work by (-rows, e), then
    the other experts with work by (-rows, e)."""
    G, E, _ = S.shape
    orders = []
    for d in range(G):
        n = S[:, :, d].sum(axis=0)
        keys = sorted((0 if home_np[e] == d else 1, -int(n[e]), e) for e in range(E) if n[e] > 0)
        orders.append([e for _, _, e in keys])
    return orders


def _arrival_times(S, home_np, me, bytes_tok, nvlink_gbs, warps=592, unit_rows=8):
    """Expert-ordered dispatch (hm_dispatch_push_ordered): the time (us from the push start) at
    which every row of each of rank me's experts has landed.  Every sender walks its units (8 rows of
    one bucket) in (position, destination) order, dealt round-robin over its `warps` warps, so ~one
    round of `warps` units is in flight at a time and completes together: a unit lands when the
    sender's remote bytes up to the end of its round have left at nvlink_gbs.  Rank me's inbound
    link carries nvlink_gbs too; local rows (g == me) cost no NVLink time."""
    G, E, _ = S.shape
    orders = _plan_orders(S, home_np)
    P = max(len(o) for o in orders)
    bw = nvlink_gbs * 1e3  # bytes per us
    done = np.zeros((G, P))  # sender g: completion time of its item (p, me)
    for g in range(G):
        unit_bytes, last_unit = [], {}
        for p in range(P):
            for d in range(G):
                if p >= len(orders[d]):
                    continue
                rows = int(S[g, orders[d][p], d])
                for r0 in range(0, rows, unit_rows):
                    unit_bytes.append(min(unit_rows, rows - r0) * bytes_tok if d != g else 0)
                if d == me and rows:
                    last_unit[p] = len(unit_bytes) - 1
        cum = np.cumsum(unit_bytes) if unit_bytes else np.zeros(1)
        for p, u in last_unit.items():
            end = min(len(unit_bytes), (u // warps + 1) * warps) - 1
            done[g, p] = cum[end] / bw
    arrive = {}
    inbound = 0.0
    for p, e in enumerate(orders[me]):
        inbound += sum(S[g, e, me] for g in range(G) if g != me) * bytes_tok
        arrive[e] = max(max(done[g, p] for g in range(G) if g != me) if G > 1 else 0.0, inbound / bw)
    return arrive, orders[me]


def project(d=2048, f=768, E=128, k=8, act="swiglu", T=16384, G=8, q=32, placement="round_robin", zipf_s=1.0,
            nvlink_gbs=900.0, handshake_us=4.0, peak_tflops=None, ranks=None, seed=0, overlap=False):
    dev = torch.device("cuda")
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device=dev)
    cfg = MoEConfig(d_model=d, d_ff=f, num_experts=E, top_k=k, activation=act, eq_tokens=q, placement=placement,
                    logical_ranks=G)
    wg, w1, w2, w3, bias = random_weights(cfg, seed, dev, zipf_s)
    wgp = torch.zeros((ops.e_pad(E), d), dtype=torch.bfloat16, device=dev)
    wgp[:E] = wg
    if act == "swiglu":
        w_in_all = pack_w13(w1, w3).view(E, 2 * f, d)
        n_in, epi = 2 * f, ops.HM_EPI_SWIGLU
    else:
        w_in_all = w1.reshape(E, f, d)
        n_in, epi = f, ops.HM_EPI_RELU
    w_out_all = w2.reshape(E, d, f)
    Tg = T // G
    x = torch.randn((T, d), device=dev, generator=torch.Generator(device=dev).manual_seed(1234)).to(torch.bfloat16)
    # routing of every rank's tokens -> m_all (what the metadata exchange hands every rank)
    idx, w, tile_hist, lrank = ops.router_topk(x, wgp, bias, G, Tg, k, k > 1, E=E)
    tiles = (Tg + 127) // 128
    m_all, tile_off = ops.hist_scan(tile_hist, G, tiles)
    home = torch.from_numpy(placement_home(cfg)).to(dev)
    home_np = placement_home(cfg)
    bytes_tok = d * 2
    out = {"config": dict(d_model=d, d_ff=f, experts=E, top_k=k, tokens=T, G=G, q=q, placement=placement,
                          zipf_s=zipf_s, nvlink_gbs=nvlink_gbs, handshake_us=handshake_us,
                          dispatch="expert-ordered push overlapped with FFN1" if overlap else "push, then FFN1")}
    overlap = overlap and G & (G - 1) == 0
    # rank-independent kernels
    xr = x[:Tg].contiguous()
    out["router_us"] = _graph_time_us(lambda: ops.router_topk(xr, wgp, bias, 1, Tg, k, k > 1, E=E), flush)
    mode = ops.HM_LAYOUT_EP_EXPERT  # the p2p transport's expert-major receive buffers
    plan0 = ops.plan(home, G, E, q, ops.HM_POLICY_REBALANCE, mode, 0, m_all=m_all)
    torch.cuda.synchronize()
    S = plan0.S.cpu().numpy().astype(np.int64)
    loads = S.sum(axis=(0, 1))
    out["moves"] = int(plan0.iters.item())
    out["load_max_over_mean"] = float(loads.max() / loads.mean())
    ranks = list(range(G)) if ranks is None else ranks
    per_rank = {}
    f1_flops_per_row = 2.0 * d * n_in
    f2_flops_per_row = 2.0 * f * d
    expert_bytes = (n_in * d + d * f) * 2
    for me in ranks:
        r = {}
        if overlap:
            r["plan_us"] = _graph_time_us(lambda: ops.plan_dispatch(home, G, E, q, ops.HM_POLICY_REBALANCE, me,
                                                                    m_all), flush)
        else:
            r["plan_us"] = _graph_time_us(lambda: ops.plan(home, G, E, q, ops.HM_POLICY_REBALANCE, mode, me,
                                                           m_all=m_all), flush)
        p = ops.plan(home, G, E, q, ops.HM_POLICY_REBALANCE, mode, me, m_all=m_all)
        lay = p.layout
        n_seg = int(lay.n_seg.item())
        n_fetch = int(lay.n_fetch.item())
        segs = lay.segs[:n_seg].cpu().numpy()
        fetched = lay.fetch[:n_fetch].cpu().numpy().tolist()
        rows = int(segs[:, 1].sum()) if n_seg else 0
        r.update(recv_rows=rows, fetched_experts=n_fetch, segments=n_seg)
        # dispatch push of my tokens into G local stand-ins for the destination buffers
        cap = int(loads.max()) + 1
        bufs = [torch.empty((cap, d), dtype=torch.bfloat16, device=dev) for _ in range(G)]
        toks = [torch.empty(cap, dtype=torch.int32, device=dev) for _ in range(G)]
        i64 = dict(dtype=torch.int64, device=dev)
        dst_rows = torch.tensor([b.data_ptr() for b in bufs], **i64)
        dst_tok = torch.tensor([t.data_ptr() for t in toks], **i64)
        sl = slice(me * Tg, (me + 1) * Tg)
        idx_me, lrank_me = idx[sl].contiguous(), lrank[sl].contiguous()
        toff_me = tile_off[me * tiles:(me + 1) * tiles].contiguous()
        x_me = x[sl].contiguous()
        r["dispatch_local_us"] = _graph_time_us(
            lambda: ops.dispatch_push(x_me, idx_me, lrank_me, toff_me, p.S, lay.slot_base, None, me, dst_rows,
                                      dst_tok), flush)
        flows = S.sum(axis=1)
        sent = int(flows[me].sum() - flows[me, me])
        recv = int(flows[:, me].sum() - flows[me, me])
        r["dispatch_nvlink_us"] = max(sent, recv) * bytes_tok / (nvlink_gbs * 1e3)
        # my receive buffer and weight slots (home experts ascending, then fetched in plan order)
        n_home = int((home_np == me).sum())
        slot_experts = [e for e in range(E) if home_np[e] == me] + fetched
        sidx = torch.tensor(slot_experts, dtype=torch.long, device=dev)
        w_in = w_in_all[sidx].reshape(-1, d).contiguous()
        w_out = w_out_all[sidx].reshape(-1, f).contiguous()
        a = torch.randn((max(rows, 1), d), device=dev).to(torch.bfloat16)
        h = torch.empty((max(rows, 1), n_in // (2 if act == "swiglu" else 1)), dtype=torch.bfloat16, device=dev)
        y = torch.empty((max(rows, 1), d), dtype=torch.bfloat16, device=dev)
        r["ffn1_us"] = _graph_time_us(lambda: ops.grouped_gemm(a, w_in, n_in, lay, epi, out=h), flush)
        if n_fetch:
            # K6 co-running: the fetch kernel (local copies standing in for the NVLink reads) on its
            # own stream beside FFN1, whose tiles of fetched experts wait on the ready flags - shows
            # whether the copy takes SMs from the persistent GEMM
            src_in = torch.tensor([w_in_all[e_].data_ptr() for e_ in range(E)], **i64)
            src_out = torch.tensor([w_out_all[e_].data_ptr() for e_ in range(E)], **i64)
            rdy_in = torch.zeros(E, dtype=torch.int32, device=dev)
            rdy_out = torch.zeros(E, dtype=torch.int32, device=dev)
            ctr = torch.zeros(2 * E, dtype=torch.int32, device=dev)
            fs = torch.cuda.Stream()

            def ffn1_fetch():
                cur = torch.cuda.current_stream()
                rdy_in.zero_()
                rdy_out.zero_()
                fs.wait_stream(cur)
                ops.fetch_experts(lay.fetch, lay.n_fetch, src_in, src_out, n_in * d * 2, d * f * 2, w_in, w_out,
                                  n_home, n_fetch, rdy_in, rdy_out, ctr, value=1, stream=fs)
                ops.grouped_gemm(a, w_in, n_in, lay, epi, out=h, slot_ready=rdy_in, ready_from_slot=n_home, epoch=1)
                cur.wait_stream(fs)

            r["ffn1_fetch_corun_local_us"] = _graph_time_us(ffn1_fetch, flush)
            r["fetch_local_us"] = _graph_time_us(
                lambda: ops.fetch_experts(lay.fetch, lay.n_fetch, src_in, src_out, n_in * d * 2, d * f * 2, w_in,
                                          w_out, n_home, n_fetch, rdy_in, rdy_out, ctr, value=1), flush)
        if overlap:
            # the push of my tokens (into G local stand-ins) with my FFN1 launched right behind it
            # (PDL), its arrival counters pre-filled with the rows the other senders deliver: what
            # one GPU can measure of the overlap (SM / HBM sharing of push and GEMM)
            _, pl = ops.plan_dispatch(home, G, E, q, ops.HM_POLICY_REBALANCE, me, m_all)
            n_e = S[:, :, me].sum(axis=0)
            pre = torch.from_numpy((n_e - S[me, :, me]).astype(np.int32)).to(dev)
            arrive = torch.zeros((G, E), dtype=torch.int32, device=dev)
            arrive_ptrs = torch.tensor([arrive[g_].data_ptr() for g_ in range(G)], **i64)
            order = torch.empty(Tg * k, dtype=torch.int32, device=dev)
            sync = torch.zeros(2, dtype=torch.int32, device=dev)
            a_me = bufs[me]

            def push():
                ops.dispatch_push_ordered(x_me, idx_me, lrank_me, toff_me, p.S, lay.slot_base, pl, me, dst_rows,
                                          dst_tok, arrive_ptrs, order, sync)

            def push_ffn1():
                arrive[me].copy_(pre)
                push()
                ops.grouped_gemm_arrive(a_me, w_in, n_in, lay, epi, arrive[me], out=h, pdl=True)

            r["push_ordered_local_us"] = _graph_time_us(lambda: (arrive.zero_(), push()), flush)
            r["push_ffn1_local_us"] = _graph_time_us(push_ffn1, flush)
        r["ffn2_us"] = _graph_time_us(lambda: ops.grouped_gemm(h, w_out, d, lay, ops.HM_EPI_STORE, out=y), flush)
        # resident experts' share of FFN1 (their segments come first in plan order)
        n_res_seg = int(sum(1 for s_ in segs if s_[2] < n_home))
        rows_res = int(segs[:n_res_seg, 1].sum()) if n_res_seg else 0
        if n_fetch and n_res_seg:
            lay_res = ops.Layout(lay.slot_base, lay.segs, torch.tensor([n_res_seg], dtype=torch.int32, device=dev),
                                 lay.mtile_prefix, lay.fetch, lay.n_fetch)
            r["ffn1_resident_us"] = _graph_time_us(lambda: ops.grouped_gemm(a, w_in, n_in, lay_res, epi, out=h),
                                                   flush)
        else:
            r["ffn1_resident_us"] = r["ffn1_us"] if not n_fetch else 0.0
        # fetch channel: plan order, every gate/up block before the down blocks (hm_fetch_experts);
        # a fetched expert's FFN1 share starts when its gate/up block has landed
        t_one = expert_bytes / (nvlink_gbs * 1e3)
        t_in = t_one * (n_in * d) / (n_in * d + d * f)
        t = r["ffn1_resident_us"]
        fetched_rows = rows - rows_res
        for j, e in enumerate(fetched):
            rows_e = int(sum(s_[1] for s_ in segs if s_[3] == e))
            share = (r["ffn1_us"] - r["ffn1_resident_us"]) * rows_e / max(fetched_rows, 1)
            t = max(t, (j + 1) * t_in) + share
        r["fetch_nvlink_us"] = n_fetch * t_one
        r["ffn1_with_fetch_us"] = max(t, r["ffn1_us"], r.get("ffn1_fetch_corun_local_us", 0.0))
        if overlap:
            # FFN1 timeline from the push start: expert e's share (its rows of FFN1, the measured
            # co-running FFN1 time) starts once its rows have landed and, if fetched, its gate/up
            # block (fetch channel as above, starting with the push)
            arr, order_me = _arrival_times(S, home_np, me, bytes_tok, nvlink_gbs)
            f1 = max(r["push_ffn1_local_us"], r["ffn1_us"])
            fetch_ready = {e: (j + 1) * t_in for j, e in enumerate(fetched)}
            seg_rows = {int(s_[3]): int(s_[1]) for s_ in segs}
            t = 0.0
            for e in order_me:
                t = max(t, arr[e], fetch_ready.get(e, 0.0)) + f1 * seg_rows.get(e, 0) / max(rows, 1)
            r["last_arrival_us"] = max(arr.values()) if arr else 0.0
            r["dispatch_ffn1_us"] = max(t, f1, r["dispatch_nvlink_us"])
        # FFN2 needs every down block; its rows for other ranks go back over NVLink in the epilogue
        back = rows - int(S[me, :, me].sum())
        r["return_nvlink_us"] = back * bytes_tok / (nvlink_gbs * 1e3)
        # the channel ends at n_fetch * t_one after FFN1 started; FFN2 reaches its fetched experts
        # (last in plan order) after its resident share
        tail = r["ffn2_us"] * fetched_rows / max(rows, 1)
        r["ffn2_with_fetch_us"] = max(r["ffn2_us"], r["return_nvlink_us"],
                                      n_fetch * t_one - (r["dispatch_ffn1_us"] if overlap else r["ffn1_with_fetch_us"])
                                      + tail)
        yk = torch.randn((Tg * k, d), device=dev).to(torch.bfloat16)
        w_me = w[sl].contiguous()
        r["combine_us"] = _graph_time_us(lambda: ops.combine(yk, None, w_me), flush)
        if overlap:  # metadata and output flags; the token flag is replaced by the arrival counters
            r["handshakes_us"] = 2 * handshake_us
            r["step_us"] = (out["router_us"] + r["handshakes_us"] + r["plan_us"] + r["dispatch_ffn1_us"] +
                            r["ffn2_with_fetch_us"] + r["combine_us"])
        else:
            r["handshakes_us"] = 3 * handshake_us
            r["step_us"] = (out["router_us"] + r["handshakes_us"] + r["plan_us"] +
                            max(r["dispatch_local_us"], r["dispatch_nvlink_us"]) + r["ffn1_with_fetch_us"] +
                            r["ffn2_with_fetch_us"] + r["combine_us"])
        r["gemm_flops"] = rows * (f1_flops_per_row + f2_flops_per_row)
        per_rank[me] = r
        del bufs, toks, a, h, y, w_in, w_out
        torch.cuda.empty_cache()
    out["per_rank"] = per_rank
    crit = max(per_rank, key=lambda m: per_rank[m]["step_us"])
    out["critical_rank"] = crit
    step = per_rank[crit]["step_us"]
    out["projected_step_us"] = step
    out["projected_tokens_per_s"] = T / (step * 1e-6)
    if peak_tflops:
        balanced = T * k * (f1_flops_per_row + f2_flops_per_row) / G
        out["gemm_roofline_us"] = balanced / (peak_tflops * 1e12) * 1e6
        out["projected_roofline_frac"] = out["gemm_roofline_us"] / step
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--G", type=int, default=8)
    ap.add_argument("--placement", default="round_robin")
    ap.add_argument("--q", type=int, default=32)
    ap.add_argument("--zipf", type=float, default=1.0)
    ap.add_argument("--peak", type=float, default=1631.3)
    ap.add_argument("--overlap", action="store_true", help="expert-ordered push overlapped with FFN1 (opt-in)")
    a = ap.parse_args()
    res = project(G=a.G, q=a.q, placement=a.placement, zipf_s=a.zipf, peak_tflops=a.peak, overlap=a.overlap)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
