"""GPU tests of the layout kernel (both layouts), the async expert fetch (K6)
and the expert-parallel block on a 1-rank NCCL group."""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import moe_oracle as orc  # noqa: E402

pytestmark = pytest.mark.gpu


def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda")


def _rand_S(G, E, T, k, s, seed, placement):
    from paper_2506_12417_b200.workload import zipf_routing_matrix

    m = zipf_routing_matrix(G, T // G, E, k, s, seed)
    home = orc.blocked_home(E, G) if placement == "blocked" else orc.round_robin_home(E, G)
    S, _ = orc.schedule(m, home, 1, True)
    return m, home, S


@pytest.mark.parametrize("G,E", [(1, 16), (4, 32), (8, 128), (3, 10)])
def test_layout_local_matches_oracle(G, E):
    from paper_2506_12417_b200 import ops

    dev = _cuda()
    m, home, S = _rand_S(G, E, 512 * G, 4 if E >= 4 else 1, 1.2, G * 7 + E, "blocked")
    St = torch.from_numpy(S.astype(np.int32)).to(dev)
    ht = torch.from_numpy(home.astype(np.int32)).to(dev)
    lay = ops.dispatch_layout(St, ht, ops.HM_LAYOUT_LOCAL)
    torch.cuda.synchronize()
    n_seg = int(lay.n_seg.item())
    segs = [tuple(r) for r in lay.segs[:n_seg].cpu().numpy().tolist()]
    assert segs == orc.local_segments(S, home)
    mp = lay.mtile_prefix[: n_seg + 1].cpu().numpy()
    assert np.array_equal(mp, np.concatenate([[0], np.cumsum([(s[1] + 127) // 128 for s in segs])]))
    assert int(lay.n_fetch.item()) == 0


@pytest.mark.parametrize("G,E,me", [(2, 16, 0), (2, 16, 1), (8, 128, 3), (4, 10, 2)])
def test_layout_ep_matches_oracle(G, E, me):
    from paper_2506_12417_b200 import ops

    dev = _cuda()
    m, home, S = _rand_S(G, E, 256 * G, 2, 1.5, G + E + me, "blocked")
    St = torch.from_numpy(S.astype(np.int32)).to(dev)
    ht = torch.from_numpy(home.astype(np.int32)).to(dev)
    lay = ops.dispatch_layout(St, ht, ops.HM_LAYOUT_EP, me)
    torch.cuda.synchronize()
    n_seg = int(lay.n_seg.item())
    segs = [tuple(r) for r in lay.segs[:n_seg].cpu().numpy().tolist()]
    assert segs == orc.ep_recv_segments(S, home, me)
    n_fetch = int(lay.n_fetch.item())
    fetched = lay.fetch[:n_fetch].cpu().numpy().tolist()
    resident = (home == me).astype(np.int32)
    order = orc.plan_order(S[:, :, me].sum(axis=0), resident)
    assert fetched == [int(e) for e in order if not resident[e]]  # plan order, one channel


@pytest.mark.parametrize("G,E,me,cache", [(2, 16, 0, 0), (2, 16, 1, 0), (8, 128, 3, 0), (4, 10, 2, 0),
                                           (8, 128, 5, 2), (4, 32, 1, 1)])
def test_layout_ep_expert_matches_oracle(G, E, me, cache):
    """Expert-major receive layout of the one-sided p2p dispatch: every bucket's row in its
    destination's buffer, one GEMM segment per expert in plan order, bounded-cache slots."""
    from paper_2506_12417_b200 import ops

    dev = _cuda()
    m, home, S = _rand_S(G, E, 256 * G, 2, 1.5, G + E + me, "blocked")
    St = torch.from_numpy(S.astype(np.int32)).to(dev)
    ht = torch.from_numpy(home.astype(np.int32)).to(dev)
    lay = ops.dispatch_layout(St, ht, ops.HM_LAYOUT_EP_EXPERT, me, cache_slots=cache)
    torch.cuda.synchronize()
    sb_ref, segs_ref = orc.ep_expert_layout(S, home, me, cache)
    assert np.array_equal(lay.slot_base.cpu().numpy(), sb_ref)
    n_seg = int(lay.n_seg.item())
    assert [tuple(r) for r in lay.segs[:n_seg].cpu().numpy().tolist()] == segs_ref
    mp = lay.mtile_prefix[: n_seg + 1].cpu().numpy()
    assert np.array_equal(mp, np.concatenate([[0], np.cumsum([(sg[1] + 127) // 128 for sg in segs_ref])]))
    resident = (home == me).astype(np.int32)
    order = orc.plan_order(S[:, :, me].sum(axis=0), resident)
    assert lay.fetch[: int(lay.n_fetch.item())].cpu().numpy().tolist() == [int(e) for e in order if not resident[e]]


def test_permute_positions_ep_match_oracle():
    """EP send layout: positions of every assignment = oracle ep_send_positions."""
    from paper_2506_12417_b200 import ops

    dev = _cuda()
    G, E, k, me, Tg, d = 4, 32, 4, 1, 384, 256
    rng = np.random.default_rng(0)
    idx = np.stack([rng.permutation(E)[:k] for _ in range(Tg)]).astype(np.int32)
    m_me = np.bincount(idx.reshape(-1), minlength=E)
    from paper_2506_12417_b200.workload import zipf_routing_matrix

    m = zipf_routing_matrix(G, Tg, E, k, 1.0, 5)
    m[me] = m_me
    home = orc.blocked_home(E, G)
    S, _ = orc.schedule(m, home, 1, True)
    St = torch.from_numpy(S.astype(np.int32)).to(dev)
    lay = ops.dispatch_layout(St, torch.from_numpy(home.astype(np.int32)).to(dev), ops.HM_LAYOUT_EP, me)
    # lrank / tile_off exactly as the router would produce them
    tiles = (Tg + 127) // 128
    lrank = np.zeros_like(idx)
    tile_hist = np.zeros((tiles, E), np.int32)
    for t in range(Tg):
        for j in range(k):
            e = idx[t, j]
            lrank[t, j] = tile_hist[t // 128, e]
            tile_hist[t // 128, e] += 1
    tile_off = (np.cumsum(tile_hist, axis=0) - tile_hist).astype(np.int32)
    x = torch.randn((Tg, d), device=dev).to(torch.bfloat16)
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    out, pos, _ = ops.permute(x, T(idx), T(lrank), T(tile_off), St, lay.slot_base, 1, Tg, me, Tg * k)
    torch.cuda.synchronize()
    assert np.array_equal(pos.cpu().numpy(), orc.ep_send_positions(idx, S, me))
    p = pos.cpu().numpy()
    for j in range(k):
        assert torch.equal(out[torch.from_numpy(p[:, j]).long().to(dev)], x)


def test_async_fetch_gates_gemm():
    """K6: GEMM tiles of fetched slots wait for the slot's ready flag while the weights
    stream in from pinned host memory on a side stream; results are exact."""
    from paper_2506_12417_b200 import ops

    dev = _cuda()
    N, K, slots, n_home = 256, 512, 6, 2
    W_host = (torch.randn((slots, N, K)) * 0.05).to(torch.bfloat16).pin_memory()
    W = torch.zeros((slots * N, K), dtype=torch.bfloat16, device=dev)
    W[: n_home * N] = W_host[:n_home].reshape(-1, K).to(dev)
    counts = [300, 200, 129, 64, 17, 250]
    segs, mt, r0 = [], [0], 0
    for s, n in enumerate(counts):
        segs.append([r0, n, s, s])
        r0 += n
        mt.append(mt[-1] + (n + 127) // 128)
    lay = (torch.tensor(segs, dtype=torch.int32, device=dev), torch.tensor([len(segs)], dtype=torch.int32, device=dev),
           torch.tensor(mt, dtype=torch.int32, device=dev))
    A = torch.randn((r0, K), device=dev).to(torch.bfloat16)
    ready = torch.zeros(slots, dtype=torch.int32, device=dev)
    fetch_stream = torch.cuda.Stream()
    for epoch in (1, 2):
        W[n_home * N:].zero_()
        torch.cuda.synchronize()
        out = ops.grouped_gemm(A, W, N, lay, ops.HM_EPI_STORE, slot_ready=ready, ready_from_slot=n_home, epoch=epoch)
        for s in range(n_home, slots):
            ops.fetch_expert(W[s * N:(s + 1) * N], W_host[s], ready_flag=ready[s:], epoch=epoch, stream=fetch_stream)
        torch.cuda.synchronize()
        ref = []
        for s, n in enumerate(counts):
            ref.append(A[sum(counts[:s]):sum(counts[:s]) + n].float() @ W_host[s].to(dev).float().T)
        ref = torch.cat(ref).to(torch.bfloat16)
        assert torch.allclose(out.float(), ref.float(), atol=2e-2, rtol=2e-2)
        assert int(ready.min().item()) >= 0 and int(ready[n_home:].min().item()) == epoch


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_ep_block_single_rank_matches_local_block():
    """EP block on a 1-rank NCCL group (all_gather, all_to_all, EP layouts, pos-gather
    combine) is bit-identical to the single-process block."""
    import torch.distributed as dist

    from paper_2506_12417_b200.block import HarMoEnyBlock, MoEConfig
    from paper_2506_12417_b200.ep import EPHarMoEnyBlock

    dev = _cuda()
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(_free_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", torch.cuda.current_device()))
    try:
        kw = dict(d_model=256, num_experts=32, d_ff=256, top_k=4, activation="swiglu", eq_tokens=4)
        loc = HarMoEnyBlock.random(MoEConfig(**kw), seed=9, device=dev, zipf_s=1.0)
        ep = EPHarMoEnyBlock.random(MoEConfig(rank=0, world_size=1, **kw), seed=9, device=dev, zipf_s=1.0)
        x = torch.randn((640, 256), device=dev).to(torch.bfloat16)
        y1 = loc(x)
        y2 = ep(x)
        torch.cuda.synchronize()
        assert torch.equal(y1, y2)
        assert torch.equal(loc.stats.schedule, ep.stats.schedule)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("E,tiles,zero_frac", [(128, 128, 0.0), (16, 3, 0.3), (60, 17, 0.5), (1024, 9, 0.9),
                                               (8, 1, 0.0)])
def test_plan_single_gpu_matches_general_kernels(E, tiles, zero_frac):
    """The G=1 planner (one thread per expert) produces exactly what the general kernels do:
    hist_scan (m, tile offsets), schedule (S = m) and dispatch_layout (rows, plan-order segments,
    tile prefix, no fetches)."""
    from paper_2506_12417_b200 import ops

    dev = _cuda()
    rng = np.random.default_rng(E + tiles)
    th = rng.integers(0, 40, size=(tiles, E)) * (rng.random((tiles, E)) >= zero_frac)
    th[:, rng.integers(0, E)] += 7  # ties in n and a hot expert
    tile_hist = torch.from_numpy(th.astype(np.int32)).to(dev)
    home = torch.zeros(E, dtype=torch.int32, device=dev)
    p = ops.plan(home, 1, E, 32, True, ops.HM_LAYOUT_LOCAL, tile_hist=tile_hist, tiles_per_rank=tiles)
    hist, tile_off = ops.hist_scan(tile_hist, 1, tiles)
    S, iters, loads = ops.schedule(hist, home, 32, True)
    lay = ops.dispatch_layout(S, home, ops.HM_LAYOUT_LOCAL)
    torch.cuda.synchronize()
    assert torch.equal(p.m_all, hist) and torch.equal(p.tile_off, tile_off)
    assert torch.equal(p.S, S) and int(p.iters.item()) == 0 and torch.equal(p.loads, loads)
    n = int(lay.n_seg.item())
    assert int(p.layout.n_seg.item()) == n and int(p.layout.n_fetch.item()) == 0
    assert torch.equal(p.layout.segs[:n], lay.segs[:n])
    assert torch.equal(p.layout.mtile_prefix[: n + 1], lay.mtile_prefix[: n + 1])
    assert torch.equal(p.layout.slot_base, lay.slot_base)


@pytest.mark.parametrize("G,E,k,d,Tg,placement", [(2, 16, 4, 256, 384, "blocked"), (4, 32, 2, 512, 256, "round_robin"),
                                                  (8, 128, 8, 2048, 512, "blocked"), (1, 8, 2, 256, 200, "blocked")])
def test_ordered_push_matches_push_and_gates_ffn1(G, E, k, d, Tg, placement):
    """Expert-ordered dispatch (hm_plan_dispatch + hm_dispatch_push_ordered): every destination's
    receive buffer, row tags and pos equal the unordered push's, each destination's arrival counter
    of expert e ends at the rows of e it holds, and FFN1 gated by those counters (plain and launched
    with PDL right behind the last push) is bit-identical to the ungated FFN1."""
    from paper_2506_12417_b200 import ops

    dev = _cuda()
    gen = torch.Generator(device=dev).manual_seed(G * 100 + E)
    wg = torch.zeros((ops.e_pad(E), d), dtype=torch.bfloat16, device=dev)
    wg[:E] = (torch.randn((E, d), device=dev, generator=gen) * 0.05).to(torch.bfloat16)
    bias = torch.linspace(2.0, -2.0, E, device=dev)  # skewed routing: rebalancing moves buckets
    xs, routed, hists = [], [], []
    for g in range(G):
        x = torch.randn((Tg, d), device=dev, generator=gen).to(torch.bfloat16)
        idx, _, tile_hist, lrank = ops.router_topk(x, wg, bias, 1, Tg, k, True, E=E)
        hist, tile_off = ops.hist_scan(tile_hist, 1, (Tg + 127) // 128)
        xs.append(x)
        routed.append((idx, lrank, tile_off))
        hists.append(hist)
    m_all = torch.cat(hists).contiguous()
    home_np = orc.blocked_home(E, G) if placement == "blocked" else orc.round_robin_home(E, G)
    home = torch.from_numpy(home_np.astype(np.int32)).to(dev)
    cap = G * Tg * k
    rows_a = [torch.zeros((cap, d), dtype=torch.bfloat16, device=dev) for _ in range(G)]
    rows_b = [torch.zeros((cap, d), dtype=torch.bfloat16, device=dev) for _ in range(G)]
    tok_a = [torch.full((cap,), -1, dtype=torch.int32, device=dev) for _ in range(G)]
    tok_b = [torch.full((cap,), -1, dtype=torch.int32, device=dev) for _ in range(G)]
    arrive = torch.zeros((G, E), dtype=torch.int32, device=dev)
    ptrs = lambda ts: torch.tensor([t.data_ptr() for t in ts], dtype=torch.int64, device=dev)  # noqa: E731
    arrive_ptrs = torch.tensor([arrive[g].data_ptr() for g in range(G)], dtype=torch.int64, device=dev)
    order = torch.empty(Tg * k, dtype=torch.int32, device=dev)
    sync = torch.zeros(2, dtype=torch.int32, device=dev)
    plans = []
    for me in range(G):
        p, pl = ops.plan_dispatch(home, G, E, 4, True, me, m_all)
        p_ref = ops.plan(home, G, E, 4, True, ops.HM_LAYOUT_EP_EXPERT, me, m_all=m_all)
        ns = int(p_ref.layout.n_seg.item())
        for a, b in ((p.S, p_ref.S), (p.layout.slot_base, p_ref.layout.slot_base),
                     (p.layout.segs[:ns], p_ref.layout.segs[:ns]), (p.layout.n_seg, p_ref.layout.n_seg),
                     (p.layout.mtile_prefix[: ns + 1], p_ref.layout.mtile_prefix[: ns + 1])):
            assert torch.equal(a, b)
        idx, lrank, tile_off = routed[me]
        pos_a = torch.empty((Tg, k), dtype=torch.int32, device=dev)
        pos_b = torch.empty((Tg, k), dtype=torch.int32, device=dev)
        ops.dispatch_push(xs[me], idx, lrank, tile_off, p.S, p.layout.slot_base, None, me, ptrs(rows_a), ptrs(tok_a),
                          pos=pos_a)
        ops.dispatch_push_ordered(xs[me], idx, lrank, tile_off, p.S, p.layout.slot_base, pl, me, ptrs(rows_b),
                                  ptrs(tok_b), arrive_ptrs, order, sync, pos=pos_b)
        assert torch.equal(pos_a, pos_b)
        plans.append(p)
    torch.cuda.synchronize()
    S = plans[0].S.cpu().numpy()
    for dd in range(G):
        assert torch.equal(rows_a[dd], rows_b[dd]) and torch.equal(tok_a[dd], tok_b[dd])
        assert np.array_equal(arrive[dd].cpu().numpy(), S[:, :, dd].sum(axis=0))
    # FFN1 of destination G-1 gated by its arrival counters, vs ungated
    dd = G - 1
    lay = plans[dd].layout
    W = (torch.randn((E * 256, d), device=dev, generator=gen) * 0.05).to(torch.bfloat16)
    h_ref = ops.grouped_gemm(rows_a[dd], W, 256, lay, ops.HM_EPI_RELU)
    h1 = ops.grouped_gemm_arrive(rows_b[dd], W, 256, lay, ops.HM_EPI_RELU, arrive[dd], pdl=False)
    # overlapped: re-push every rank (counters restarted) with FFN1 launched right behind the last push
    arrive.zero_()
    for me in range(G):
        p, pl = ops.plan_dispatch(home, G, E, 4, True, me, m_all)
        idx, lrank, tile_off = routed[me]
        ops.dispatch_push_ordered(xs[me], idx, lrank, tile_off, p.S, p.layout.slot_base, pl, me, ptrs(rows_b),
                                  ptrs(tok_b), arrive_ptrs, order, sync)
    h2 = ops.grouped_gemm_arrive(rows_b[dd], W, 256, lay, ops.HM_EPI_RELU, arrive[dd], pdl=True)
    torch.cuda.synchronize()
    n = int(S[:, :, dd].sum())  # receive rows of dd (dense, expert-major)
    assert torch.equal(h1[:n], h_ref[:n]) and torch.equal(h2[:n], h_ref[:n])
