"""Expert-parallel plumbing on CPU with the gloo backend (world sizes 2 and 4).

Every rank runs the EP protocol of paper_2506_12417_b200/ep.py with the
product's host-side plumbing (ep_counts, exchange_metadata, exchange_tokens,
return_tokens) and the oracle standing in for the device kernels (this is a
CPU test: the kernels themselves are covered by the -m gpu suite).  The
result on every rank must equal the single-process oracle block on that
rank's token slice, and every rank must derive the identical schedule.
"""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _problem(seed=3, T=96, d=64, E=8, f=128, k=2):
    from oracle import moe_oracle as orc

    rng = np.random.default_rng(seed)
    x = orc.f32_to_bf16(rng.standard_normal((T, d)).astype(np.float32))
    wg = orc.f32_to_bf16((rng.standard_normal((E, d)) / np.sqrt(d)).astype(np.float32))
    w1 = orc.f32_to_bf16((rng.standard_normal((E, f, d)) * 0.1).astype(np.float32))
    w3 = orc.f32_to_bf16((rng.standard_normal((E, f, d)) * 0.1).astype(np.float32))
    w2 = orc.f32_to_bf16((rng.standard_normal((E, d, f)) * 0.1).astype(np.float32))
    bias = np.log(np.arange(1, E + 1, dtype=np.float64) ** -1.5).astype(np.float32)
    return x, wg, w1, w2, w3, bias, k


def _worker(rank, world, port, q, placement, out_q):
    import sys

    sys.path.insert(0, REPO)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import moe_oracle as orc
        from paper_2506_12417_b200.ep import ep_counts, exchange_metadata, exchange_tokens, return_tokens

        x, wg, w1, w2, w3, bias, k = _problem()
        T, d = x.shape
        E = wg.shape[0]
        Tg = T // world
        home = orc.blocked_home(E, world) if placement == "blocked" else orc.round_robin_home(E, world)
        xl = x[rank * Tg:(rank + 1) * Tg]
        _, idx, w = orc.router(xl, wg, bias, k, True)
        # step 2: metadata exchange (product plumbing)
        hist = torch.from_numpy(orc.histogram(idx, E)).reshape(1, E)
        m_all = exchange_metadata(hist).numpy()
        # step 3: replicated schedule
        S, iters = orc.schedule(m_all, home, q, True)
        # step 4: scatter into the dest-major send buffer, all_to_all
        pos = orc.ep_send_positions(idx, S, rank)
        send_counts, recv_counts = ep_counts(S, rank)
        xf = orc.bf16_to_f32(xl)
        send = np.zeros((Tg * k, d), np.float32)
        for j in range(k):
            send[pos[:, j]] = xf
        recv = exchange_tokens(torch.from_numpy(send), send_counts, recv_counts).numpy()
        # step 5: experts over the receive segments (expert, source) in plan order
        yr = np.zeros((max(sum(recv_counts), 1), d), np.float32)
        for (r0, n, _wslot, e) in orc.ep_recv_segments(S, home, rank):
            yr[r0:r0 + n] = orc.expert_ffn(recv[r0:r0 + n], w1[e], w2[e], "swiglu", w3[e])
        # step 6: gather back + combine in slot order
        ys = return_tokens(torch.from_numpy(yr), send_counts, recv_counts).numpy()
        acc = np.zeros((Tg, d), np.float32)
        for j in range(k):
            acc = (acc + w[:, j:j + 1] * ys[pos[:, j]]).astype(np.float32)
        out_q.put((rank, orc.f32_to_bf16(acc), S, iters, np.asarray(send_counts), np.asarray(recv_counts)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,q,placement", [(2, 1, "blocked"), (2, 8, "round_robin"), (4, 1, "blocked")])
def test_ep_protocol_matches_single_process(world, q, placement):
    from oracle import moe_oracle as orc

    ctx = mp.get_context("spawn")
    out_q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, placement, out_q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, y, S, iters, sc, rc = out_q.get(timeout=240)
        res[r] = (y, S, iters, sc, rc)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    x, wg, w1, w2, w3, bias, k = _problem()
    y_ref, _, _, _ = orc.moe_block(x, wg, bias, w1, w2, k, "swiglu", True, w3)
    Tg = x.shape[0] // world
    S0 = res[0][1]
    for r in range(world):
        y, S, iters, sc, rc = res[r]
        assert np.array_equal(S, S0), "schedules must be replicated bit-identically"
        assert sc.sum() == Tg * k
        yr = orc.bf16_to_f32(y_ref[r * Tg:(r + 1) * Tg]).astype(np.float64)
        yg = orc.bf16_to_f32(y).astype(np.float64)
        assert np.all(np.abs(yg - yr) <= 1e-2 + 2e-2 * np.abs(yr))
    # the rebalanced schedule actually moved work between ranks (skewed routing)
    loads = S0.sum(axis=(0, 1))
    if q == 1:
        assert loads.max() / loads.mean() <= 1.1
