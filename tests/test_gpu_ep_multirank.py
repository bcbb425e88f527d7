"""Expert parallelism with 2 real ranks on the GPU box's single B200.

NCCL refuses two ranks on one device, so the two processes talk over gloo (the EP
exchange helpers stage CUDA tensors through host memory for non-NCCL groups).  Every
device-side piece of the EP path runs for real: EP layout (send/receive), the send-buffer
scatter, the grouped GEMM over (expert, source) segments, the position-gather combine,
and K6 - experts homed on the other rank are fetched through CUDA IPC pointers (or
pinned host memory) on the fetch stream while the GEMM waits on per-slot ready flags.
Each rank's output must be bit-identical to the single-process block on the same tokens.
"""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

pytestmark = pytest.mark.gpu
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KW = dict(d_model=256, num_experts=16, d_ff=256, top_k=2, activation="swiglu", eq_tokens=2, placement="blocked")
T = 1024


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, fetch_source, transport, out_q, cache=0):
    import sys

    sys.path.insert(0, REPO)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2506_12417_b200.block import MoEConfig
        from paper_2506_12417_b200.ep import EPHarMoEnyBlock

        cfg = MoEConfig(rank=rank, world_size=world, fetch_source=fetch_source, transport=transport.split("-")[0],
                        max_tokens_per_rank=T // world, async_fetch="sync" not in transport,
                        expert_cache_size=cache, overlap_dispatch="-ov" in transport, **KW)
        blk = EPHarMoEnyBlock.random(cfg, seed=7, device="cuda", zipf_s=1.3, std=0.05)
        g = torch.Generator(device="cuda").manual_seed(99)
        x = torch.randn((T, 256), device="cuda", generator=g).to(torch.bfloat16)
        Tg = T // world
        xl = x[rank * Tg:(rank + 1) * Tg].contiguous()
        outs = []
        if "graph" in transport:
            cap = blk.capture(Tg)  # every rank captures; replays synchronise through the flags
            cap.x.copy_(xl)
            for _ in range(3):
                outs.append(cap.replay().clone().cpu())
        else:
            for _ in range(3):  # later forwards re-use the fetch slots and the peer flags
                outs.append(blk(xl).cpu())
        torch.cuda.synchronize()
        out_q.put((rank, outs[0].view(torch.int16).numpy(), outs[2].view(torch.int16).numpy(),
                   blk.stats.schedule.cpu().numpy(), int(blk.stats.extras["layout"].n_fetch.item())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("fetch_source,transport,world,cache", [
    ("peer", "nccl", 2, 0), ("host", "nccl", 2, 0), ("peer", "p2p", 2, 0), ("host", "p2p", 2, 0),
    ("peer", "p2p", 4, 0), ("peer", "p2p-graph", 2, 0), ("host", "p2p-graph", 4, 0), ("peer", "nccl-sync", 2, 0),
    ("peer", "p2p-sync", 2, 0), ("peer", "p2p-ov", 2, 0), ("host", "p2p-graph-ov", 4, 0), ("peer", "p2p-ov", 4, 1),
    # bounded expert cache (engine.py:204-275 overwrite semantics): fewer slots than fetches
    ("peer", "nccl", 2, 1), ("host", "nccl", 4, 1), ("peer", "p2p", 2, 1), ("host", "p2p", 4, 1),
    ("peer", "p2p-graph", 2, 1), ("peer", "p2p-graph", 4, 1), ("peer", "nccl", 4, 1)])
def test_ep_ranks_one_gpu_bit_identical(fetch_source, transport, world, cache):
    """transport "nccl": exchanges through the process group (gloo here, host-staged);
    transport "p2p": one-sided pushes into the other ranks' IPC-mapped buffers + stream flags,
    no collective and no host round trip inside the forward; "-ov": the expert-ordered dispatch
    overlapped with FFN1 (per-expert arrival counters, PDL) instead of the unordered push + token
    flag exchange.  "-sync": the synchronous-loading
    ablation (expert fetches in stream order ahead of FFN1, SimFlags.async_loading_enabled=False).
    cache > 0: expert_cache_size slots, fewer than the experts a rank fetches, so fetches reuse
    slots as the GEMMs finish their occupants; outputs stay bit-identical."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2506_12417_b200.block import HarMoEnyBlock, MoEConfig

    ctx = mp.get_context("spawn")
    out_q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, fetch_source, transport, out_q, cache))
             for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    try:
        for _ in range(world):
            r, y0, y1, S, n_fetch = out_q.get(timeout=120)
            res[r] = (y0, y1, S, n_fetch)
        for p in procs:
            p.join(timeout=60)
            assert p.exitcode == 0
    finally:
        for p in procs:  # a rank stuck on a flag must not outlive the test
            if p.is_alive():
                p.kill()
    # single-process reference on the full batch (same weights / routing; G=1)
    ref = HarMoEnyBlock.random(MoEConfig(**KW), seed=7, device="cuda", zipf_s=1.3, std=0.05)
    g = torch.Generator(device="cuda").manual_seed(99)
    x = torch.randn((T, 256), device="cuda", generator=g).to(torch.bfloat16)
    y_ref = ref(x).cpu().view(torch.int16).numpy()
    Tg = T // world
    for r in range(1, world):
        assert np.array_equal(res[0][2], res[r][2]), "replicated schedules differ"
    assert sum(res[r][3] for r in range(world)) > 0, "the skewed schedule should make some rank fetch experts"
    if cache:
        assert max(res[r][3] for r in range(world)) > cache, "some rank must fetch more experts than it has slots"
    for r in range(world):
        y0, y1, _, _ = res[r]
        assert np.array_equal(y0, y_ref[r * Tg:(r + 1) * Tg])
        assert np.array_equal(y1, y0)


def _fallback_worker(rank, world, port, out_q, fail_at="hm_ipc_open"):
    import sys

    sys.path.insert(0, REPO)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2506_12417_b200 import _lib
        from paper_2506_12417_b200.block import MoEConfig
        from paper_2506_12417_b200.ep import EPHarMoEnyBlock, PeerAccessError

        if rank == 1:  # this rank cannot map its peer's memory
            real_check = _lib.check

            def failing_check(rc, what):
                if what == fail_at:
                    raise RuntimeError("injected: peer mapping refused")
                return real_check(rc, what)

            _lib.check = failing_check
        cfg = MoEConfig(rank=rank, world_size=world, transport="p2p", max_tokens_per_rank=T // world, **KW)
        raised = False
        try:
            EPHarMoEnyBlock.random(cfg, seed=7, device="cuda", zipf_s=1.3, std=0.05)
        except PeerAccessError:
            raised = True
        cfg = MoEConfig(rank=rank, world_size=world, transport="nccl", fetch_source="host",
                        max_tokens_per_rank=T // world, **KW)
        blk = EPHarMoEnyBlock.random(cfg, seed=7, device="cuda", zipf_s=1.3, std=0.05)
        g = torch.Generator(device="cuda").manual_seed(99)
        x = torch.randn((T, 256), device="cuda", generator=g).to(torch.bfloat16)
        Tg = T // world
        y = blk(x[rank * Tg:(rank + 1) * Tg].contiguous()).cpu()
        out_q.put((rank, raised, y.view(torch.int16).numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("fail_at", ["hm_ipc_open", "hm_ipc_get_handle"])
def test_peer_access_failure_is_collective(fail_at):
    """A rank that cannot export or map peer memory makes EVERY rank raise PeerAccessError at the
    same point, so all of them can rebuild with the NCCL transport + host fetch (what bench.py
    does) - no rank is left waiting in a collective."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2506_12417_b200.block import HarMoEnyBlock, MoEConfig

    world = 2
    ctx = mp.get_context("spawn")
    out_q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_fallback_worker, args=(r, world, port, out_q, fail_at)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    try:
        for _ in range(world):
            r, raised, y = out_q.get(timeout=120)
            res[r] = (raised, y)
        for p in procs:
            p.join(timeout=60)
            assert p.exitcode == 0
    finally:
        for p in procs:
            if p.is_alive():
                p.kill()
    assert res[0][0] and res[1][0], "both ranks must see the failure"
    ref = HarMoEnyBlock.random(MoEConfig(**KW), seed=7, device="cuda", zipf_s=1.3, std=0.05)
    g = torch.Generator(device="cuda").manual_seed(99)
    x = torch.randn((T, 256), device="cuda", generator=g).to(torch.bfloat16)
    y_ref = ref(x).cpu().view(torch.int16).numpy()
    Tg = T // world
    for r in range(world):
        assert np.array_equal(res[r][1], y_ref[r * Tg:(r + 1) * Tg])

