"""2 EP ranks on one GPU, bounded cache: print layouts and watch the done counters."""
import os, sys, socket, time
import torch, torch.distributed as dist, torch.multiprocessing as mp
REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
KW = dict(d_model=256, num_experts=16, d_ff=256, top_k=2, activation="swiglu", eq_tokens=2, placement="blocked")
T = 1024

def worker(rank, world, port, transport, cache):
    sys.path.insert(0, REPO)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2506_12417_b200.block import MoEConfig
    from paper_2506_12417_b200.ep import EPHarMoEnyBlock
    cfg = MoEConfig(rank=rank, world_size=world, transport=transport, max_tokens_per_rank=T // world,
                    expert_cache_size=cache, **KW)
    blk = EPHarMoEnyBlock.random(cfg, seed=7, device="cuda", zipf_s=1.3, std=0.05)
    print(rank, 'n_home', blk.n_home, 'n_cache', blk.n_cache, 'bounded', blk.bounded, 'reserve', blk.reserve_sms, flush=True)
    g = torch.Generator(device="cuda").manual_seed(99)
    x = torch.randn((T, 256), device="cuda", generator=g).to(torch.bfloat16)
    Tg = T // world
    xl = x[rank * Tg:(rank + 1) * Tg].contiguous()
    y = blk(xl)
    ev = torch.cuda.Event(); ev.record()
    t0 = time.time()
    while not ev.query() and time.time() - t0 < 4:
        time.sleep(0.05)
    lay = blk.stats.extras['layout']
    s2 = torch.cuda.Stream()
    with torch.cuda.stream(s2):
        vals = [t.to('cpu', non_blocking=True) for t in (lay.segs, lay.n_seg, lay.fetch, lay.n_fetch, blk.done_in, blk.done_out, blk.ready_in, blk.ready_out, lay.mtile_prefix)]
    s2.synchronize()
    segs, nseg, fetch, nf, di, do, ri, ro, mp_ = vals
    n = int(nseg[0]); f = int(nf[0])
    print(rank, 'completed' if ev.query() else 'HUNG', 'segs', segs[:n].tolist(), 'fetch', fetch[:f].tolist(),
          'done_in', di.tolist(), 'done_out', do.tolist(), 'ready_in', ri.tolist(), 'ready_out', ro.tolist(), 'mp', mp_[:n+1].tolist(), flush=True)
    os._exit(0)

if __name__ == '__main__':
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]
    world, transport, cache = int(sys.argv[1]), sys.argv[2], int(sys.argv[3])
    ctx = mp.get_context('spawn')
    ps = [ctx.Process(target=worker, args=(r, world, port, transport, cache)) for r in range(world)]
    [p.start() for p in ps]
    [p.join(60) for p in ps]
    [p.kill() for p in ps if p.is_alive()]
