"""Debug: 2 EP ranks on one GPU (gloo), compare with the single-process block per variant."""
import os, sys, socket
import numpy as np
import torch, torch.distributed as dist, torch.multiprocessing as mp
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
KW = dict(d_model=256, num_experts=16, d_ff=256, top_k=2, activation="swiglu", eq_tokens=2, placement="blocked")
T = 1024

def worker(rank, world, port, variant, q):
    sys.path.insert(0, REPO)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2506_12417_b200.block import MoEConfig
    from paper_2506_12417_b200.ep import EPHarMoEnyBlock
    pol, src = variant
    cfg = MoEConfig(rank=rank, world_size=world, fetch_source=src, scheduling_policy=pol, **KW)
    blk = EPHarMoEnyBlock.random(cfg, seed=7, device="cuda", zipf_s=1.3, std=0.05)
    g = torch.Generator(device="cuda").manual_seed(99)
    x = torch.randn((T, 256), device="cuda", generator=g).to(torch.bfloat16)
    Tg = T // world
    y = blk(x[rank * Tg:(rank + 1) * Tg].contiguous())
    torch.cuda.synchronize()
    st = blk.stats
    q.put((rank, y.cpu().view(torch.int16).numpy(), st.extras["topk_idx"].cpu().numpy(), st.schedule.cpu().numpy(),
           st.extras["n_fetch"], st.extras["layout"].segs[: int(st.extras["layout"].n_seg.item())].cpu().numpy(),
           blk.home_np))
    dist.destroy_process_group()

def main():
    from paper_2506_12417_b200.block import HarMoEnyBlock, MoEConfig
    ref = HarMoEnyBlock.random(MoEConfig(**KW), seed=7, device="cuda", zipf_s=1.3, std=0.05)
    g = torch.Generator(device="cuda").manual_seed(99)
    x = torch.randn((T, 256), device="cuda", generator=g).to(torch.bfloat16)
    y_ref = ref(x).cpu().view(torch.int16).numpy()
    idx_ref = ref.stats.extras["topk_idx"].cpu().numpy()
    for variant in [("round_robin", "host"), ("harmony", "host"), ("harmony", "peer")]:
        ctx = mp.get_context("spawn"); q = ctx.Queue(); port = socket.socket(); port.bind(("127.0.0.1", 0)); pn = port.getsockname()[1]; port.close()
        ps = [ctx.Process(target=worker, args=(r, 2, pn, variant, q)) for r in range(2)]
        [p.start() for p in ps]
        res = {}
        for _ in range(2):
            r, y, idx, S, nf, segs, home = q.get(timeout=120); res[r] = (y, idx, S, nf, segs, home)
        [p.join() for p in ps]
        for r in range(2):
            y, idx, S, nf, segs, home = res[r]
            sl = slice(r * 512, (r + 1) * 512)
            eq_rows = np.all(y == y_ref[sl], axis=1)
            bad_t = np.nonzero(~eq_rows)[0]
            bad_experts = np.unique(idx[bad_t]) if len(bad_t) else []
            print(variant, "rank", r, "rows equal", eq_rows.mean(), "idx equal", np.array_equal(idx, idx_ref[sl]), "n_fetch", nf,
                  "bad experts", list(bad_experts)[:16], "home", list(home))
            if r == 1: print("  segs r1", segs.tolist()[:20])
        print("  S[:,:,1] rows", res[0][2][:, :, 1].tolist())

if __name__ == "__main__":
    main()
