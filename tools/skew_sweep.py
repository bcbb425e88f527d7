"""BASELINE config 5: skew sweep (uniform -> Zipf s=1.5) x ranks {1,2,4,8} x rebalancing on/off.

Runs the real block in LOCAL mode (G logical ranks = G token shards on one GPU) so the
schedule is HarMoEny's schedule of G GPUs, and reports per config the max/mean per-GPU
token load (the <= 1.1 target), the scheduler's move count, and the block's tokens/s on
this one GPU.  Placement "blocked" (hot experts all homed on GPU 0).

    python tools/skew_sweep.py [workload] [q]  > profiles/r1_skew_sweep.jsonl
"""

import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_12417_b200.block import HarMoEnyBlock, MoEConfig  # noqa: E402

WL = {"qwen128": (2048, 768, 128, 8, "swiglu", 16384), "switch128": (768, 3072, 128, 1, "relu", 4096),
      "mixtral8": (4096, 14336, 8, 2, "swiglu", 16384)}


def timed(fn, it=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(it):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / it


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "qwen128"
    q = int(sys.argv[2]) if len(sys.argv) > 2 else 32
    d, f, E, k, act, T = WL[name]
    g = torch.Generator(device="cuda").manual_seed(1234)
    x = torch.randn((T, d), device="cuda", generator=g).to(torch.bfloat16)
    for s in (0.0, 0.5, 1.0, 1.5):
        for G in (1, 2, 4, 8):
            for policy in ("round_robin", "harmony", "even_split"):
                cfg = MoEConfig(d_model=d, d_ff=f, num_experts=E, top_k=k, activation=act, eq_tokens=q,
                                logical_ranks=G, placement="blocked", scheduling_policy=policy)
                blk = HarMoEnyBlock.random(cfg, seed=0, zipf_s=s)
                ms = timed(lambda: blk(x))
                loads = blk.stats.loads.double().cpu()
                rec = dict(workload=name, zipf_s=s, G=G, rebalance=policy == "harmony", policy=policy, q=q,
                           load_max_over_mean=round(float(loads.max() / loads.mean()), 4),
                           moves=int(blk.stats.iters.item()), block_ms_one_gpu=round(ms, 4),
                           tokens_per_s_one_gpu=round(T / ms * 1e3))
                print(json.dumps(rec), flush=True)
                del blk
                torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
