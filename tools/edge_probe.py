import sys, torch, numpy as np
sys.path.insert(0, '.')
from paper_2506_12417_b200.block import HarMoEnyBlock, MoEConfig
from oracle import moe_oracle as orc
dev = torch.device('cuda')
def bits(t): return t.contiguous().view(torch.int16).cpu().numpy().view(np.uint16)
for (T, G, E, k, d, f, act) in [(1,1,16,2,256,256,'swiglu'), (3,1,16,4,256,256,'swiglu'), (130,2,16,2,256,256,'swiglu'),
                                 (8,4,8,8,256,256,'swiglu'), (257,1,60,4,128,256,'relu'), (0,1,16,2,256,256,'swiglu')]:
    cfg = MoEConfig(logical_ranks=G, eq_tokens=1, placement='blocked', d_model=d, num_experts=E, d_ff=f, top_k=k, activation=act)
    blk = HarMoEnyBlock.random(cfg, seed=1, device=dev, zipf_s=1.0, std=0.05)
    x = torch.randn((T, d), device=dev).to(torch.bfloat16)
    try:
        y = blk(x); torch.cuda.synchronize()
        print(T, G, E, k, 'ok', tuple(y.shape), float(y.float().abs().max()) if T else None)
    except Exception as e:
        print(T, G, E, k, 'ERR', type(e).__name__, e)
