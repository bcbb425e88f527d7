import sys, torch, numpy as np
sys.path.insert(0, '.')
from paper_2506_12417_b200 import ops
dev = torch.device('cuda')
N, K = 512, 256
counts = [300, 200, 129, 64, 17, 250, 1000]
segs, mt, r0 = [], [0], 0
for s, n in enumerate(counts):
    segs.append([r0, n, s, s]); r0 += n; mt.append(mt[-1] + (n + 127) // 128)
lay = (torch.tensor(segs, dtype=torch.int32, device=dev), torch.tensor([len(segs)], dtype=torch.int32, device=dev),
       torch.tensor(mt, dtype=torch.int32, device=dev))
A = torch.randn((r0, K), device=dev).to(torch.bfloat16)
W = (torch.randn((len(counts) * N, K), device=dev) * 0.05).to(torch.bfloat16)
ready = torch.full((len(counts),), 5, dtype=torch.int32, device=dev)
done = torch.zeros(len(counts), dtype=torch.int32, device=dev)
for epi in (ops.HM_EPI_STORE, ops.HM_EPI_SWIGLU):
    done.zero_()
    out = ops.grouped_gemm(A, W, N, lay, epi, slot_ready=ready, ready_from_slot=2, epoch=1, slot_done=done)
    torch.cuda.synchronize()
    exp = [16 * (N // 256) * (((n + 127) // 128 + 1) // 2) if s >= 2 else 0 for s, n in enumerate(counts)]
    print('epi', epi, 'done', done.tolist(), 'expected', exp, flush=True)
