import os, sys, torch
sys.path.insert(0, '.')
from paper_2506_12417_b200 import ops
T, d, E, k = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
x = torch.randn((T, d), device="cuda").to(torch.bfloat16)
wg = (torch.randn((ops.e_pad(E), d), device="cuda") * 0.02).to(torch.bfloat16)
for _ in range(4):
    ops.router_topk(x, wg, None, 1, T, k, k > 1, E=E)
torch.cuda.synchronize()
