"""Single-process check of the in-GEMM K6 fetch pairs with a bounded cache: experts 2..6 fetched
through C cache slots while FFN-like GEMMs (phase 1: W_in, phase 2: W_out) consume them."""
import sys, time, torch
sys.path.insert(0, '.')
from paper_2506_12417_b200 import ops, _lib
dev = torch.device('cuda')
N, K, n_home = 512, 256, 2
C = int(sys.argv[1]) if len(sys.argv) > 1 else 1
counts = [300, 200, 129, 64, 17, 250, 1000]
E = len(counts)
print("resident pairs", [_lib.load().hm_gemm_resident_pairs(e, g) for e in (0, 1, 2) for g in (0, 1)], flush=True)
segs, mt, r0 = [], [0], 0
for e, n in enumerate(counts):
    ws = e if e < n_home else n_home + (e - n_home) % C
    segs.append([r0, n, ws, e]); r0 += n; mt.append(mt[-1] + (n + 127) // 128)
i32 = dict(dtype=torch.int32, device=dev)
segs_t, nseg_t, mt_t = torch.tensor(segs, **i32), torch.tensor([len(segs)], **i32), torch.tensor(mt, **i32)
fetch = list(range(n_home, E))
fetch_t = torch.tensor(fetch + [0] * (E - len(fetch)), **i32)
nf = torch.tensor([len(fetch)], **i32)
lay = ops.Layout(None, segs_t, nseg_t, mt_t, fetch_t, nf)
A = torch.randn((r0, K), device=dev).to(torch.bfloat16)
Win = (torch.randn((E, N, K), device=dev) * 0.05).to(torch.bfloat16)
Wout = (torch.randn((E, N, K), device=dev) * 0.05).to(torch.bfloat16)
src_in = torch.tensor([Win[e].data_ptr() for e in range(E)], dtype=torch.int64, device=dev)
src_out = torch.tensor([Wout[e].data_ptr() for e in range(E)], dtype=torch.int64, device=dev)
W1 = torch.zeros(((n_home + C) * N, K), dtype=torch.bfloat16, device=dev)
W2 = torch.zeros(((n_home + C) * N, K), dtype=torch.bfloat16, device=dev)
W1[:n_home * N] = Win[:n_home].reshape(-1, K)
W2[:n_home * N] = Wout[:n_home].reshape(-1, K)
lay_all = (torch.tensor([[r[0], r[1], r[3], r[3]] for r in segs], **i32), nseg_t, mt_t)
ref1 = ops.grouped_gemm(A, Win.reshape(-1, K), N, lay_all, ops.HM_EPI_STORE)
ref2 = ops.grouped_gemm(A, Wout.reshape(-1, K), N, lay_all, ops.HM_EPI_STORE)
ready_in = torch.zeros(E, **i32); ready_out = torch.zeros(E, **i32)
done_in = torch.zeros(E, **i32); done_out = torch.zeros(E, **i32)
cnt = torch.zeros(2 * E, **i32)
for epoch in (1, 2, 3):
    W1[n_home * N:].zero_(); W2[n_home * N:].zero_(); done_in.zero_(); done_out.zero_()
    fp1 = ops.fetch_plan(fetch_t, nf, src_in, src_out, W1, W2, N * K * 2, N * K * 2, n_home, C, ready_in, ready_out, cnt, epoch, 1)
    o1 = ops.grouped_gemm(A, W1, N, lay, ops.HM_EPI_STORE, slot_ready=ready_in, ready_from_slot=n_home, epoch=epoch,
                          slot_done=done_in, fetch=fp1)
    fp2 = ops.fetch_plan(fetch_t, nf, src_in, src_out, W1, W2, N * K * 2, N * K * 2, n_home, C, ready_in, ready_out, cnt, epoch, 2)
    o2 = ops.grouped_gemm(A, W2, N, lay, ops.HM_EPI_STORE, slot_ready=ready_out, ready_from_slot=n_home, epoch=epoch,
                          slot_done=done_out, fetch=fp2)
    ev = torch.cuda.Event(); ev.record(); t0 = time.time()
    while not ev.query():
        time.sleep(0.01)
        if time.time() - t0 > 20: print("HANG", flush=True); sys.exit(1)
    torch.cuda.synchronize()
    print('C', C, 'epoch', epoch, 'ffn1', torch.equal(o1, ref1), 'ffn2', torch.equal(o2, ref2), 'done', done_in.tolist(), done_out.tolist(),
          'ready', ready_in.tolist(), ready_out.tolist(), flush=True)
