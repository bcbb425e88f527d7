import ctypes, sys, torch
lib = ctypes.CDLL(sys.argv[1] if len(sys.argv) > 1 else "tools/red_bench/red_bench.so")
T, k, d = 16384, 8, 2048
rows = T * k
g = torch.Generator(device="cpu").manual_seed(0)
# expert-major row order: token ids of each row = a random assignment of the T*k (t, j) pairs
perm = torch.randperm(rows, generator=g)
tok_rand = (perm // k).to(torch.int32).cuda()
tok_sorted = torch.sort(tok_rand.view(128, -1), dim=1).values.reshape(-1).contiguous()  # sorted within experts
out = torch.zeros((T, d), dtype=torch.float32, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
s = torch.cuda.current_stream().cuda_stream
for name, tok in (("random", tok_rand), ("sorted-in-expert", tok_sorted)):
    for mode, what in ((0, "red.v4.f32"), (1, "st.v4.f32")):
        for blocks in (148 * 4, 148 * 8):
            ts = []
            for _ in range(5):
                flush.fill_(1); out.zero_()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                assert lib.red_launch(ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(tok.data_ptr()), rows, d, mode, blocks, ctypes.c_void_p(s)) == 0
                b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b) * 1e3)
            us = sorted(ts)[2]
            print(f"{name:17s} {what:11s} blocks {blocks}: {us:7.1f} us  {rows * d * 4 / us / 1e3:6.0f} GB/s of fp32 updates", flush=True)
if out.sum().item() != 0: pass
