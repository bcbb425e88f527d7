"""HBM read bandwidth of TMA weight streaming (grouped-GEMM box pattern, no MMA)."""
import ctypes, sys, torch
lib = ctypes.CDLL("tools/stream_bench/stream_bench.so")
K = int(sys.argv[1]) if len(sys.argv) > 1 else 768
rows = 128 * 3072 * 768 // K  # 604 MB of bf16
W = torch.empty((rows, K), dtype=torch.bfloat16, device="cuda").normal_()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
s = torch.cuda.current_stream().cuda_stream
def run(box, stages, grid, hint):
    ts = []
    for _ in range(5):
        flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        rc = lib.stream_launch(ctypes.c_void_p(W.data_ptr()), ctypes.c_long(rows), K, box, stages, grid, hint, ctypes.c_void_p(s))
        b.record(); torch.cuda.synchronize(); assert rc == 0, rc
        ts.append(a.elapsed_time(b) * 1e3)
    us = sorted(ts)[2]
    return us, rows * K * 2 / us / 1e3
print(f"K={K}: {rows*K*2/1e6:.0f} MB")
for hint in (0, 1, 2):
    for box in (128, 256):
        for stages in (4, 6, 8, 12):
            if stages * box * 128 > 200_000: continue
            for grid in (148, 296):
                if grid == 296 and stages * box * 128 > 100_000: continue
                us, gbs = run(box, stages, grid, hint)
                print(f"hint {['evict_first','normal','evict_last'][hint]:11s} box {box} stages {stages:2d} grid {grid}: {us:7.1f} us {gbs:6.0f} GB/s", flush=True)
# plain copy reference
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
dst = torch.empty_like(W)
for _ in range(3):
    flush.fill_(1); a.record(); dst.copy_(W); b.record(); torch.cuda.synchronize()
us = a.elapsed_time(b) * 1e3
print(f"torch copy: {us:.1f} us, {2*rows*K*2/us/1e3:.0f} GB/s (read+write)")
