"""Host<->device copy bandwidth from pinned memory (diagnostics for the e2e bound)."""
import torch

n = 64 * 1024 * 1024
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for _ in range(3):
    d.copy_(h, non_blocking=True); h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for name, fn in [("H2D", lambda: d.copy_(h, non_blocking=True)), ("D2H", lambda: h2.copy_(d2, non_blocking=True))]:
    a.record(); [fn() for _ in range(10)]; b.record(); torch.cuda.synchronize()
    print(f"{name}: {10 * n / a.elapsed_time(b) / 1e6:.1f} GB/s")
a.record()
for _ in range(10):
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
b.record(); torch.cuda.synchronize()
print(f"bidirectional: {20 * n / a.elapsed_time(b) / 1e6:.1f} GB/s total")
