"""Raw pinned host<->device copy bandwidth (the e2e ceiling)."""
import time
import torch
n = 1 << 28  # 2 GiB of f64
h = torch.empty(n, dtype=torch.float64, pin_memory=True)
d = torch.empty(n, dtype=torch.float64, device="cuda")
for name, fn in (("H2D", lambda: d.copy_(h, non_blocking=True)), ("D2H", lambda: h.copy_(d, non_blocking=True))):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    t = (time.perf_counter() - t0) / 3
    print(f"{name}: {n * 8 / t / 1e9:.1f} GB/s")
# both directions at once on two streams
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
h2 = torch.empty(n, dtype=torch.float64, pin_memory=True)
d2 = torch.empty(n, dtype=torch.float64, device="cuda")
torch.cuda.synchronize()
t0 = time.perf_counter()
with torch.cuda.stream(s1):
    d.copy_(h, non_blocking=True)
with torch.cuda.stream(s2):
    h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize()
t = time.perf_counter() - t0
print(f"bidirectional: {2 * n * 8 / t / 1e9:.1f} GB/s total")
