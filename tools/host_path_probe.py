"""Host-pointer path throughput: pinned vs pageable buffers (f64, fused S/C/T)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2502_10831_b200 as ft
n = 1 << 26
for kind in ("pageable", "pinned"):
    if kind == "pinned":
        x = torch.empty(n, dtype=torch.float64, pin_memory=True).numpy()
        outs = {k: torch.empty(n, dtype=torch.float64, pin_memory=True).numpy() for k in ("sin", "cos", "tan")}
    else:
        x = np.empty(n); outs = {k: np.empty(n) for k in ("sin", "cos", "tan")}
    x[:] = np.linspace(-1e3, 1e3, n)
    ft.proposed_batch(x, 7, out=outs)
    ts = []
    for _ in range(3):
        t0 = time.perf_counter(); ft.proposed_batch(x, 7, out=outs); ts.append(time.perf_counter() - t0)
    t = min(ts)
    print(f"{kind:9s} n={n} {t*1e3:8.1f} ms  {n/t/1e9:6.3f} Gelem/s  {32*n/t/1e9:6.1f} GB/s host<->device")
