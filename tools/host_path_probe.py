"""Host-pointer path throughput: pinned vs pageable buffers (fused S/C/T), f64 and f32."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2502_10831_b200 as ft
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 26
for tdt, ndt in ((torch.float64, np.float64), (torch.float32, np.float32)):
    es = np.dtype(ndt).itemsize
    for kind in ("pageable", "pinned"):
        if kind == "pinned":
            x = torch.empty(n, dtype=tdt, pin_memory=True).numpy()
            outs = {k: torch.empty(n, dtype=tdt, pin_memory=True).numpy() for k in ("sin", "cos", "tan")}
        else:
            x = np.empty(n, ndt); outs = {k: np.empty(n, ndt) for k in ("sin", "cos", "tan")}
        x[:] = np.linspace(-1e3, 1e3, n)
        ft.proposed_batch(x, 7, out=outs)
        ts = []
        for _ in range(3):
            t0 = time.perf_counter(); ft.proposed_batch(x, 7, out=outs); ts.append(time.perf_counter() - t0)
        t = min(ts)
        print(json.dumps({"dtype": np.dtype(ndt).name, "buffers": kind, "n": n, "ms": round(t * 1e3, 1),
                          "gelem_s": round(n / t / 1e9, 3), "host_device_gbs": round(4 * es * n / t / 1e9, 1)}))
