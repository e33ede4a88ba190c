"""Per-launch K1/K2 time without the sustained power cap: idle 2 s, then time
single launches with CUDA events (min / median of --reps).  Prints one JSON line.

    python tools/burst.py --config cfg2 [--reps 5]
"""
import argparse
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2502_10831_b200 as ft  # noqa: E402
from paper_2502_10831_b200.configs import CONFIGS  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg2")
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--mode", default="fisr1", choices=["fisr1", "fisr2", "fisr3", "exact"])
a = ap.parse_args()
w = CONFIGS[a.config]
n = min(w.n, 1 << 30)
dt = torch.float32 if w.itemsize == 4 else torch.float64
x = ft.gen_inputs(n, dt, w.dist, w.lo, w.hi, w.seed)
out = {nm: torch.empty_like(x) for j, nm in enumerate(("sin", "cos", "tan")) if w.mask & (1 << j)}


mode = {"fisr1": ft.SqrtMode(), "fisr2": ft.SqrtMode.fisr(2), "fisr3": ft.SqrtMode.fisr(3),
        "exact": ft.SqrtMode.exact()}[a.mode]


def step():
    if w.kind == 0:
        ft.proposed_eval(x, w.mask, mode, out=out)
    else:
        ft.taylor_eval(x, w.n_terms, w.mask, out=out)


step()
torch.cuda.synchronize()
times = []
for _ in range(a.reps):
    time.sleep(2.0)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    step()
    e1.record()
    torch.cuda.synchronize()
    times.append(e0.elapsed_time(e1))
ms = min(times)
print(json.dumps({"config": a.config, "mode": a.mode, "n": n, "burst_ms_min": ms, "burst_ms_median": statistics.median(times),
                  "gelem_s": n / (ms / 1e3) / 1e9, "gbs": w.bytes_per_elem * n / (ms / 1e3) / 1e9}))
