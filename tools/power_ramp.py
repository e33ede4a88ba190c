"""Throughput of back-to-back launches as a function of time since the stream
started: segments of --seg launches, one CUDA event between segments.  Shows
whether a short bench run is already inside the board-power plateau (early
segments faster than late ones) and which build is faster before / after it.

    python tools/power_ramp.py --config cfg3 [--segs 40 --seg 50 --idle 1.0]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2502_10831_b200 as ft  # noqa: E402
from paper_2502_10831_b200.configs import CONFIGS  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg3")
ap.add_argument("--segs", type=int, default=40)
ap.add_argument("--seg", type=int, default=50)
ap.add_argument("--idle", type=float, default=1.0)
ap.add_argument("--elements", type=int, default=0)
a = ap.parse_args()
w = CONFIGS[a.config]
n = a.elements or min(w.n, 1 << 30)
dt = torch.float32 if w.itemsize == 4 else torch.float64
# Buffers larger than L2 in total: rotate over copies when one batch fits in L2.
copies = max(1, -(-3 * 126 * 2**20 // (n * w.bytes_per_elem)))
xs = [ft.gen_inputs(n, dt, w.dist, w.lo, w.hi, w.seed) for _ in range(copies)]
outs = [{nm: torch.empty_like(xs[0]) for j, nm in enumerate(("sin", "cos", "tan")) if w.mask & (1 << j)}
        for _ in range(copies)]
mode = ft.SqrtMode()
k = 0


def step():
    global k
    i = k % copies
    k += 1
    if w.kind == 0:
        ft.proposed_eval(xs[i], w.mask, mode, out=outs[i])
    else:
        ft.taylor_eval(xs[i], w.n_terms, w.mask, out=outs[i])


for _ in range(20):
    step()
torch.cuda.synchronize()
time.sleep(a.idle)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(a.segs + 1)]
ev[0].record()
for s in range(a.segs):
    for _ in range(a.seg):
        step()
    ev[s + 1].record()
torch.cuda.synchronize()
ms = [ev[s].elapsed_time(ev[s + 1]) for s in range(a.segs)]
rate = [round(n * a.seg / (m / 1e3) / 1e9, 1) for m in ms]
t_end = []
acc = 0.0
for m in ms:
    acc += m
    t_end.append(round(acc, 1))
print(json.dumps({"config": a.config, "n": n, "launches_per_segment": a.seg, "copies": copies,
                  "segment_end_ms": t_end, "gelem_s": rate,
                  "lib": os.environ.get("FASTTRIG_B200_LIB", "default")}))
