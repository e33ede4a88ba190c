"""Determinism soak: every config's kernel launched back to back for --seconds,
its outputs compared bit for bit with the first launch's every --every launches
(under the sustained power cap, clocks moving).  One JSON line per config.

    python tools/soak.py --seconds 30
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
ap.add_argument("--seconds", type=float, default=30.0)
ap.add_argument("--every", type=int, default=25)
ap.add_argument("--configs", default="cfg2,cfg1,cfg3,cfg4_f32,cfg4_f64,cfg5")
a = ap.parse_args()
for name in a.configs.split(","):
    w = CONFIGS[name]
    n = min(w.n, 1 << 28)
    dt = torch.float32 if w.itemsize == 4 else torch.float64
    x = ft.gen_inputs(n, dt, w.dist, w.lo, w.hi, w.seed)
    names = [nm for j, nm in enumerate(("sin", "cos", "tan")) if w.mask & (1 << j)]
    out = {nm: torch.empty_like(x) for nm in names}
    mode = ft.SqrtMode()

    def step():
        if w.kind == 0:
            ft.proposed_eval(x, w.mask, mode, out=out)
        else:
            ft.taylor_eval(x, w.n_terms, w.mask, out=out)

    step()
    torch.cuda.synchronize()
    first = {nm: o.view(torch.int32 if w.itemsize == 4 else torch.int64).clone() for nm, o in out.items()}
    launches = checks = bad = 0
    t0 = time.time()
    while time.time() - t0 < a.seconds:
        for _ in range(a.every):
            step()
        launches += a.every
        for nm, o in out.items():
            checks += 1
            bad += int(not torch.equal(o.view(first[nm].dtype), first[nm]))
        for o in out.values():
            o.zero_()
    torch.cuda.synchronize()
    print(json.dumps({"config": name, "elements": n, "launches": launches, "output_comparisons": checks,
                      "mismatching_comparisons": bad, "seconds": round(time.time() - t0, 1)}), flush=True)
    del x, out, first
    torch.cuda.empty_cache()
