"""f32 throughput of the two policies over input ranges (where the relaxed
kernels' |x| < 2^16 certificate stops holding).  One JSON line per range.

    python tools/policy_probe.py [--n 67108864] [--reps 200]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2502_10831_b200 as ft  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1 << 26)
ap.add_argument("--reps", type=int, default=200)
a = ap.parse_args()
for hi in (6.283185307179586, 1e3, 6.5e4, 1e5, 1e6, 1e8):
    x = ft.gen_inputs(a.n, torch.float32, 0, -hi, hi, 12345)
    out = {nm: torch.empty_like(x) for nm in ("sin", "cos", "tan")}
    row = {"range": [-hi, hi], "n": a.n}
    for pol in ("ulp2", "bitwise"):
        with ft.f32_policy(pol):
            for _ in range(5):
                ft.proposed_eval(x, 7, out=out)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(a.reps):
                ft.proposed_eval(x, 7, out=out)
            e1.record()
            torch.cuda.synchronize()
            row[pol] = round(a.n / (e0.elapsed_time(e1) / a.reps / 1e3) / 1e9, 1)
    print(json.dumps(row), flush=True)
