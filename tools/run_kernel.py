"""Minimal driver for profiling: generate one config's inputs on the device and
launch its evaluation kernel `--reps` times (ncu captures; no timing here).

    python tools/run_kernel.py --config cfg2 --reps 3 [--elements N] [--mode fisr1|exact|fisr2]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2502_10831_b200 as ft  # noqa: E402
from paper_2502_10831_b200.configs import CONFIGS  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg2")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--elements", type=int, default=0)
ap.add_argument("--mode", default="fisr1")
ap.add_argument("--mask", type=int, default=0)
ap.add_argument("--check", action="store_true", help="also launch K3 (parity/error reduction) once")
a = ap.parse_args()
w = CONFIGS[a.config]
n = a.elements or min(w.n, 1 << 30)
mask = a.mask or w.mask
dt = torch.float32 if w.itemsize == 4 else torch.float64
x = ft.gen_inputs(n, dt, w.dist, w.lo, w.hi, w.seed)
mode = {"fisr1": ft.SqrtMode(), "exact": ft.SqrtMode.exact(), "fisr2": ft.SqrtMode.fisr(2)}[a.mode]
out = {nm: torch.empty_like(x) for j, nm in enumerate(("sin", "cos", "tan")) if mask & (1 << j)}
for _ in range(a.reps):
    if w.kind == 0:
        ft.proposed_eval(x, mask, mode, out=out)
    else:
        ft.taylor_eval(x, w.n_terms, mask, out=out)
if a.check:
    st = ft.parity_reduce(x, out, mask, kind=w.kind, mode=mode, n_terms=w.n_terms, ulp_tol=2)
    print("K3", {k: st[k] for k in ("n_checked", "max_ulp", "n_bit_mismatch")})
torch.cuda.synchronize()
print(f"ran {a.reps} x {a.config} n={n} mask={mask} mode={a.mode}")
