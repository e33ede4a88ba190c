"""Every binary64 high word: all 2^32 doubles whose low word is `--lo` (every sign,
exponent and top-20-bit mantissa, incl. subnormals, infinities and NaNs) through
the production f64 kernels (fused S/C/T, TMA bulk stores), checked by K3 against
the device restatement of the reference (itself pinned bit for bit to the
reference library by the test suite).  The fast path's quadrant and row
decisions compare high words, so this walks every value those compares can see.
One JSON line per low word.

    python tools/f64_hiword_sweep.py --lo 0 ffffffff 80000000 [--mode fisr1]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2502_10831_b200 as ft  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--lo", nargs="+", default=["0"])
ap.add_argument("--random", type=int, default=0, help="also this many seeded random low words")
ap.add_argument("--mode", default="fisr1", choices=["fisr1", "exact", "fisr2"])
ap.add_argument("--chunk", type=int, default=1 << 28)
ap.add_argument("--taylor", type=int, default=0, help="N > 0: the Taylor kernel K2 with N terms instead of K1")
ap.add_argument("--mask", type=int, default=7)
a = ap.parse_args()
mode = {"fisr1": ft.SqrtMode(), "exact": ft.SqrtMode.exact(), "fisr2": ft.SqrtMode.fisr(2)}[a.mode]
los = [int(v, 16) for v in a.lo]
if a.random:
    g = torch.Generator().manual_seed(2024873)
    los += [int(v) for v in torch.randint(0, 1 << 32, (a.random,), generator=g, dtype=torch.int64)]
for lo in los:
    t0 = time.time()
    tot = {"n": 0, "max_ulp": [0, 0, 0], "bit_mismatch": [0, 0, 0], "nan": [0, 0, 0], "inf": [0, 0, 0]}
    out = None
    for start in range(0, 1 << 32, a.chunk):
        hi = torch.arange(start, start + a.chunk, dtype=torch.int64, device="cuda")
        x = ((hi << 32) | lo).view(torch.float64)
        del hi
        if out is None:
            out = {nm: torch.empty_like(x) for j, nm in enumerate(("sin", "cos", "tan")) if a.mask & (1 << j)}
        if a.taylor:
            ft.taylor_eval(x, a.taylor, a.mask, out=out)
            st = ft.parity_reduce(x, out, a.mask, kind=1, n_terms=a.taylor, ulp_tol=0)
        else:
            ft.proposed_eval(x, a.mask, mode, out=out)
            st = ft.parity_reduce(x, out, a.mask, mode=mode, ulp_tol=0)
        tot["n"] += st["n_checked"]
        for j in range(3):
            tot["max_ulp"][j] = max(tot["max_ulp"][j], st["max_ulp"][j])
            tot["bit_mismatch"][j] += st["n_bit_mismatch"][j]
            tot["nan"][j] += st["n_nan"][j]
            tot["inf"][j] += st["n_inf"][j]
        del x
    print(json.dumps({"low_word": f"{lo:08x}", "kernel": f"taylor-{a.taylor}" if a.taylor else "proposed",
                      "mask": a.mask, "mode": a.mode, "checked": tot["n"], "max_ulp_vs_restatement": tot["max_ulp"],
                      "bit_mismatches": tot["bit_mismatch"], "nan": tot["nan"], "inf": tot["inf"],
                      "seconds": round(time.time() - t0, 1)}), flush=True)
