"""Every float32 input through the f32 kernels: the relaxed policy (FT_F32_ULP2)
against the bit-exact one (FT_F32_BITWISE, itself pinned to the reference).

For each 2^28-element chunk of the 2^32 bit patterns (generated on the device):
  * production (non-SEG) relaxed kernel vs production bit-exact kernel, through
    K3 with the bit-exact outputs as the oracle arrays: max ulp, > 2 ulp count,
    raw-bit mismatches;
  * the SEG variants of both: segment choices compared element for element;
  * Taylor (NT 5/7/9) relaxed vs bit-exact the same way.
Prints one JSON line per (kind, mask, mode).  Usage (GPU box):
    python tools/f32_exhaustive.py [--masks 7,3,4] [--modes fisr1,exact] [--chunk-log2 28]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

MODES = {"fisr1": (1, 1), "exact": (0, 0), "fisr2": (1, 2), "fisr3": (1, 3)}


def chunk_bits(torch, start: int, n: int):
    """float32 tensor whose bit patterns are start .. start+n-1 (mod 2^32)."""
    s = start - (1 << 32) if start >= (1 << 31) else start
    b = torch.arange(n, dtype=torch.int32, device="cuda")
    b.add_(s)  # int32 wrap-around
    return b.view(torch.float32)


def run(kind: str, mask: int, mode: str, nterms: int, chunk_log2: int, total_log2: int = 32,
        seg: bool = True) -> dict:
    import torch

    import paper_2502_10831_b200 as ft

    n = 1 << chunk_log2
    sm = ft.SqrtMode(*MODES[mode])
    agg = {"kind": kind, "mask": mask, "mode": mode if kind == "proposed" else None,
           "n_terms": nterms if kind == "taylor" else None, "inputs": 0, "max_ulp": [0, 0, 0],
           "n_over_2ulp": [0, 0, 0], "n_bit_mismatch": [0, 0, 0], "seg_mismatch": [0, 0]}
    buf = torch.zeros(312, dtype=torch.uint8, device="cuda")
    t0 = time.time()
    for start in range(0, 1 << total_log2, n):
        x = chunk_bits(torch, start, n)
        if kind == "proposed":
            with ft.f32_policy("ulp2"):
                got = ft.proposed_eval(x, mask, sm)
            with ft.f32_policy("bitwise"):
                ref = ft.proposed_eval(x, mask, sm)
        else:
            with ft.f32_policy("ulp2"):
                got = ft.taylor_eval(x, nterms, mask)
            with ft.f32_policy("bitwise"):
                ref = ft.taylor_eval(x, nterms, mask)
        st = ft.parity_reduce(x, got, mask, kind=0 if kind == "proposed" else 1, mode=sm,
                              n_terms=nterms, refs=ref, ulp_tol=2, stats_buf=buf)
        del got, ref
        for j in range(3):
            agg["max_ulp"][j] = max(agg["max_ulp"][j], int(st["max_ulp"][j]))
            agg["n_over_2ulp"][j] += int(st["n_over_tol"][j])
            agg["n_bit_mismatch"][j] += int(st["n_bit_mismatch"][j])
        agg["inputs"] += int(st["n_checked"])
        if kind == "proposed" and seg:
            with ft.f32_policy("ulp2"):
                gs = ft.proposed_eval(x, mask, sm, seg=True)
            with ft.f32_policy("bitwise"):
                rs = ft.proposed_eval(x, mask, sm, seg=True)
            agg["seg_mismatch"][0] += int((gs["seg_sc"] != rs["seg_sc"]).sum())
            agg["seg_mismatch"][1] += int((gs["seg_t"] != rs["seg_t"]).sum())
            del gs, rs
    torch.cuda.synchronize()
    agg["seconds"] = round(time.time() - t0, 2)
    return agg


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--masks", default="7,3,4,1,2,5,6")
    ap.add_argument("--modes", default="fisr1,exact")
    ap.add_argument("--taylor", default="5,7,9")
    ap.add_argument("--taylor-masks", default="3,7")
    ap.add_argument("--chunk-log2", type=int, default=28)
    ap.add_argument("--total-log2", type=int, default=32)
    a = ap.parse_args()
    for mode in [m for m in a.modes.split(",") if m]:
        for mask in [int(m) for m in a.masks.split(",") if m]:
            print(json.dumps(run("proposed", mask, mode, 5, a.chunk_log2, a.total_log2)), flush=True)
    for nt in [int(t) for t in a.taylor.split(",") if t]:
        for mask in [int(m) for m in a.taylor_masks.split(",") if m]:
            print(json.dumps(run("taylor", mask, "fisr1", nt, a.chunk_log2, a.total_log2)), flush=True)


if __name__ == "__main__":
    main()
