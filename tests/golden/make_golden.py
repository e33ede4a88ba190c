"""Generate tests/golden/*.npz from the REAL reference (oracle/_ref).

Run here, where /root/reference exists:  python tests/golden/make_golden.py
The fixtures hold raw bit patterns: inputs x and the reference outputs of
proposed_{sin,cos,tan} (R:proj/include/fasttrig/kernels.hpp:46-67) plus the
per-element segment choice (segments.hpp:70-73 on reduce_sin / reduce_tan;
255 inside the tan pole window), computed by the unmodified reference headers
compiled by oracle/Makefile.  f32 rows are (float)proposed_*((double)x).

Taylor rows (no reference code exists) come from the C
restatement and are labelled source="port"; they are pinned separately by the
SPEC known-answer tests in tests/test_oracle_pin.py.
"""
from __future__ import annotations

import math
import os
import sys

import numpy as np

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), "..", ".."))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from paper_2502_10831_b200.configs import CONFIGS, PAPER_PROTOCOL  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
N_SAMPLE = 2048


def ulps_around(v: np.ndarray, k: int, dtype) -> np.ndarray:
    out = [v]
    up, dn = v.copy(), v.copy()
    inf = np.array(np.inf, dtype)
    for _ in range(k):
        up = np.nextafter(up, inf)
        dn = np.nextafter(dn, -inf)
        out += [up, dn]
    return np.concatenate(out)


def edge_cases(dtype) -> np.ndarray:
    d = np.dtype(dtype)
    pi, hp = math.pi, 0.5 * math.pi
    table = O.segment_table("ref")
    knots = table[42:49]
    special = [0.0, -0.0, 5e-324, -5e-324, 1e-310, 1e-300, 1e-30, 1e-10, 0.1, 1.0, -1.0, pi, -pi,
               2 * pi, hp, -hp, pi / 4, pi / 3, 2 * pi / 3, 3 * pi / 4, pi / 6, 5 * pi / 6, 1.5645,
               1.5707, 1e6, -1e6, 1e15, -1e15, 2.0**52, 2.0**53, 1e300, -1e300,
               np.finfo(np.float64).max, -np.finfo(np.float64).max, 3.4e38, -3.4e38,
               np.inf, -np.inf, np.nan, -np.nan]
    vals = [np.array(special, np.float64)]
    # knots (segment boundaries, red == x on [0, pi/2)) +- 3 ulps
    vals.append(ulps_around(knots.astype(d), 3, d).astype(np.float64))
    # quadrant edges and their thresholds, tan pole guard edges, +- 3 ulps
    edges = [m * hp for m in range(0, 9)] + [hp - 1e-3, hp + 1e-3, pi + hp - 1e-3, pi + hp + 1e-3]
    vals.append(ulps_around(np.array(edges, np.float64).astype(d), 3, d).astype(np.float64))
    # near-integer quotients: j*2pi, j*pi, j*pi/2 for assorted j, +- 2 ulps, both signs
    rng = np.random.default_rng(7)
    j = np.concatenate([np.arange(1, 40), rng.integers(40, 10**6, 200)]).astype(np.float64)
    mult = np.concatenate([j * 2 * pi, j * pi, j * hp, -j * pi])
    vals.append(ulps_around(mult.astype(d), 2, d).astype(np.float64))
    # wide magnitudes, both signs
    mag = 10.0 ** rng.uniform(-12, 25, 400)
    vals.append(np.concatenate([mag, -mag]).astype(d).astype(np.float64))
    x = np.concatenate(vals).astype(d)
    return x


def rows_for(name: str, x: np.ndarray, modes) -> dict:
    out = {}
    for mname, (m, s) in modes.items():
        r = O.proposed(x, 7, m, s, seg=True, impl="ref")
        key = f"{name}__{mname}"
        out[key + "__x"] = x
        for fn in ("sin", "cos", "tan"):
            out[key + "__" + fn] = r[fn]
        out[key + "__seg_sc"] = r["seg_sc"]
        out[key + "__seg_t"] = r["seg_t"]
    return out


def tan_stress_host(n: int, seed: int) -> np.ndarray:
    """Host stand-in for the device tan-stress generator (same distribution)."""
    rng = np.random.default_rng(seed)
    k = rng.integers(-1000, 1001, n)
    delta = np.clip(rng.normal(0.0, 1e-3, n), -0.05, 0.05)
    return ((2 * k + 1) * (0.5 * math.pi) + delta).astype(np.float32)


def main() -> None:
    assert O.ref_available(), "oracle/_ref not built: run `make -C oracle` where /root/reference exists"
    modes_all = {"fisr1": (1, 1), "exact": (0, 0), "fisr2": (1, 2), "fisr0": (1, 0)}
    modes_def = {"fisr1": (1, 1)}
    data = {}
    for cname in ("cfg1", "cfg2", "cfg5"):
        w = CONFIGS[cname]
        x = O.gen_uniform(N_SAMPLE, w.lo, w.hi, w.seed, 0, np.dtype(w.dtype).type)
        data.update(rows_for(cname, x, modes_all if cname == "cfg2" else modes_def))
    data.update(rows_for("cfg3", tan_stress_host(N_SAMPLE, 3), modes_def))
    p = PAPER_PROTOCOL
    data.update(rows_for("paper", O.gen_uniform(p.n, p.lo, p.hi, p.seed), modes_all))
    data.update(rows_for("edge64", edge_cases(np.float64), modes_all))
    data.update(rows_for("edge32", edge_cases(np.float32), modes_all))
    # Taylor (port-generated; SPEC-pinned)
    for cname in ("cfg4_f32", "cfg4_f64"):
        w = CONFIGS[cname]
        x = O.gen_uniform(N_SAMPLE, w.lo, w.hi, w.seed, 0, np.dtype(w.dtype).type)
        for nt in (5, 7, 9):
            r = O.taylor(x, nt, 7)
            key = f"taylor_{cname}__n{nt}"
            data[key + "__x"] = x
            for fn in ("sin", "cos", "tan"):
                data[key + "__" + fn] = r[fn]
    data["segment_table"] = O.segment_table("ref")
    path = os.path.join(OUT, "golden_v1.npz")
    np.savez_compressed(path, **data)
    print(f"wrote {path}: {len(data)} arrays, {os.path.getsize(path)} bytes")


if __name__ == "__main__":
    main()
