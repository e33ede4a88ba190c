"""Re-derive the segment table from the paper's construction (SPEC.md:268-346,
PAPER.md Appendix A) and check it against the table the kernels carry.

The reference hard-codes the degree-space integer rationals
(R:proj/include/fasttrig/segments.hpp:33-40) and converts them to radians
(segments.hpp:42-62).  This tool rebuilds that chain:

  1. interp_sin_segment(k): linear interpolation of sine between the 15-degree
     knots (Appendix Eqs. 1-4);
  2. derive_tan_mid(k): tan x ~ interp_sin(x) / interp_sin(90 - x) for the four
     middle segments (Eqs. 5-8, scaled by 15 as printed in the paper);
  3. the published integer rationals of the middle segments are checked
     functionally against (2) -- SPEC.md "we treat the published integers as
     canonical constants and verify them functionally" -- within 1% on a
     1000-point grid;
  4. derive_tan_outer(low/high): the two outer segments follow EXACTLY from the
     [30, 45] integer segment by tan(45 -/+ x') = (1 -/+ t)/(1 +/- t)
     (Eqs. 9-10), in exact rational arithmetic;
  5. sincos_from_tan / to_radian_coeffs: X = a^2+c^2, Y = 2(ab+cd), Z = b^2+d^2
     and the degree -> radian conversion in the reference's own binary64
     operation order (segments.hpp:44-50), giving the radian table whose bits
     must equal fasttrig::segment_table and the kernels' copies.

    python tools/derive_table.py        # prints the report, exit 1 on mismatch
"""
from __future__ import annotations

import json
import math
import sys
from fractions import Fraction

KNOTS_DEG = [0, 15, 30, 45, 60, 75, 90]
# The published integer rationals (a x + b) / (c x + d), x in degrees, for the
# middle segments [15k, 15(k+1)], k = 1..4 (PAPER.md Appendix, Eqs. 5-8 rounded
# to integers; segments.hpp:34-39 rows 1-4).  The outer rows are derived below.
MID_INTEGER = {1: (10, 10, -4, 657), 2: (6, 46, -5, 541), 3: (10, 217, -13, 1252), 4: (4, 297, -10, 910)}


def interp_sin_segment(k: int) -> tuple[float, float]:
    """Degree-space line through (15k, sin 15k) and (15(k+1), sin 15(k+1))."""
    t1, t2 = 15.0 * k, 15.0 * (k + 1)
    s1, s2 = math.sin(math.radians(t1)), math.sin(math.radians(t2))
    return (s2 - s1) / 15.0, (t2 * s1 - t1 * s2) / 15.0


def derive_tan_mid(k: int) -> tuple[tuple[float, float], tuple[float, float]]:
    """tan x ~ interp_sin(x) / interp_sin(90 - x) on [15k, 15(k+1)], both scaled
    by 15 as the paper prints them: ((num slope, num int), (den slope, den int))."""
    sn, in_ = interp_sin_segment(k)
    sd, id_ = interp_sin_segment(5 - k)  # 90 - x lies in the complementary interval
    return (15.0 * sn, 15.0 * in_), (-15.0 * sd, 15.0 * (90.0 * sd + id_))


def rational(coef, x):
    a, b, c, d = coef
    return (a * x + b) / (c * x + d)


def verify_mid(k: int, tol_rel: float = 0.01, points: int = 1000) -> float:
    """Max relative difference between the published integer rational and the
    interpolation quotient on the segment's grid."""
    (na, nb), (da, db) = derive_tan_mid(k)
    lo, hi = 15.0 * k, 15.0 * (k + 1)
    worst = 0.0
    for i in range(points):
        x = lo + (hi - lo) * i / (points - 1)
        exact = (na * x + nb) / (da * x + db)
        worst = max(worst, abs(rational(MID_INTEGER[k], x) - exact) / abs(exact))
    if worst > tol_rel:
        raise AssertionError(f"segment {k}: integer rational off by {worst:.3g} > {tol_rel}")
    return worst


def derive_tan_outer(side: str) -> tuple[int, int, int, int]:
    """Outer segments from the [30, 45] segment t(y) = (6y + 46) / (541 - 5y):
    low  x in [0, 15]:  y = 45 - x, tan x = (1 - t) / (1 + t);
    high x in [75, 90]: y = x - 45, tan x = (1 + t) / (1 - t).
    Exact rational arithmetic; returns integer (a, b, c, d)."""
    a2, b2, c2, d2 = MID_INTEGER[2]
    # t(y) = (a2 y + b2) / (c2 y + d2) with y = s x + o
    s, o = (-1, 45) if side == "low" else (1, -45)
    tn = (a2 * s, a2 * o + b2)  # numerator of t as (x coef, const)
    td = (c2 * s, c2 * o + d2)
    if side == "low":  # (td - tn) / (td + tn)
        num, den = (td[0] - tn[0], td[1] - tn[1]), (td[0] + tn[0], td[1] + tn[1])
    else:  # (td + tn) / (td - tn)
        num, den = (td[0] + tn[0], td[1] + tn[1]), (td[0] - tn[0], td[1] - tn[1])
    g = math.gcd(math.gcd(abs(num[0]), abs(num[1])), math.gcd(abs(den[0]), abs(den[1])))
    return (num[0] // g, num[1] // g, den[0] // g, den[1] // g)


def degree_segments() -> list[tuple[int, int, int, int]]:
    """All six degree-space integer rationals, outer rows derived, middle rows the
    functionally verified published integers (segments.hpp:33-40 order)."""
    return [derive_tan_outer("low"), *(MID_INTEGER[k] for k in range(1, 5)), derive_tan_outer("high")]


def sincos_from_tan(a, b, c, d):
    """Appendix Eq. (14): radicand coefficients (exact rationals for exact input)."""
    return a * a + c * c, 2 * (a * b + c * d), b * b + d * d


def to_radian_table(deg) -> list[float]:
    """The reference's binary64 conversion (segments.hpp:42-62), same operation
    order (Python floats are IEEE binary64, no contraction): 6 x {a,b,c,d,X,Y,Z}
    then the 7 knots -- the layout of ft_segment_table / ref_segment_table."""
    pi = math.pi
    deg_per_rad = 180.0 / pi
    out = []
    for a_, b_, c_, d_ in deg:
        a = float(a_) * deg_per_rad
        b = float(b_)
        c = float(c_) * deg_per_rad
        d = float(d_)
        out += [a, b, c, d, a * a + c * c, 2.0 * (a * b + c * d), b * b + d * d]
    out += [0.0, pi / 12.0, pi / 6.0, pi / 4.0, pi / 3.0, 5.0 * pi / 12.0, pi / 2.0]
    return out


def report() -> dict:
    rep = {"mid_segments_max_rel_diff": {k: verify_mid(k) for k in range(1, 5)}}
    deg = degree_segments()
    rep["degree_segments"] = [list(r) for r in deg]
    # degree-space Eq. (14) identities, exact
    rep["eq14_Z_equals_b2_plus_d2"] = all(
        sincos_from_tan(*map(Fraction, r))[2] == r[1] ** 2 + r[3] ** 2 for r in deg)
    rep["paper_eq5_k1"] = [round(v, 4) for pair in derive_tan_mid(1) for v in pair]
    rep["radian_table"] = [float.hex(v) for v in to_radian_table(deg)]
    return rep


def main() -> int:
    rep = report()
    ok = rep["degree_segments"] == [[11, 0, -1, 632], [10, 10, -4, 657], [6, 46, -5, 541],
                                    [10, 217, -13, 1252], [4, 297, -10, 910], [1, 542, -11, 990]]
    try:
        sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__file__)))
        from oracle import oracle as O

        ref = O.segment_table("ref" if O.ref_available() else "port")
        same = [float.hex(float(v)) for v in ref] == rep["radian_table"]
        rep["radian_table_equals_reference_bits"] = same
        ok = ok and same
    except Exception as e:  # noqa: BLE001
        rep["radian_table_equals_reference_bits"] = f"not checked: {e}"
    print(json.dumps(rep, indent=1))
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
