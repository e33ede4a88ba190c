"""the segment table re-derived from the paper's construction
(tools/derive_table.py) equals the reference's table bit for
bit, and the kernels' host copy is that table."""
from __future__ import annotations

import os
import sys

import numpy as np

from conftest import ROOT
from oracle import oracle as O

sys.path.insert(0, os.path.join(ROOT, "tools"))
import derive_table as D  # noqa: E402


def test_outer_segments_follow_exactly_from_the_30_45_segment():
    assert D.derive_tan_outer("low") == (11, 0, -1, 632)    # PAPER Eq. (9): 11x / (632 - x)
    assert D.derive_tan_outer("high") == (1, 542, -11, 990)  # PAPER Eq. (10): (x + 542) / (990 - 11x)


def test_middle_integer_rationals_match_the_interpolation_quotient():
    for k in range(1, 5):
        assert D.verify_mid(k, tol_rel=0.01) < 0.002
    # the interpolation passes through its knots
    for k in range(1, 5):
        s, i = D.interp_sin_segment(k)
        for t in (15 * k, 15 * (k + 1)):
            assert abs(s * t + i - np.sin(np.radians(t))) < 1e-15
    # Eq. (5) numerator as printed (0.2411x + 0.2645)
    (na, nb), (da, _) = D.derive_tan_mid(1)
    assert abs(na - 0.2411) < 2e-4 and abs(nb - 0.2645) < 2e-4 and abs(da + 0.0999) < 2e-4


def test_radian_table_bits_equal_reference_and_kernels(ft):
    derived = np.array(D.to_radian_table(D.degree_segments()))
    ref = O.segment_table("ref" if O.ref_available() else "port")
    assert np.array_equal(derived.view(np.uint64), ref.view(np.uint64))
    assert np.array_equal(derived.view(np.uint64), ft.segment_table().view(np.uint64))


def test_sincos_from_tan_examples():
    assert D.sincos_from_tan(1, 542, -11, 990) == (122, -20696, 1273864)  # SPEC.md sincos_from_tan
    assert D.sincos_from_tan(11, 0, -1, 632) == (122, -1264, 399424)
    assert D.sincos_from_tan(0, 1, 0, 1) == (0, 0, 2)
