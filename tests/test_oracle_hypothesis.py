"""Property-based pin of the C restatement against the live reference build
(oracle/_ref): arbitrary doubles / floats, every SqrtMode, bit for bit, plus
segment choice.  CPU only; skipped where the reference was not built."""
from __future__ import annotations

import math

import numpy as np
import pytest

hypothesis = pytest.importorskip("hypothesis")
from hypothesis import given, settings  # noqa: E402
from hypothesis import strategies as st  # noqa: E402

from conftest import same_bits  # noqa: E402
from oracle import oracle as O  # noqa: E402

pytestmark = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")

modes = st.sampled_from([(1, 1), (0, 0), (1, 2), (1, 0), (1, 5)])
doubles = st.floats(allow_nan=True, allow_infinity=True, allow_subnormal=True, width=64)
near_multiples = st.builds(lambda k, j, s: s * float(np.nextafter(k * (math.pi / 2), math.inf) if j else k * (math.pi / 2)),
                           st.integers(0, 10**7), st.booleans(), st.sampled_from([1.0, -1.0]))


@settings(max_examples=300, deadline=None)
@given(st.lists(st.one_of(doubles, near_multiples), min_size=1, max_size=64), modes)
def test_port_equals_reference_f64(xs, mode):
    x = np.array(xs, dtype=np.float64)
    a = O.proposed(x, 7, *mode, seg=True, threads=1)
    b = O.proposed(x, 7, *mode, seg=True, threads=1, impl="ref")
    for k in ("sin", "cos", "tan"):
        assert same_bits(a[k], b[k]), k
    assert np.array_equal(a["seg_sc"], b["seg_sc"]) and np.array_equal(a["seg_t"], b["seg_t"])


@settings(max_examples=200, deadline=None)
@given(st.lists(st.floats(width=32, allow_nan=True, allow_infinity=True, allow_subnormal=True),
                min_size=1, max_size=64), modes)
def test_port_equals_reference_f32(xs, mode):
    x = np.array(xs, dtype=np.float32)
    a = O.proposed(x, 7, *mode, seg=True, threads=1)
    b = O.proposed(x, 7, *mode, seg=True, threads=1, impl="ref")
    for k in ("sin", "cos", "tan"):
        assert same_bits(a[k], b[k]), k
    assert np.array_equal(a["seg_sc"], b["seg_sc"]) and np.array_equal(a["seg_t"], b["seg_t"])


@settings(max_examples=100, deadline=None)
@given(doubles)
def test_batch_equals_scalar(x):
    """kernels.hpp:82-83 on the reference itself: the batch element is the scalar call."""
    R = O.ref()
    for which in range(3):
        out = np.empty(1)
        arr = np.array([x])
        R.ref_api_batch(which, arr.ctypes.data, 1, 1, 1, out.ctypes.data)
        assert same_bits(out, np.array([R.ref_scalar(which, x, 1, 1)]))
