"""C-ABI library checks that need no GPU: it loads, exports every symbol
include/fasttrig_b200.h declares, carries the reference's constants bit for
bit, and rejects bad arguments before touching CUDA."""
from __future__ import annotations

import ctypes as C
import math
import os
import re
import subprocess

import numpy as np
import pytest

from conftest import ROOT
from oracle import oracle as O

HEADER = os.path.join(ROOT, "include", "fasttrig_b200.h")


def declared_symbols() -> set[str]:
    src = open(HEADER).read()
    return set(re.findall(r"^\s*(?:int|uint64_t|const char\*)\s+(ft_\w+)\s*\(", src, re.M))


def test_exports_every_declared_symbol(ft):
    from paper_2502_10831_b200 import _lib

    syms = declared_symbols()
    assert len(syms) >= 20
    assert syms == set(_lib.EXPORTS)
    L = _lib.lib()
    for s in syms:
        assert hasattr(L, s), s
    nm = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    for s in syms:
        assert re.search(rf"\bT {s}\b", nm), s
    assert L.ft_abi_version() == 2


def test_device_table_is_reference_table(ft, golden):
    t = ft.segment_table()
    assert np.array_equal(t.view(np.uint64), golden["segment_table"].view(np.uint64))


def test_taylor_coefficients_match_oracle(ft):
    s, c, t = ft.taylor_coeffs()
    a = [np.empty(9) for _ in range(3)]
    O.port().ora_taylor_coeffs(a[0].ctypes.data, a[1].ctypes.data, a[2].ctypes.data)
    for x, y in zip((s, c, t), a):
        assert np.array_equal(x.view(np.uint64), y.view(np.uint64))


def test_thresholds_are_exact(ft):
    """quad[j] is the least r >= 0 with floor(r / (pi/2)) >= j+1, and guard the least
    red with |red - pi/2| < 1e-3 (IEEE division/subtraction, as in reduction.hpp)."""
    th = ft.thresholds()
    hp = 0.5 * math.pi
    # the constants compiled into the kernels are the bisection results, bit for bit
    assert np.array_equal(th[:4].view(np.uint64), th[4:].view(np.uint64))
    for j in range(3):
        t = th[j]
        below = np.nextafter(t, 0.0)
        assert math.floor(t / hp) >= j + 1 and math.floor(below / hp) < j + 1
        assert abs(t - (j + 1) * hp) < 1e-14
    g = th[3]
    assert abs(g - hp) < 1e-3 and not abs(np.nextafter(g, 0.0) - hp) < 1e-3


def test_hiword_constants(ft):
    """The high-word compares of the fast path (ft_core.cuh kHi*) use the high
    words of the bisection thresholds, and the zone argument holds: an r that
    shares a threshold's high word but is given the lower quadrant folds
    (red = |r - c|, c = 0, pi, pi, 2pi) to a red that no row bracket accepts --
    below row 0's lower bound 2^-17 (r ~ pi, r ~ 2pi) or with the high word of
    pi/2 or above (r ~ pi/2, 3pi/2)."""
    src = open(os.path.join(ROOT, "paper_2502_10831_b200", "csrc", "ft_core.cuh")).read()
    const = {k: int(v, 16) for k, v in re.findall(r"constexpr int (kHi\w+) = (0x[0-9a-f]+);", src)}
    th = ft.thresholds()
    hi = lambda v: int(np.float64(v).view(np.uint64) >> np.uint64(32))  # noqa: E731
    assert const == {"kHiHalfPi": hi(th[0]), "kHiPiQ": hi(th[1]), "kHiThreeHalfPi": hi(th[2]),
                     "kHiRow0Lo": hi(2.0 ** -17), "kHiGuard": hi(th[3]), "kHiRelaxLo": hi(2.0 ** -11),
                     "kHiRelaxCos": hi(0.5 * math.pi - 2.0 ** -11)}
    assert hi(th[0]) == hi(0.5 * math.pi)  # tan fold threshold (r > pi/2) shares it
    P = math.pi
    bottom = lambda t: (np.uint64(hi(t)) << np.uint64(32)).view(np.float64)  # noqa: E731
    top = lambda t: ((np.uint64(hi(t)) << np.uint64(32)) | np.uint64(0xFFFFFFFF)).view(np.float64)  # noqa: E731
    for k, t in enumerate(th[:3]):
        r = np.array([t, top(t)])  # the wrongly-folded part of the bucket
        red = np.abs([r, r - P, r - P][k])  # lower-quadrant fold
        if k == 1:
            assert all(hi(v) <= const["kHiRow0Lo"] for v in red)  # -> fails row 0
        else:
            assert all(hi(v) >= const["kHiHalfPi"] for v in red)  # -> fails row 5's khi
    # r sharing 2pi's high word passes `valid`, folds with c = 2pi: tiny red
    r = np.array([bottom(2 * P), 2 * P, top(2 * P)])
    assert all(hi(v) <= const["kHiRow0Lo"] for v in np.abs(r - 2 * P))


def test_fisr_seed_identity():
    """ft_core.cuh fisr_seed: magic - (b >> 1) == (2*magic + 1 - b) >> 1 for
    every positive double bit pattern b (fisr.hpp:38-40)."""
    M = 0x5FE6EB50C7B537A9
    rng = np.random.default_rng(5)
    bs = [int(v) for v in rng.integers(0, 0x7FF0000000000000, 200000, dtype=np.uint64)]
    bs += [0, 1, 2, 0x7FEFFFFFFFFFFFFF, 0x7FF0000000000000, 0x3FF0000000000000, 0x3FF0000000000001]
    for b in bs:
        assert M - (b >> 1) == (2 * M + 1 - b) >> 1


def test_markstein_free_floor_is_caught():
    """ft_core.cuh fast_reduce (proposed path) floors q0 = RN(a * RN(1/2pi))
    instead of RN(a/2pi).  Wherever the floors differ (a within ~a*2^-52 of a
    multiple of 2pi or pi), the r it produces must be rejected downstream:
    r < 2^-17, or r within 2^-17 of the period (folds below row 0's bound).
    Checked on the adversarial neighbourhoods of k*2pi and k*pi for |x| < 2^30
    (plus random a), in binary64 with the reference's operation order."""
    P = math.pi
    y = 1.0 / (2.0 * P)
    rng = np.random.default_rng(11)
    ks = np.unique(np.concatenate([np.arange(1, 5000), rng.integers(1, 2**27, 20000)])).astype(np.float64)
    checked = 0
    for period, scale in ((2.0 * P, 1.0), (P, 2.0)):
        base = ks * period
        a = base[:, None].copy()
        # +-8 ulps around each multiple
        offs = np.arange(-8, 9)
        a = (base[:, None].view(np.int64) + offs[None, :]).view(np.float64).ravel()
        a = a[(a > 0) & (a < 2.0**30)]
        q0 = a * y
        q1 = a / (2.0 * P)
        f0 = np.floor(q0 * scale)  # tan: floor(2*q0) (exact doubling)
        f1 = np.floor(q1 * scale)
        diff = f0 != f1
        r_ref = a[diff] - period * f1[diff]
        r_ours = a[diff] - period * f0[diff]
        # ours is off by one period: below 2^-17 (negative, or an exact 0 when
        # a == RN(period*k)), or within 2^-17 of `period`
        assert ((r_ours < 2.0**-17) | (np.abs(r_ours - period) < 2.0**-17)).all()
        checked += int(diff.sum())
        assert (np.abs(np.abs(r_ours - r_ref) - period) < 1e-6).all()
    assert checked > 0  # the neighbourhoods do contain floor disagreements


def _hi(v):
    return int(np.float64(v).view(np.uint64) >> np.uint64(32))


def test_shared_row_margin(ft):
    """ft_core.cuh fast_proposed_core: fused kernels give the tangent the
    sine's segment row without a bracket check of its own.  Pins the two facts
    that argument rests on: (1) every high-word bracket a row accepts lies at
    least 5.2e-8 inside its knots, (2) the fused path's red and red_t (kernel
    operation order, exact FMA) differ by at most 2^-52*a + 2^-49 < 3e-8 for
    a < 2^27 -- checked on random a and on a near k*pi + knot."""
    from fractions import Fraction

    T = ft.segment_table()
    knots = T[42:49]
    # (1) margins of the high-word brackets (rows 1..5 lower, rows 0..4 upper)
    margins = []
    for kn in knots[1:6]:
        lo_edge = ((np.uint64(_hi(kn) + 1) << np.uint64(32))).view(np.float64)  # smallest accepted above
        hi_edge = ((np.uint64(_hi(kn)) << np.uint64(32)) - np.uint64(1)).view(np.float64)  # largest accepted below
        margins += [lo_edge - kn, kn - hi_edge]
    assert min(margins) > 5.2e-8

    # (2) red vs red_t in the kernel's operation order
    P = math.pi
    TWO_PI = 2.0 * P
    y = 1.0 / TWO_PI

    def fma(a, b, c):
        return float(Fraction(a) * Fraction(b) + Fraction(c))

    rng = np.random.default_rng(3)
    a_s = list(rng.uniform(0, 2.0**27, 3000)) + list(rng.uniform(0, 10.0, 1000))
    ks = rng.integers(0, 2**27 / P, 3000)
    a_s += [float(k * P + kn + d) for k, kn, d in zip(ks, rng.choice(knots[1:6], 3000), rng.uniform(-1e-7, 1e-7, 3000))]
    worst = 0.0
    for a in a_s:
        a = float(a)
        if not (0.0 < a < 2.0**27):
            continue
        q0 = a * y
        k = math.floor(q0)
        r = a - TWO_PI * k
        rh = _hi(r)
        p1, p2, p3 = rh > 0x3FF921FB, rh > 0x400921FB, rh > 0x4012D97C
        c = 2 * P if p3 else (P if p1 else 0.0)
        red = abs(r - c)
        rt = a - fma(float(k), TWO_PI, P if p2 else 0.0)
        up = _hi(rt) > 0x3FF921FB
        redt = abs(rt - (P if up else 0.0))
        if red < 2.0**-17 or _hi(red) >= 0x3FF921FB or not (0 <= rh <= 0x401921FB):
            continue  # rejected by the sine's checks
        diff = abs(red - redt)
        assert diff <= 2.0**-52 * a + 2.0**-49
        worst = max(worst, diff)
    assert worst < 3e-8


def test_invalid_arguments_fail_without_gpu(ft):
    from paper_2502_10831_b200 import _lib

    L = _lib.lib()
    m = _lib.SqrtModeC(1, 1)
    x = C.c_void_p(16)
    assert L.ft_proposed_eval(7, x, 4, 7, m, x, x, x, None) == _lib.FT_ERR_INVALID_ARG
    assert L.ft_proposed_eval(1, x, 4, 0, m, x, x, x, None) == _lib.FT_ERR_INVALID_ARG
    assert L.ft_proposed_eval(1, x, 4, 8, m, x, x, x, None) == _lib.FT_ERR_INVALID_ARG
    assert L.ft_proposed_eval(1, None, 4, 1, m, x, None, None, None) == _lib.FT_ERR_INVALID_ARG
    assert L.ft_proposed_eval(1, x, 4, 3, m, x, None, None, None) == _lib.FT_ERR_INVALID_ARG
    assert b"NULL" in L.ft_last_error_string()
    assert L.ft_proposed_eval(1, x, 4, 1, _lib.SqrtModeC(5, 1), x, None, None, None) == _lib.FT_ERR_INVALID_ARG
    assert L.ft_taylor_eval(1, x, 4, 1, 0, x, None, None, None) == _lib.FT_ERR_INVALID_ARG
    assert L.ft_taylor_eval(1, x, 4, 1, 10, x, None, None, None) == _lib.FT_ERR_INVALID_ARG
    assert L.ft_gen_inputs(1, 9, 0.0, 1.0, 1, 0, 4, x, None) == _lib.FT_ERR_INVALID_ARG
    # n == 0 is a no-op success (the reference maps an empty span to an empty vector)
    assert L.ft_proposed_eval(1, None, 0, 7, m, None, None, None, None) == 0
    assert L.ft_proposed_sin_batch(None, 0, m, None) == 0


def test_python_mirror_sqrtmode_semantics():
    from paper_2502_10831_b200 import SqrtMode

    assert SqrtMode() == SqrtMode(1, 1)  # fisr.hpp:17-18 default fisr(1)
    assert SqrtMode.exact() == SqrtMode(0, 0)
    assert SqrtMode.fisr(0) == SqrtMode(1, 1) and SqrtMode.fisr(3) == SqrtMode(1, 3)


def test_missing_library_fails_loudly(tmp_path, monkeypatch):
    """No CPU fallback: a missing .so raises instead of computing anything."""
    from paper_2502_10831_b200 import _lib

    monkeypatch.setattr(_lib, "_lib", None)
    monkeypatch.setattr(_lib, "LIB_PATH", str(tmp_path / "missing.so"))
    with pytest.raises(_lib.FasttrigError):
        _lib.lib()


def test_fold_needs_no_clamp(ft):
    """The fast path drops the reference's final clamp of red to [0, pi/2]
    (reduction.hpp:32-35 called from :51 and :89).  Sound because each quadrant's
    red = RN(base +- r) is monotone in r, so its extremes sit at the quadrant
    edges (the bisected thresholds); check every edge in IEEE binary64."""
    th = ft.thresholds()
    T1, T2, T3 = th[:3]
    pi, hp, tp = math.pi, 0.5 * math.pi, 2.0 * math.pi
    prev = lambda v: float(np.nextafter(v, 0.0))  # noqa: E731
    nxt = lambda v: float(np.nextafter(v, 10.0))  # noqa: E731
    assert prev(T1) <= hp                                   # q=0: red = r < T1
    assert 0.0 <= pi - prev(T2) and pi - T1 <= hp           # q=1: red = pi - r
    assert 0.0 <= T2 - pi and prev(T3) - pi <= hp           # q=2: red = r - pi
    assert 0.0 <= tp - prev(tp) and tp - T3 <= hp           # q=3: red = 2pi - r
    assert 0.0 <= pi - prev(pi) and pi - nxt(hp) <= hp      # tan upper: red = pi - r


def test_host_device_setting_roundtrip(ft):
    assert ft.get_host_devices() == 1  # default: the current device only
    ft.set_host_devices(0)
    assert ft.get_host_devices() == 0
    ft.set_host_devices(1)


def _rn_fma_reduce(a: float) -> tuple[float, int]:
    """The relaxed f32 reduction (ft_core.cuh relaxed_proposed_core) in exact
    rational arithmetic: m = rint(a * RN(1/pi)) (one FMA with 1.5*2^52),
    d = RN(a - pi*m) (one FMA)."""
    from fractions import Fraction as F

    inv_pi = F(2.0 * (1.0 / (2.0 * math.pi)))  # RN(1/pi) = 2 RN(1/2pi), as in kFast.inv_pi
    t = float(F(a) * inv_pi + F(float.fromhex("0x1.8p52")))  # RN of the exact FMA result
    m = int(t - float.fromhex("0x1.8p52"))
    d = float(F(a) - F(math.pi) * m)
    return d, m


def test_relaxed_reduction_error_bound():
    """DESIGN.md section 3 / ft_core.cuh relaxed_*: for |x| < 2^16 the one-FMA
    signed reduction |d| differs from the reference's red (reduce_sin, reduce_tan)
    by <= 2^-37.9, and the sign bits it implies equal the reference's signs
    wherever the relaxed brackets accept the lane (2^-11 <= |d| < hi(pi/2))."""
    from oracle import oracle as O

    L = O.port()
    rng = np.random.default_rng(5)
    k = rng.integers(1, 20860, 4000)  # multiples of pi/2 up to 2^15
    xs = np.concatenate([rng.uniform(0, 65536, 6000), rng.uniform(0, 8, 2000),
                         k * (math.pi / 2) + rng.uniform(-1e-3, 1e-3, k.size)]).astype(np.float32)
    worst = 0.0
    for xf in xs:
        a = float(xf)
        if a == 0.0:
            continue
        d, m = _rn_fma_reduce(a)
        for which in (0, 2):
            red, sign = C.c_double(), C.c_double()
            getattr(L, "ora_reduce_sin" if which == 0 else "ora_reduce_tan")(a, C.byref(red), C.byref(sign))
            worst = max(worst, abs(abs(d) - red.value))
            if 2.0 ** -11 <= abs(d) < 0.5 * math.pi - 3.1e-7:
                want = (-1.0 if d < 0 else 1.0) * (-1.0 if (which == 0 and m % 2) else 1.0)
                assert sign.value == want, (a, which)
    assert worst <= 2.0 ** -37.9, worst


def test_relaxed_guard_bucket_margin():
    """The relaxed kernels decide the pole guard from hi(red) and reject
    hi(red) == hi(guard): the guard must sit well inside its high-word bucket
    (>> the 2^-37.9 reduction error), so the decision is the reference's."""
    g = float.fromhex("0x1.91de2c0cf70aep+0")
    b = int(np.float64(g).view(np.uint64))
    lo = (np.uint64(b >> 32 << 32)).view(np.float64)
    hi = (np.uint64((b >> 32 << 32) | 0xFFFFFFFF)).view(np.float64)
    assert g - lo > 2.3e-7 and hi - g > 2.3e-7


def test_new_entry_points_validate_without_gpu(ft):
    """Round-2 ABI additions reject bad arguments before touching CUDA, and the
    f32 policy round-trips (process-wide)."""
    from paper_2502_10831_b200 import _lib

    L = _lib.lib()
    assert L.ft_device_rows(9, C.c_void_p(16)) == _lib.FT_ERR_INVALID_ARG
    assert L.ft_device_rows(0, None) == _lib.FT_ERR_INVALID_ARG
    assert L.ft_device_const_table(7, C.c_void_p(16)) == _lib.FT_ERR_INVALID_ARG
    assert L.ft_device_const_table(0, None) == _lib.FT_ERR_INVALID_ARG
    assert L.ft_set_f32_policy(2) == _lib.FT_ERR_INVALID_ARG
    assert b"policy" in L.ft_last_error_string()
    assert ft.get_f32_policy() == "ulp2"  # default
    with ft.f32_policy("bitwise"):
        assert ft.get_f32_policy() == "bitwise" and L.ft_get_f32_policy() == _lib.FT_F32_BITWISE
    assert ft.get_f32_policy() == "ulp2"
    # without a visible device ft_release reports the CUDA error instead of crashing
    rc = L.ft_release(-1)
    assert rc in (_lib.FT_OK, _lib.FT_ERR_NO_DEVICE, _lib.FT_ERR_CUDA)


def test_python_outputs_are_validated(ft):
    """caller-supplied host outputs of the wrong dtype, size or layout
    are rejected before any pointer reaches the C ABI."""
    x = np.zeros(16, np.float64)
    with pytest.raises(TypeError):
        ft.proposed_batch(x, 1, out={"sin": np.zeros(16, np.float32)})
    with pytest.raises(ValueError):
        ft.proposed_batch(x, 1, out={"sin": np.zeros(8, np.float64)})
    with pytest.raises(ValueError):
        ft.proposed_batch(x, 1, out={"sin": np.zeros(32, np.float64)[::2]})
    with pytest.raises(TypeError):
        ft.proposed_batch(x, 3, out={"sin": np.zeros(16, np.float64)})  # cos missing
    with pytest.raises(ValueError):
        ft.proposed_batch(x, 0)
