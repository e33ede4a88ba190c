"""GPU parity: the sm_100a path (through the C ABI) against the oracle.

Bar (BASELINE.json north_star): at most 2 ulp from the reference's own output
and identical segment choice per element.  This module runs the bit-exact
kernels (f32 policy FT_F32_BITWISE for the whole module) and asserts 0 ulp: f64
outputs bitwise equal to proposed_*(x), f32 outputs bitwise equal to
(float)proposed_*((double)x).  The default f32 policy (FT_F32_ULP2) is covered
by tests/test_f32_exhaustive_gpu.py.
"""
from __future__ import annotations

import math
import os
import subprocess

import numpy as np
import pytest

from conftest import MODES, ROOT, golden_cases, same_bits, ulp_dist
from oracle import oracle as O
from paper_2502_10831_b200.configs import CONFIGS, PAPER_PROTOCOL, shard

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
ULP_TOL = 2  # north_star tolerance (ulps of the output dtype)


@pytest.fixture(autouse=True)
def _bitwise_policy(ft):
    with ft.f32_policy("bitwise"):
        yield


def dev(a: np.ndarray):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def host(t) -> np.ndarray:
    return t.cpu().numpy()


def check_against(x: np.ndarray, out: dict, ref: dict, fns=("sin", "cos", "tan"), seg=True):
    for f in fns:
        g = host(out[f])
        d = ulp_dist(g, ref[f])
        assert d.max() <= ULP_TOL, (f, d.max())
        assert same_bits(g, ref[f]), f  # design target: 0 ulp
    if seg:
        assert np.array_equal(host(out["seg_sc"]), ref["seg_sc"])
        assert np.array_equal(host(out["seg_t"])[: x.size], ref["seg_t"])


def test_k1_matches_golden_reference_vectors(ft, golden):
    """Every golden vector (edge cases, configs' first elements, paper protocol)
    through the segment-writing K1 and through the production kernels (no
    segment output: for f64 the TMA-bulk-store instantiations), every mask."""
    n = 0
    for case, mode, x, ref in golden_cases(golden):
        sm = ft.SqrtMode(*MODES[mode])
        out = ft.proposed_eval(dev(x), 7, sm, seg=True)
        torch.cuda.synchronize()
        check_against(x, out, ref)
        for mask in (7, 3, 4, 1):
            out = ft.proposed_eval(dev(x), mask, sm)
            torch.cuda.synchronize()
            fns = [f for j, f in enumerate(("sin", "cos", "tan")) if mask & (1 << j)]
            check_against(x, out, ref, fns=fns, seg=False)
        n += x.size
    assert n > 20000


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("mask", range(1, 8))
def test_k1_every_mask_ragged_and_misaligned(ft, dtype, mask):
    rng = np.random.default_rng(mask)
    base = rng.uniform(-3e3, 3e3, 70001).astype(dtype)
    for off in (0, 1, 3):
        for n in (0, 1, 2, 3, 5, 17, 1023, 4097, 70001 - off):
            x = base[off:off + n]
            xd = dev(base)[off:off + n]  # offset views -> unaligned pointers
            out = {nm: torch.empty(max(n + 1, 1), dtype=xd.dtype, device="cuda")[1:n + 1]
                   for j, nm in enumerate(("sin", "cos", "tan")) if mask & (1 << j)}
            ft.proposed_eval(xd, mask, out=out)
            torch.cuda.synchronize()
            if n == 0:
                continue
            ref = O.proposed(x, mask)
            for f in out:
                assert same_bits(host(out[f]), ref[f]), (off, n, f)


@pytest.mark.parametrize("mode", list(MODES) + ["fisr3"])
@pytest.mark.parametrize("cfg", ["cfg1", "cfg2", "cfg5"])
def test_k1_config_samples_vs_oracle(ft, cfg, mode):
    w = CONFIGS[cfg]
    m, s = MODES.get(mode, (1, 3))
    n = 1 << 21
    x = O.gen_uniform(n, w.lo, w.hi, w.seed, 12345, np.dtype(w.dtype).type)
    out = ft.proposed_eval(dev(x), 7, ft.SqrtMode(m, s), seg=True)
    torch.cuda.synchronize()
    check_against(x, out, O.proposed(x, 7, m, s, seg=True))


def test_k1_adversarial_quotients(ft):
    """Inputs whose |x|/(2pi), |x|/pi, r/(pi/2) quotients sit within a few ulps of
    integers: the places a non-IEEE floor(a/P) would differ (Markstein step)."""
    rng = np.random.default_rng(3)
    j = np.concatenate([np.arange(1, 5000), rng.integers(5000, 10**7, 200000)]).astype(np.float64)
    base = np.concatenate([j * 2 * math.pi, j * math.pi, j * 0.5 * math.pi,
                           rng.uniform(0, 1e15, 20000)])
    xs = [base]
    up, dn = base.copy(), base.copy()
    for _ in range(4):
        up, dn = np.nextafter(up, np.inf), np.nextafter(dn, -np.inf)
        xs += [up, dn]
    x = np.concatenate(xs)
    x = np.concatenate([x, -x])
    for m, s in ((1, 1), (0, 0)):
        out = ft.proposed_eval(dev(x), 7, ft.SqrtMode(m, s), seg=True)
        torch.cuda.synchronize()
        check_against(x, out, O.proposed(x, 7, m, s, seg=True))
        xf = x.astype(np.float32)
        out = ft.proposed_eval(dev(xf), 7, ft.SqrtMode(m, s), seg=True)
        torch.cuda.synchronize()
        check_against(xf, out, O.proposed(xf, 7, m, s, seg=True))


def test_certify_or_redo_boundaries(ft):
    """The fast paths' certificates (ft_core.cuh fast_reduce / fast_proposed_core
    / fast_taylor): inputs straddling each bound they rest on must still return
    the reference's bits in every output mask, f32 and f64, proposed and Taylor:
    |x| around the `valid` limit 2^24*2pi (= 2^25*pi for tan-only), odd and even
    multiples of pi and pi/2 up to that limit (tangent floor taken from the
    sine's k, off-by-one floors), and reduced angles around row 0's bound 2^-17."""
    rng = np.random.default_rng(17)
    P = math.pi
    lim = 2.0**24 * 2 * P
    parts = [lim * (1 + rng.uniform(-1e-3, 1e-3, 20000)),
             lim + np.arange(-2000, 2000) * np.spacing(lim)]
    k = np.concatenate([rng.integers(1, int(lim / P), 30000), np.arange(1, 3000)]).astype(np.float64)
    for mult in (P, 0.5 * P):
        b = k * mult
        b = b[b < 1.05 * lim]
        parts += [b + d * np.spacing(b) for d in (-3, -1, 0, 1, 3)]
    kk = np.arange(0, 64).astype(np.float64)
    for e in (-17.0, -16.0, -18.0):
        d = 2.0**e * (1 + rng.uniform(-1e-3, 1e-3, kk.size))
        parts += [kk * P + d, kk * P - d, kk * P + 0.5 * P + d]
    x = np.concatenate(parts)
    x = np.concatenate([x, -x])
    for dtype in (np.float64, np.float32):
        xd = x.astype(dtype)
        for mask in range(1, 8):
            out = ft.proposed_eval(dev(xd), mask, seg=mask == 7)
            torch.cuda.synchronize()
            ref = O.proposed(xd, mask, seg=mask == 7)
            fns = [f for j, f in enumerate(("sin", "cos", "tan")) if mask & (1 << j)]
            check_against(xd, out, ref, fns=fns, seg=mask == 7)
        for mask in (3, 7, 4):
            out = ft.taylor_eval(dev(xd), 5, mask)
            torch.cuda.synchronize()
            ref = O.taylor(xd, 5, mask)
            for j, f in enumerate(("sin", "cos", "tan")):
                if mask & (1 << j):
                    assert same_bits(host(out[f]), ref[f]), (dtype, mask, f)


def test_k1_hiword_zones(ft):
    """The fast path compares high words only (quadrant, tan fold, row bracket,
    ft_core.cuh fast_reduce/SmemTable): inputs whose r or red shares its high
    word with pi/2, pi, RN(3pi/2) or a knot must still return the reference's
    bits (they are assigned a conservative choice and redone exactly)."""
    rng = np.random.default_rng(11)
    xs = []
    # r itself in each threshold's high-word bucket (x = r, period 0)
    for hi in (0x3FF921FB, 0x400921FB, 0x4012D97C):
        lo = np.concatenate([rng.integers(0, 1 << 32, 60000, dtype=np.uint64),
                             np.arange(0, 64, dtype=np.uint64), (1 << 32) - 1 - np.arange(64, dtype=np.uint64)])
        xs.append(((np.uint64(hi) << np.uint64(32)) | lo).view(np.float64))
    # centres m*pi/12 (every knot and quadrant boundary of ~40 periods) +- a few
    # high-word buckets
    m = np.arange(0, 24 * 40)
    c = np.repeat(m * (math.pi / 12), 2000)
    xs.append(c + rng.uniform(-4e-6, 4e-6, c.size) * np.maximum(1.0, c / 8))
    x = np.concatenate(xs)
    x = np.concatenate([x, -x])
    for m_, s in ((1, 1), (1, 2), (0, 0)):
        out = ft.proposed_eval(dev(x), 7, ft.SqrtMode(m_, s), seg=True)
        torch.cuda.synchronize()
        check_against(x, out, O.proposed(x, 7, m_, s, seg=True))
        for mask in (3, 4):  # sin/cos-only and tan-only kernels reduce once
            out = ft.proposed_eval(dev(x), mask, ft.SqrtMode(m_, s))
            torch.cuda.synchronize()
            ref = O.proposed(x, mask, m_, s)
            for f in out:
                assert same_bits(host(out[f]), ref[f]), (mask, f)
        xf = x.astype(np.float32)
        out = ft.proposed_eval(dev(xf), 7, ft.SqrtMode(m_, s), seg=True)
        torch.cuda.synchronize()
        check_against(xf, out, O.proposed(xf, 7, m_, s, seg=True))


@pytest.mark.parametrize("dtype", ["float32", "float64"])
def test_device_generator_matches_host(ft, dtype):
    for w in (CONFIGS["cfg1"], CONFIGS["cfg2"], CONFIGS["cfg5"], PAPER_PROTOCOL):
        n = 100003
        for off in (0, 77, (1 << 32) + 5):
            xd = ft.gen_inputs(n, getattr(torch, dtype), 0, w.lo, w.hi, w.seed, off)
            xh = O.gen_uniform(n, w.lo, w.hi, w.seed, off, np.dtype(dtype).type)
            assert same_bits(host(xd), xh), (w.name, off)
    p = PAPER_PROTOCOL
    x = ft.gen_inputs(p.n, torch.float64, 0, p.lo, p.hi, p.seed)
    assert host(x)[0] == -316094.96443841327


def test_taylor_matches_oracle(ft, golden):
    for key in sorted({k.rsplit("__", 1)[0] for k in golden if k.startswith("taylor_")}):
        x = golden[key + "__x"]
        nt = int(key.rsplit("__n", 1)[1])
        out = ft.taylor_eval(dev(x), nt, 7)
        torch.cuda.synchronize()
        for f in ("sin", "cos", "tan"):
            assert same_bits(host(out[f]), golden[key + "__" + f]), (key, f)
    rng = np.random.default_rng(9)
    for dt in (np.float32, np.float64):
        x = rng.uniform(-2e3, 2e3, 300001).astype(dt)
        for nt in range(1, 10):
            for mask in (1, 2, 3, 4, 7):
                out = ft.taylor_eval(dev(x), nt, mask)
                torch.cuda.synchronize()
                ref = O.taylor(x, nt, mask)
                for f in ref:
                    assert same_bits(host(out[f]), ref[f]), (dt, nt, mask, f)


def test_mirror_kernel_is_the_oracle(ft):
    """The device restatement used by K3 equals the CPU oracle bit for bit."""
    w = CONFIGS["cfg2"]
    x = O.gen_uniform(1 << 20, w.lo, w.hi, w.seed, 999)
    for m, s in ((1, 1), (0, 0), (1, 2)):
        out = ft.mirror_eval(dev(x), 7, 0, ft.SqrtMode(m, s), seg=True)
        torch.cuda.synchronize()
        check_against(x, out, O.proposed(x, 7, m, s, seg=True))
    out = ft.mirror_eval(dev(x), 7, 1, n_terms=7)
    torch.cuda.synchronize()
    ref = O.taylor(x, 7, 7)
    for f in ref:
        assert same_bits(host(out[f]), ref[f])


def test_mirror_vs_reference_library_over_the_high_words(ft):
    """K3's oracle against the unmodified reference over the whole binary64
    range: every 32nd high word (2^27 doubles: every sign and exponent, 15 top
    mantissa bits, seeded random low words) evaluated by the device restatement
    and by oracle/_ref on the host, all three functions and both segment
    choices bit for bit, in the default SqrtMode and in exact mode."""
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    n = 1 << 27
    gen = torch.Generator(device="cuda").manual_seed(77)
    hi = torch.arange(0, 1 << 32, 32, dtype=torch.int64, device="cuda")
    lo = torch.randint(0, 1 << 32, (n,), dtype=torch.int64, device="cuda", generator=gen)
    xd = ((hi << 32) | lo).view(torch.float64)
    del hi, lo
    chunk = 1 << 25
    for m, s in ((1, 1), (0, 0)):
        out = ft.mirror_eval(xd, 7, 0, ft.SqrtMode(m, s), seg=True)
        torch.cuda.synchronize()
        for c0 in range(0, n, chunk):
            x = host(xd[c0:c0 + chunk])
            ref = O.proposed(x, 7, m, s, seg=True, impl="ref")
            for f in ("sin", "cos", "tan"):
                assert same_bits(host(out[f][c0:c0 + chunk]), ref[f]), (f, m, s, c0)
            assert np.array_equal(host(out["seg_sc"][c0:c0 + chunk]), ref["seg_sc"])
            assert np.array_equal(host(out["seg_t"][c0:c0 + chunk]), ref["seg_t"])
    # the Taylor restatement against the CPU port, same inputs
    out = ft.mirror_eval(xd, 7, 1, n_terms=5)
    torch.cuda.synchronize()
    for c0 in range(0, n, chunk):
        ref = O.taylor(host(xd[c0:c0 + chunk]), 5, 7)
        for f in ref:
            assert same_bits(host(out[f][c0:c0 + chunk]), ref[f]), ("taylor", f, c0)


def test_k3_with_host_oracle_arrays(ft):
    w = CONFIGS["cfg1"]
    x = O.gen_uniform(1 << 20, w.lo, w.hi, w.seed, 0, np.float32)
    xd = dev(x)
    out = ft.proposed_eval(xd, 7, seg=True)
    ref = O.proposed(x, 7)
    st = ft.parity_reduce(xd, out, 7, refs={f: dev(ref[f]) for f in ref}, ulp_tol=ULP_TOL)
    assert st["n_checked"] == x.size
    assert st["max_ulp"] == [0, 0, 0] and st["n_over_tol"] == [0, 0, 0]
    # checksum = wrap-around sum of the output bit patterns
    for j, f in enumerate(("sin", "cos", "tan")):
        assert st["checksum"][j] == int(ref[f].view(np.uint32).astype(np.uint64).sum()) % (1 << 64)
    # an injected 1-ulp / 3-ulp error is seen
    bad = out["sin"].clone()
    bad[5] = torch.from_numpy(np.nextafter(ref["sin"][5:6], np.float32(np.inf))).cuda()[0]
    bad[9] = torch.from_numpy(ref["sin"][9:10].view(np.int32) + 3).view(torch.float32).cuda()[0]
    st = ft.parity_reduce(xd, {"sin": bad}, 1, refs={"sin": dev(ref["sin"])}, ulp_tol=ULP_TOL)
    assert st["max_ulp"][0] == 3 and st["n_over_tol"][0] == 1


def test_k3_full_cfg2_parity_and_paper_bounds(ft):
    """configs[1] at full size (2^28 f64): zero mismatches against the device
    restatement, identical segments, and the paper's error bounds vs libm."""
    w = CONFIGS["cfg2"]
    xd = ft.gen_inputs(w.n, torch.float64, 0, w.lo, w.hi, w.seed)
    out = ft.proposed_eval(xd, 7, seg=True)
    st = ft.parity_reduce(xd, out, 7, ulp_tol=ULP_TOL, check_seg=True)
    assert st["n_checked"] == w.n
    assert st["max_ulp"] == [0, 0, 0] and st["seg_mismatch"] == [0, 0]
    assert st["n_nan"] == [0, 0, 0]
    # sin/cos abs max vs libm ~1.5317e-3 (0.001532); tan rel ~6.4e-3
    assert abs(st["max_abs_vs_libm"][0] - 1.5317e-3) < 2e-6
    assert abs(st["max_abs_vs_libm"][1] - 1.5317e-3) < 2e-6
    assert st["max_rel_vs_libm"][2] < 6.5e-3
    # cross-check a sample against the CPU oracle
    idx = slice(12345678, 12345678 + (1 << 18))
    x = host(xd[idx])
    check_against(x, {k: v[idx] for k, v in out.items()}, O.proposed(x, 7, seg=True))


def test_full_cfg2_production_kernel_vs_reference_library(ft):
    """configs[1] at full size through the production kernel (fused, no segment
    output: TMA bulk stores), every one of the 2^28 x 3 outputs compared bit for
    bit with the unmodified reference library on the host cores (chunks of 2^25
    elements) -- no device-side oracle involved."""
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    w = CONFIGS["cfg2"]
    xd = ft.gen_inputs(w.n, torch.float64, 0, w.lo, w.hi, w.seed)
    out = ft.proposed_eval(xd, 7)
    torch.cuda.synchronize()
    chunk = 1 << 25
    for lo in range(0, w.n, chunk):
        x = host(xd[lo:lo + chunk])
        ref = O.proposed(x, 7, impl="ref")
        for f in ("sin", "cos", "tan"):
            assert same_bits(host(out[f][lo:lo + chunk]), ref[f]), (f, lo)


def test_full_cfg4_f64_taylor_vs_cpu_oracle(ft):
    """configs[3] f64 at full size (2^28, Taylor-5 sin+cos, the TMA-store K2)
    against the CPU restatement of SPEC.md:224-256, bit for bit."""
    w = CONFIGS["cfg4_f64"]
    xd = ft.gen_inputs(w.n, torch.float64, 0, w.lo, w.hi, w.seed)
    out = ft.taylor_eval(xd, w.n_terms, w.mask)
    torch.cuda.synchronize()
    chunk = 1 << 25
    for lo in range(0, w.n, chunk):
        x = host(xd[lo:lo + chunk])
        ref = O.taylor(x, w.n_terms, w.mask)
        for f in ref:
            assert same_bits(host(out[f][lo:lo + chunk]), ref[f]), (f, lo)


def test_tan_stress_cfg3_full(ft):
    """configs[2]: 2^26 f32 near the poles; device-generated x copied to the host
    oracle; bitwise parity, +-inf count (~68%), finite max error vs libm."""
    w = CONFIGS["cfg3"]
    xd = ft.gen_inputs(w.n, torch.float32, 1, w.lo, w.hi, w.seed)
    out = ft.proposed_eval(xd, 4, seg=True)
    x = host(xd)
    d = x.astype(np.float64)
    k = np.round((d - 0.5 * math.pi) / math.pi)
    assert np.all(np.abs(d - (k * math.pi + 0.5 * math.pi)) <= 0.0501)
    ref = O.proposed(x, 4, seg=True)
    check_against(x, out, ref, fns=("tan",))
    st = ft.parity_reduce(xd, out, 4, ulp_tol=ULP_TOL)
    frac_inf = st["n_inf"][2] / w.n
    assert 0.6 < frac_inf < 0.75
    assert st["max_ulp"][2] == 0


def test_cfg5_sharded_equals_unsharded(ft):
    """configs[4] host logic on one GPU: 8 contiguous shards generated in place
    (global index as the counter) give the same checksums and maxima as one pass,
    and the full 2^33 array (8 shards of 2^30) has zero mismatches."""
    w = CONFIGS["cfg5"]
    n = 1 << 28
    xd = ft.gen_inputs(n, torch.float32, 0, w.lo, w.hi, w.seed)
    whole = ft.parity_reduce(xd, ft.proposed_eval(xd, 7), 7, ulp_tol=ULP_TOL)
    del xd
    parts = []
    for r in range(8):
        lo, hi = shard(n, r, 8)
        xs = ft.gen_inputs(hi - lo, torch.float32, 0, w.lo, w.hi, w.seed, lo)
        parts.append(ft.parity_reduce(xs, ft.proposed_eval(xs, 7), 7, ulp_tol=ULP_TOL))
    for j in range(3):
        assert sum(p["checksum"][j] for p in parts) % (1 << 64) == whole["checksum"][j]
        assert max(p["max_abs_vs_libm"][j] for p in parts) == whole["max_abs_vs_libm"][j]
        assert sum(p["n_inf"][j] for p in parts) == whole["n_inf"][j]
    # full-size cfg5 parity, shard by shard (2^30 elements each)
    total = 0
    for r in range(8):
        lo, hi = shard(w.n, r, 8)
        xs = ft.gen_inputs(hi - lo, torch.float32, 0, w.lo, w.hi, w.seed, lo)
        st = ft.parity_reduce(xs, ft.proposed_eval(xs, 7), 7, ulp_tol=ULP_TOL)
        assert st["max_ulp"] == [0, 0, 0], r
        total += st["n_checked"]
        del xs
        torch.cuda.empty_cache()
    assert total == w.n


def test_host_batch_api(ft):
    p = PAPER_PROTOCOL
    x = O.gen_uniform(p.n, p.lo, p.hi, p.seed)
    ref = O.proposed(x, 7)
    assert same_bits(ft.proposed_sin_batch(x), ref["sin"])
    assert same_bits(ft.proposed_cos_batch(x), ref["cos"])
    assert same_bits(ft.proposed_tan_batch(x), ref["tan"])
    assert ft.proposed_sin_batch(np.empty(0)).size == 0
    # chunked pipeline across several chunks, f32 fused
    w = CONFIGS["cfg1"]
    xf = O.gen_uniform((1 << 24) + 77, w.lo, w.hi, w.seed, 0, np.float32)
    r = ft.proposed_batch(xf, 7)
    ref = O.proposed(xf, 7)
    for f in ref:
        assert same_bits(r[f], ref[f])
    t = ft.taylor_batch(xf[:100000], 5, 3)
    ref = O.taylor(xf[:100000], 5, 3)
    for f in ref:
        assert same_bits(t[f], ref[f])


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_host_staged_path_misaligned_views_and_guard_bands(ft, dtype):
    """Pageable buffers at odd element offsets (destinations not 64-byte aligned,
    sizes not multiples of the copy block or the staging chunk) through the staged
    host path, whose pool copies use non-temporal stores on an aligned middle
    part: results bitwise equal to the oracle, nothing written outside the views."""
    n = (5 << 20) + 12345  # three staging chunks, ragged tail
    w = CONFIGS["cfg2"]
    base = O.gen_uniform(n + 64, w.lo, w.hi, w.seed).astype(dtype)
    canary = dtype(-777.25)
    for xo, oo in ((1, 3), (7, 0), (0, 5)):
        x = base[xo:xo + n]
        bufs = {nm: np.full(n + 64, canary, dtype) for nm in ("sin", "cos", "tan")}
        outs = {nm: b[oo:oo + n] for nm, b in bufs.items()}
        ft.proposed_batch(x, 7, out=outs)
        ref = O.proposed(np.ascontiguousarray(x), 7)
        for nm, b in bufs.items():
            assert same_bits(outs[nm], ref[nm]), (nm, xo, oo)
            assert np.all(b[:oo] == canary) and np.all(b[oo + n:] == canary), (nm, xo, oo)
    # a single-output reference-shaped call on the same kind of view
    x = base[3:3 + n].astype(np.float64)
    assert same_bits(ft.proposed_tan_batch(x), O.proposed(x, 4)["tan"])


def test_paper_protocol_bounds_from_gpu(ft):
    """PAPER.md:240 protocol through the GPU path; host glibc as the reference."""
    p = PAPER_PROTOCOL
    x = O.gen_uniform(p.n, p.lo, p.hi, p.seed)
    r = ft.proposed_batch(x, 7)
    se = np.abs(r["sin"] - np.sin(x))
    assert abs(se.max() - 0.001532) < 5e-7
    te = np.abs(r["tan"] - np.tan(x)) / np.abs(np.tan(x))
    assert abs(te.max() - 0.006394) < 5e-7


def test_cpp_dropin_program(ft, tmp_path):
    exe = tmp_path / "test_gpu_api"
    libdir = os.path.join(ROOT, "paper_2502_10831_b200", "lib")
    subprocess.run(["g++", "-std=c++20", "-O2", "-I" + os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "test_gpu_api.cpp"), "-L" + libdir,
                    "-lfasttrig_b200", "-Wl,-rpath," + libdir, "-o", str(exe)], check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr


def test_launch_counter_counts_kernels(ft):
    before = ft.launch_count()
    x = ft.gen_inputs(1000, torch.float32, 0, 0.0, 1.0, 1)
    ft.proposed_eval(x, 7)
    ft.taylor_eval(x, 5, 3)
    torch.cuda.synchronize()
    assert ft.launch_count() - before == 3


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_no_out_of_bounds_writes(ft, dtype):
    """compute-sanitizer is closed on this pool, so bounds are checked directly:
    every output (and the segment arrays) is a view into a larger buffer filled
    with a canary; after K1 / K2 / K4 the canary outside each view is intact."""
    guard = 4099
    canary = -12345.678 if dtype == torch.float64 else -1234.5
    for n in (1, 3, 17, 4096, 20011):
        for off in (0, 1, 2):
            x = ft.gen_inputs(n + off, dtype, 0, -500.0, 500.0, 11)[off:]
            bufs = {nm: torch.full((n + 2 * guard + off,), canary, dtype=dtype, device="cuda")
                    for nm in ("sin", "cos", "tan")}
            views = {nm: b[guard + off: guard + off + n] for nm, b in bufs.items()}
            ft.proposed_eval(x, 7, out=views)
            ft.taylor_eval(x, 5, 7, out=views)
            gbuf = torch.full((n + 2 * guard + off,), canary, dtype=dtype, device="cuda")
            ft.gen_inputs(n, dtype, 0, 0.0, 1.0, 3, out=gbuf[guard + off: guard + off + n])
            torch.cuda.synchronize()
            for b in list(bufs.values()) + [gbuf]:
                h = b.cpu().numpy()
                assert np.all(h[: guard + off] == np.array(canary, h.dtype)), (n, off)
                assert np.all(h[guard + off + n:] == np.array(canary, h.dtype)), (n, off)


def test_arrays_longer_than_one_launch(ft):
    """Launches are split at 2^30 elements (32-bit in-kernel indexing): results
    on both sides of every split point equal the oracle and the launch count
    reflects the split."""
    n = (1 << 30) + 4099
    w = CONFIGS["cfg5"]
    xd = ft.gen_inputs(n, torch.float32, 0, w.lo, w.hi, w.seed, 77)
    before = ft.launch_count()
    out = ft.proposed_eval(xd, 7)
    torch.cuda.synchronize()
    assert ft.launch_count() - before == 2
    for lo, hi in ((0, 4096), ((1 << 30) - 4096, n)):
        x = host(xd[lo:hi])
        ref = O.proposed(x, 7)
        for f in ref:
            assert same_bits(host(out[f][lo:hi]), ref[f]), (lo, f)
    st = ft.parity_reduce(xd, out, 7, ulp_tol=ULP_TOL)
    assert st["n_checked"] == n and st["max_ulp"] == [0, 0, 0]


@pytest.mark.parametrize("mode", list(MODES) + ["fisr3"])
def test_host_batch_api_every_sqrt_mode(ft, mode):
    """The reference-shaped host API (kernels.hpp:84-94) in every SqrtMode, f64 and
    f32, on the golden edge cases: bitwise equal to the oracle."""
    m, s = MODES.get(mode, (1, 3))
    sm = ft.SqrtMode(m, s)
    x = np.concatenate([np.linspace(-20, 20, 40001), [0.0, -0.0, np.inf, -np.inf, np.nan, 1e300, -1e-310]])
    ref = O.proposed(x, 7, m, s)
    assert same_bits(ft.proposed_sin_batch(x, sm), ref["sin"])
    assert same_bits(ft.proposed_cos_batch(x, sm), ref["cos"])
    assert same_bits(ft.proposed_tan_batch(x, sm), ref["tan"])
    with np.errstate(over="ignore"):
        xf = x.astype(np.float32)  # 1e300 -> inf on purpose
    r = ft.proposed_batch(xf, 7, sm)
    ref = O.proposed(xf, 7, m, s)
    for f in ref:
        assert same_bits(r[f], ref[f]), f


@pytest.mark.parametrize("lo", [0x00000000, 0xFFFFFFFF, 0x80000000, 0x00000001, 0x5A5A5A5A])
def test_every_f64_high_word_production_kernel(ft, lo):
    """All 2^32 doubles with the given low word -- every sign, exponent and
    top-20-bit mantissa, incl. subnormals, infinities and NaNs: every value the
    fast path's high-word compares (quadrant thresholds, row brackets, guard) can
    see -- through the production fused f64 kernel (TMA bulk stores), K3 against
    the device restatement: 0 raw-bit mismatches.  (tools/f64_hiword_sweep.py
    runs 64 low words in every SqrtMode: profiles/r02cd_f64_hiword.jsonl.)"""
    chunk = 1 << 28
    out = None
    nan = 0
    for start in range(0, 1 << 32, chunk):
        hi = torch.arange(start, start + chunk, dtype=torch.int64, device="cuda")
        x = ((hi << 32) | lo).view(torch.float64)
        del hi
        if out is None:
            out = {nm: torch.empty_like(x) for nm in ("sin", "cos", "tan")}
        ft.proposed_eval(x, 7, out=out)
        st = ft.parity_reduce(x, out, 7, ulp_tol=0)
        assert st["n_checked"] == chunk
        assert st["n_bit_mismatch"] == [0, 0, 0] and st["max_ulp"] == [0, 0, 0], (hex(start), hex(lo))
        nan += st["n_nan"][0]
    assert nan == 2 * (1 << 20)  # exponent 0x7ff, either sign: infinities and NaNs give NaN (reduction.hpp:60-62)


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_random_bit_patterns_full_range(ft, dtype):
    """2^26 uniformly random bit patterns (every exponent and sign, incl. subnormals,
    huge arguments, NaN/inf) through K1, checked by K3 against the device
    restatement (itself bitwise-pinned to the CPU oracle) in every SqrtMode."""
    n = 1 << 26
    gen = torch.Generator(device="cuda").manual_seed(1234)
    if dtype == torch.float64:
        bits = torch.randint(-(2**63), 2**63 - 1, (n,), dtype=torch.int64, device="cuda", generator=gen)
    else:
        bits = torch.randint(-(2**31), 2**31 - 1, (n,), dtype=torch.int32, device="cuda", generator=gen)
    x = bits.view(dtype)
    for m, s in ((1, 1), (0, 0), (1, 2)):
        mode = ft.SqrtMode(m, s)
        out = ft.proposed_eval(x, 7, mode, seg=True)
        st = ft.parity_reduce(x, out, 7, mode=mode, ulp_tol=ULP_TOL, check_seg=True)
        assert st["n_checked"] == n
        assert st["max_ulp"] == [0, 0, 0], (m, s, st["max_ulp"])
        assert st["n_bit_mismatch"] == [0, 0, 0]
        assert st["seg_mismatch"] == [0, 0]
        prod = ft.proposed_eval(x, 7, mode)  # production instantiation (f64: TMA bulk stores)
        st = ft.parity_reduce(x, prod, 7, mode=mode, ulp_tol=ULP_TOL)
        assert st["n_bit_mismatch"] == [0, 0, 0], (m, s)
    # the mirror is K3's oracle and the fast path's fallback: pin a sample of the
    # elements that take that fallback (|x| >= 2^24 * 2pi, non-finite, tiny)
    # directly to the unmodified reference on the host
    xh = host(x)
    with np.errstate(invalid="ignore"):
        a = np.abs(xh.astype(np.float64))
        slow = ~(a < 2.0**24 * 2 * math.pi) | (a < 2.0**-17)
    idx = np.flatnonzero(slow)[: 1 << 22]
    assert idx.size > (1 << 20)
    xs = np.ascontiguousarray(xh[idx])
    ref = O.proposed(xs, 7, 1, 2, impl="ref" if O.ref_available() else "port")  # the loop's last mode
    for m_out in (prod, out):
        for f in ("sin", "cos", "tan"):
            assert same_bits(host(m_out[f])[idx], ref[f]), f


@pytest.mark.parametrize("devices", [2, 3, 0])
def test_host_api_sharded_over_devices(ft, devices):
    """ft_set_host_devices: one host call split into shards, one host thread and
    device pipeline each (on a single-GPU box the shards share the device), both
    for pinned and pageable buffers; bitwise equal to the oracle."""
    w = CONFIGS["cfg2"]
    n = (1 << 24) + 12345
    x = O.gen_uniform(n, w.lo, w.hi, w.seed, 0)
    ref = O.proposed(x, 7)
    try:
        ft.set_host_devices(devices)
        r = ft.proposed_batch(x, 7)  # pageable numpy buffers
        for f in ref:
            assert same_bits(r[f], ref[f]), f
        xp = torch.from_numpy(x).pin_memory()
        outs = {f: torch.empty(n, dtype=torch.float64, pin_memory=True).numpy() for f in ref}
        ft.proposed_batch(xp.numpy(), 7, out=outs)
        for f in ref:
            assert same_bits(outs[f], ref[f]), f
        t = ft.taylor_batch(x.astype(np.float32), 5, 3)
        tr = O.taylor(x.astype(np.float32), 5, 3)
        for f in tr:
            assert same_bits(t[f], tr[f]), f
    finally:
        ft.set_host_devices(1)


def test_concurrent_callers(ft):
    """Several host threads on their own streams, mixing device-pointer and
    host-pointer calls at the same time (the C ABI's occupancy cache, launch
    counter, host pipelines and error strings are shared state)."""
    import threading

    w = CONFIGS["cfg2"]
    x = O.gen_uniform(1 << 20, w.lo, w.hi, w.seed, 4242)
    ref = O.proposed(x, 7)
    xd = dev(x)
    errors = []

    def device_worker(k):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                for _ in range(5):
                    out = ft.proposed_eval(xd, 7, stream=s)
                    s.synchronize()
                    for f in ref:
                        assert same_bits(host(out[f]), ref[f])
        except Exception as e:  # noqa: BLE001
            errors.append(repr(e))

    def host_worker(k):
        try:
            for _ in range(3):
                r = ft.proposed_batch(x, 7)
                for f in ref:
                    assert same_bits(r[f], ref[f])
                bad = None
                try:
                    ft.taylor_batch(x, 99, 3)
                except Exception as e:  # noqa: BLE001
                    bad = str(e)
                assert bad and "n_terms" in bad  # this thread's own error text
        except Exception as e:  # noqa: BLE001
            errors.append(repr(e))

    th = [threading.Thread(target=device_worker, args=(k,)) for k in range(4)]
    th += [threading.Thread(target=host_worker, args=(k,)) for k in range(3)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    assert not errors, errors


def test_device_tables_read_back_bitwise(ft):
    """the constant tables as the GPU holds them -- the __constant__
    copy of every translation unit and the shared-memory rows the K1 kernels
    stage (bit-exact and relaxed), copied out by a kernel -- carry the reference's
    segment_table bits (R:segments.hpp:33-66) and the documented brackets."""
    ref = O.segment_table("ref" if O.ref_available() else "port")
    for unit in range(4):
        assert same_bits(ft.device_const_table(unit), ref), unit
    coef = ref[:42].reshape(6, 7)
    knots = ref[42:]
    hi = lambda v: int(np.int64(np.float64(v).view(np.int64)) >> 32)  # noqa: E731
    rows = ft.device_rows(0)
    for i in range(8):
        k = min(i, 5)
        got = np.array([rows[i][f] for f in ("a", "b", "c", "d", "X", "Y", "Z")])
        assert same_bits(got, coef[k]), i
        klo = hi(2.0**-17) if i == 0 else 0 if i >= 6 else hi(knots[k])
        khi = hi(0.5 * math.pi) if i == 5 else 0 if i >= 6 else hi(knots[k + 1])
        assert (int(rows[i]["klo_hi"]), int(rows[i]["khi_hi"])) == (klo, khi), i
    for mask in range(1, 8):
        rr = ft.device_rows(mask)
        for i in range(8):
            k = min(i, 5)
            got = np.array([rr[i][f] for f in ("a", "b", "c", "d")])
            assert same_bits(got, coef[k][:4]), (mask, i)
            lo_needed = bool(mask & 5)
            cos_in = bool(mask & 2)
            klo = 0x7FFFFFFF if i >= 6 else (hi(2.0**-11) if lo_needed else -1) if i == 0 else hi(knots[k])
            khi = 0 if i >= 6 else (hi(0.5 * math.pi - 2.0**-11) if cos_in else hi(0.5 * math.pi)) if i == 5 \
                else hi(knots[k + 1])
            assert (int(rr[i]["klo_hi"]), int(rr[i]["khi_hi"])) == (klo, khi), (mask, i)


def test_launches_capture_into_cuda_graph(ft):
    """The K1/K2 launches (cudaLaunchKernelEx with programmatic dependent launch)
    are stream-capturable: a CUDA graph of fused proposed + Taylor steps replays
    to the same bits as eager launches."""
    w = CONFIGS["cfg2"]
    x64 = ft.gen_inputs(1 << 20, torch.float64, 0, w.lo, w.hi, w.seed)
    x32 = (x64 * 0.01).float()
    eager = {"p64": ft.proposed_eval(x64, 7), "p32": ft.proposed_eval(x32, 7), "t32": ft.taylor_eval(x32, 5, 3)}
    torch.cuda.synchronize()
    outs = {"p64": {nm: torch.empty_like(x64) for nm in ("sin", "cos", "tan")},
            "p32": {nm: torch.empty_like(x32) for nm in ("sin", "cos", "tan")},
            "t32": {nm: torch.empty_like(x32) for nm in ("sin", "cos")}}
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        ft.proposed_eval(x64, 7, out=outs["p64"], stream=s)  # warm-up outside capture
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            for _ in range(3):
                ft.proposed_eval(x64, 7, out=outs["p64"], stream=s)
                ft.proposed_eval(x32, 7, out=outs["p32"], stream=s)
                ft.taylor_eval(x32, 5, 3, out=outs["t32"], stream=s)
    for o in outs.values():
        for t in o.values():
            t.zero_()
    g.replay()
    torch.cuda.synchronize()
    for k in eager:
        for nm, t in eager[k].items():
            assert torch.equal(t.view(torch.int64 if t.dtype == torch.float64 else torch.int32),
                               outs[k][nm].view(torch.int64 if t.dtype == torch.float64 else torch.int32)), (k, nm)
