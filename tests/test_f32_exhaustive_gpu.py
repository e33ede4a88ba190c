"""The default f32 policy (FT_F32_ULP2) and the bit-exact one over EVERY float.

The reference is double-only; for f32 inputs its result is
(float)proposed_*((double)x) (R:proj/include/fasttrig/kernels.hpp:46-67).  The
f32 domain has 2^32 inputs, so parity here is proven, not sampled:

* the production relaxed kernels (ft_core.cuh relaxed_*) against the production
  bit-exact kernels, all 2^32 bit patterns, through K3 with the bit-exact outputs
  as the oracle arrays: <= 2 ulp (the north-star tolerance; <= 1 observed) and
  identical segment choices (SEG instantiations compared element for element);
* the production bit-exact kernels against the device restatement (K3, 0 ulp);
* both, for fisr(1) and all three outputs, against the UNMODIFIED reference
  library on the host (oracle/_ref, all host threads): values and segments.
"""
from __future__ import annotations

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

MODES = {"fisr1": (1, 1), "exact": (0, 0), "fisr2": (1, 2), "fisr0": (1, 0), "fisr3": (1, 3)}
# every mask in the default mode and exact; the other sqrt modes (unrolled fisr(2),
# the runtime-step kernel for fisr(0) / fisr(3)) on the fused mask
CASES = ([(m, "fisr1") for m in (7, 3, 4, 1, 2, 5, 6)] + [(m, "exact") for m in (7, 3, 4)]
         + [(7, "fisr2"), (7, "fisr0"), (7, "fisr3")])
CHUNK = 1 << 28
ALL = 1 << 32


def chunk_bits(start: int, n: int):
    """float32 CUDA tensor whose bit patterns are start .. start+n-1."""
    s = start - (1 << 32) if start >= (1 << 31) else start
    b = torch.arange(n, dtype=torch.int32, device="cuda")
    b.add_(s)
    return b.view(torch.float32)


def _stats_buf():
    return torch.zeros(312, dtype=torch.uint8, device="cuda")


@pytest.mark.parametrize("mask,mode", CASES)
def test_every_float_relaxed_within_2ulp_same_segments(ft, mask, mode):
    sm = ft.SqrtMode(*MODES[mode])
    buf = _stats_buf()
    max_ulp, over, seg_mm, checked = [0, 0, 0], [0, 0, 0], [0, 0], 0
    for start in range(0, ALL, CHUNK):
        x = chunk_bits(start, CHUNK)
        with ft.f32_policy("ulp2"):
            got = ft.proposed_eval(x, mask, sm)
        with ft.f32_policy("bitwise"):
            ref = ft.proposed_eval(x, mask, sm)
        st = ft.parity_reduce(x, got, mask, mode=sm, refs=ref, ulp_tol=2, stats_buf=buf)
        checked += st["n_checked"]
        for j in range(3):
            max_ulp[j] = max(max_ulp[j], st["max_ulp"][j])
            over[j] += st["n_over_tol"][j]
        del got, ref
        with ft.f32_policy("ulp2"):
            gs = ft.proposed_eval(x, mask, sm, seg=True)
        with ft.f32_policy("bitwise"):
            rs = ft.proposed_eval(x, mask, sm, seg=True)
        seg_mm[0] += int((gs["seg_sc"] != rs["seg_sc"]).sum())
        seg_mm[1] += int((gs["seg_t"] != rs["seg_t"]).sum())
        del gs, rs
    assert checked == ALL
    assert over == [0, 0, 0] and max(max_ulp) <= 2, max_ulp
    assert seg_mm == [0, 0]


@pytest.mark.parametrize("mask", [3, 7])
@pytest.mark.parametrize("nt", [5, 7, 9])
def test_every_float_relaxed_taylor_within_2ulp(ft, nt, mask):
    buf = _stats_buf()
    max_ulp, over = [0, 0, 0], [0, 0, 0]
    for start in range(0, ALL, CHUNK):
        x = chunk_bits(start, CHUNK)
        with ft.f32_policy("ulp2"):
            got = ft.taylor_eval(x, nt, mask)
        with ft.f32_policy("bitwise"):
            ref = ft.taylor_eval(x, nt, mask)
        st = ft.parity_reduce(x, got, mask, kind=1, n_terms=nt, refs=ref, ulp_tol=2, stats_buf=buf)
        for j in range(3):
            max_ulp[j] = max(max_ulp[j], st["max_ulp"][j])
            over[j] += st["n_over_tol"][j]
    assert over == [0, 0, 0] and max(max_ulp) <= 2, max_ulp


@pytest.mark.parametrize("case", ["fisr1-7", "fisr1-3", "fisr1-4", "exact-7", "taylor5-3"])
def test_every_float_bitwise_production_vs_restatement(ft, case):
    """The production (non-SEG) bit-exact kernels against the device restatement
    (itself pinned to the CPU oracle): 0 ulp and identical bits on every float."""
    kind, mask = case.split("-")
    mask = int(mask)
    buf = _stats_buf()
    tot = {"max_ulp": [0, 0, 0], "bits": [0, 0, 0]}
    for start in range(0, ALL, CHUNK):
        x = chunk_bits(start, CHUNK)
        with ft.f32_policy("bitwise"):
            if kind == "taylor5":
                out = ft.taylor_eval(x, 5, mask)
                st = ft.parity_reduce(x, out, mask, kind=1, n_terms=5, ulp_tol=0, stats_buf=buf)
            else:
                sm = ft.SqrtMode(*MODES[kind])
                out = ft.proposed_eval(x, mask, sm)
                st = ft.parity_reduce(x, out, mask, mode=sm, ulp_tol=0, stats_buf=buf)
        for j in range(3):
            tot["max_ulp"][j] = max(tot["max_ulp"][j], st["max_ulp"][j])
            tot["bits"][j] += st["n_bit_mismatch"][j]
    assert tot["max_ulp"] == [0, 0, 0] and tot["bits"] == [0, 0, 0], tot


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("policy", ["bitwise", "ulp2"])
def test_every_float_vs_reference_library(ft, policy):
    """fisr(1), all three outputs and both segment choices, every float, against
    the unmodified reference compiled on the host (oracle/_ref)."""
    n = 1 << 26
    hs = {f: torch.empty(n, dtype=torch.float32, pin_memory=True) for f in ("sin", "cos", "tan")}
    hg = {f: torch.empty(n, dtype=torch.uint8, pin_memory=True) for f in ("seg_sc", "seg_t")}
    tot = {"max_ulp": [0, 0, 0], "n_bit_mismatch": [0, 0, 0], "n_over_2ulp": [0, 0, 0], "seg_mismatch": [0, 0]}
    for start in range(0, ALL, n):
        x = chunk_bits(start, n)
        with ft.f32_policy(policy):
            out = ft.proposed_eval(x, 7)
            seg = ft.proposed_eval(x, 7, seg=True)
        for f in hs:
            hs[f].copy_(out[f])
        for f in hg:
            hg[f].copy_(seg[f])
        torch.cuda.synchronize()
        r = O.ref_check_f32_range(start, {**{f: hs[f].numpy() for f in hs}, **{f: hg[f].numpy() for f in hg}})
        for j in range(3):
            tot["max_ulp"][j] = max(tot["max_ulp"][j], r["max_ulp"][j])
            tot["n_bit_mismatch"][j] += r["n_bit_mismatch"][j]
            tot["n_over_2ulp"][j] += r["n_over_2ulp"][j]
        for j in range(2):
            tot["seg_mismatch"][j] += r["seg_mismatch"][j]
    print(policy, tot)
    assert tot["seg_mismatch"] == [0, 0]
    assert tot["n_over_2ulp"] == [0, 0, 0]
    if policy == "bitwise":
        assert tot["n_bit_mismatch"] == [0, 0, 0] and tot["max_ulp"] == [0, 0, 0]
    else:
        assert max(tot["max_ulp"]) <= 2


def _ulp32(a: np.ndarray, b: np.ndarray) -> int:
    ia, ib = a.view(np.int32).astype(np.int64), b.view(np.int32).astype(np.int64)
    oa = np.where(ia < 0, -(ia & 0x7FFFFFFF), ia)
    ob = np.where(ib < 0, -(ib & 0x7FFFFFFF), ib)
    na, nb = np.isnan(a), np.isnan(b)
    d = np.abs(oa - ob)
    d[na & nb] = 0
    d[na ^ nb] = 1 << 40
    return int(d.max()) if d.size else 0


@pytest.mark.parametrize("mask", range(1, 8))
def test_relaxed_ragged_misaligned_every_mask(ft, mask):
    """The default-policy f32 kernels on offset views (unaligned pointers -> the
    scalar tail path) and ragged sizes: within 2 ulp of the oracle and equal to
    the aligned vectorised run of the same elements."""
    rng = np.random.default_rng(100 + mask)
    base = rng.uniform(-3e3, 3e3, 70001).astype(np.float32)
    full = ft.proposed_eval(torch.from_numpy(base).cuda(), mask)
    for off in (0, 1, 3):
        for n in (1, 2, 3, 5, 17, 1023, 4097, 70001 - off):
            xd = torch.from_numpy(base).cuda()[off:off + n]
            out = {nm: torch.empty(n + 1, dtype=torch.float32, device="cuda")[1:n + 1]
                   for j, nm in enumerate(("sin", "cos", "tan")) if mask & (1 << j)}
            ft.proposed_eval(xd, mask, out=out)
            torch.cuda.synchronize()
            ref = O.proposed(base[off:off + n], mask)
            for f in out:
                g = out[f].cpu().numpy()
                assert _ulp32(g, ref[f]) <= 2, (off, n, f)
                assert np.array_equal(g.view(np.uint32), full[f][off:off + n].cpu().numpy().view(np.uint32))


def test_relaxed_golden_vectors_and_segments(ft, golden):
    """Every f32 golden vector (edge cases, knots +- ulps, quadrant edges, pole
    guard, +-0, huge, non-finite) in every SqrtMode of the fixture: within 2 ulp
    of the reference's outputs and the identical segment choices."""
    from conftest import MODES as GM, golden_cases

    n = 0
    for case, mode, x, ref in golden_cases(golden):
        if x.dtype != np.float32:
            continue
        out = ft.proposed_eval(torch.from_numpy(x).cuda(), 7, ft.SqrtMode(*GM[mode]), seg=True)
        torch.cuda.synchronize()
        for f in ("sin", "cos", "tan"):
            assert _ulp32(out[f].cpu().numpy(), ref[f]) <= 2, (case, mode, f)
        assert np.array_equal(out["seg_sc"].cpu().numpy(), ref["seg_sc"]), (case, mode)
        assert np.array_equal(out["seg_t"].cpu().numpy(), ref["seg_t"]), (case, mode)
        n += x.size
    assert n > 5000


@pytest.mark.parametrize("mask", [7, 4, 3])
def test_relaxed_range_dispatch_mixed_warps(ft, mask):
    """Warps holding any |x| >= 2^16 evaluate their vector bit-exactly (the
    range dispatch of the relaxed kernels): dense and sparse large arguments,
    NaN and infinities mixed into small ones -- within 2 ulp of the oracle and,
    for the all-large vectors, bitwise equal to the bit-exact policy; Taylor too."""
    rng = np.random.default_rng(7 + mask)
    n = 1 << 20
    small = rng.uniform(-300.0, 300.0, n).astype(np.float32)
    cases = {}
    x = small.copy()
    x[::4] = rng.uniform(-1e7, 1e7, n // 4).astype(np.float32)  # every vector has a large lane
    cases["dense"] = x
    x = small.copy()
    idx = rng.choice(n, n // 997, replace=False)
    x[idx] = rng.uniform(-1e6, 1e6, idx.size).astype(np.float32)
    x[idx[:50]] = np.array([np.inf, -np.inf, np.nan, 65536.0, -65535.99] * 10, np.float32)
    cases["sparse"] = x
    for name, x in cases.items():
        xd = torch.from_numpy(x).cuda()
        got = ft.proposed_eval(xd, mask)
        with ft.f32_policy("bitwise"):
            bit = ft.proposed_eval(xd, mask)
        ref = O.proposed(x, mask)
        big = ~(np.abs(x) < 65536.0)
        one = {f: np.concatenate([ft.proposed_eval(xd[i:i + 1], mask)[f].cpu().numpy()
                                  for i in range(0, 64)]) for f in got}  # scalar path, one element each
        for f in got:
            g = got[f].cpu().numpy()
            assert _ulp32(g, ref[f]) <= 2, (name, f)
            # large arguments are bit-exact; every element is what the scalar path gives it
            assert np.array_equal(g[big].view(np.uint32), bit[f].cpu().numpy()[big].view(np.uint32)), f
            assert np.array_equal(g[:64].view(np.uint32), one[f].view(np.uint32)), (name, f)
        # the unaligned view runs the scalar path on every element: same bits
        buf = torch.empty(n + 1, dtype=torch.float32, device="cuda")
        buf[1:].copy_(xd)
        shifted = ft.proposed_eval(buf[1:], mask)
        for f in got:
            assert torch.equal(shifted[f].view(torch.int32), got[f].view(torch.int32)), (name, f)
        t = ft.taylor_eval(xd, 5, 3)
        tr = O.taylor(x, 5, 3)
        for f in t:
            assert _ulp32(t[f].cpu().numpy(), tr[f]) <= 2, (name, "taylor", f)
