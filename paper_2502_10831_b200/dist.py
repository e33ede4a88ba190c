"""Multi-GPU plumbing for the sharded path.

The path is an elementwise map: GPU g of G owns the contiguous shard
[g*N/G, (g+1)*N/G) of one global array, generated in place by K4 with the
global index as the generator counter, so no element data ever moves between
GPUs.  The only collective is the final reduction of the 312-byte K3 statistics
(ft_stats): maxima with MAX, counters and checksums with SUM.  Checksums are
wrap-around uint64 sums of output bit patterns, so any G gives the same value.

Works with any torch.distributed backend: NCCL on the B200 box, gloo in the
CPU tests (tests/test_dist_gloo.py).
"""
from __future__ import annotations

from .configs import shard  # noqa: F401  (re-exported: contiguous equal shards)

IMAX_FIELDS = ("max_ulp",)
MAX_FIELDS = ("max_abs_vs_oracle", "max_abs_vs_libm", "max_rel_vs_libm")
SUM_FIELDS = ("n_checked", "n_over_tol", "seg_mismatch", "n_inf", "n_nan", "n_finite_libm",
              "checksum", "n_bit_mismatch")
I64_MAX = (1 << 63) - 1
FSUM_FIELDS = ("sum_abs_vs_libm", "sum_rel_vs_libm")
U64 = 1 << 64


def _as_list(v):
    return list(v) if isinstance(v, (list, tuple)) else [v]


def _to_i64(u: int) -> int:
    return u - U64 if u >= (1 << 63) else u


def reduce_stats(st: dict, device=None, group=None) -> dict:
    """All-reduce one rank's ft_stats dict across the process group.

    max_ulp is reduced as int64 MAX after clamping to 2^63-1 (K3 reports ~0 --
    2^64-1 -- when exactly one side is NaN; the clamp keeps it "huge"), the other
    maxima (non-negative doubles) as float64 MAX, counters and checksums as int64
    SUM with two's-complement wrap (== uint64 wrap-around), float sums as float64
    SUM.  Fields missing from `st` are treated as zero.  Returns a new dict with
    the same keys and shapes."""
    import torch
    import torch.distributed as dist

    dev = device if device is not None else "cpu"
    st = dict(st)
    st.setdefault("n_bit_mismatch", [0, 0, 0])
    imaxv, maxv, sumv, fsumv, shape = [], [], [], [], {}
    for k in IMAX_FIELDS:
        vals = _as_list(st[k])
        shape[k] = (len(vals), isinstance(st[k], (list, tuple)))
        imaxv += [min(int(v), I64_MAX) for v in vals]
    for k in MAX_FIELDS:
        vals = _as_list(st[k])
        shape[k] = (len(vals), isinstance(st[k], (list, tuple)))
        maxv += [float(v) for v in vals]
    for k in SUM_FIELDS:
        vals = _as_list(st[k])
        shape[k] = (len(vals), isinstance(st[k], (list, tuple)))
        sumv += [_to_i64(int(v) % U64) for v in vals]
    for k in FSUM_FIELDS:
        vals = _as_list(st[k])
        shape[k] = (len(vals), isinstance(st[k], (list, tuple)))
        fsumv += [float(v) for v in vals]
    ti = torch.tensor(imaxv, dtype=torch.int64, device=dev)
    tm = torch.tensor(maxv, dtype=torch.float64, device=dev)
    ts = torch.tensor(sumv, dtype=torch.int64, device=dev)
    tf = torch.tensor(fsumv, dtype=torch.float64, device=dev)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(ti, op=dist.ReduceOp.MAX, group=group)
        dist.all_reduce(tm, op=dist.ReduceOp.MAX, group=group)
        dist.all_reduce(ts, op=dist.ReduceOp.SUM, group=group)
        dist.all_reduce(tf, op=dist.ReduceOp.SUM, group=group)
    out = {}
    li, lm, ls, lf = ti.cpu().tolist(), tm.cpu().tolist(), ts.cpu().tolist(), tf.cpu().tolist()
    for keys, src, conv in ((IMAX_FIELDS, li, "int"), (MAX_FIELDS, lm, None), (SUM_FIELDS, ls, "u64"),
                            (FSUM_FIELDS, lf, None)):
        for k in keys:
            n, is_list = shape[k]
            vals, src[:] = src[:n], src[n:]
            if conv == "u64":
                vals = [int(v) % U64 for v in vals]
            elif conv == "int":
                vals = [int(v) for v in vals]
            out[k] = vals if is_list else vals[0]
    return out
