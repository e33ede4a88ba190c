"""N>1 host logic on CPU: world_size-2 `gloo` process group.

Each rank owns a contiguous shard of one global cfg5-recipe array, generated
from the global index (no data exchange), computes the K3 statistics of its
shard, and the ranks all-reduce them with paper_2502_10831_b200.dist.reduce_stats
(the code bench.py runs over NCCL).  The reduced statistics must equal the
unsharded ones: maxima, counts and wrap-around checksums exactly.
"""
from __future__ import annotations

import math
import os
import socket

import numpy as np
import pytest

from oracle import oracle as O
from paper_2502_10831_b200.configs import CONFIGS
from paper_2502_10831_b200.dist import reduce_stats, shard

N = 1 << 18


def host_stats(x: np.ndarray, out: dict, ref: dict) -> dict:
    """numpy restatement of the ft_stats fields K3 produces (for f32 outputs)."""
    st = {"n_checked": x.size, "max_ulp": [0, 0, 0], "n_over_tol": [0, 0, 0], "seg_mismatch": [0, 0],
          "n_inf": [0, 0, 0], "n_nan": [0, 0, 0], "n_finite_libm": [0, 0, 0], "checksum": [0, 0, 0],
          "max_abs_vs_oracle": [0.0] * 3, "max_abs_vs_libm": [0.0] * 3, "max_rel_vs_libm": [0.0] * 3,
          "sum_abs_vs_libm": [0.0] * 3, "sum_rel_vs_libm": [0.0] * 3}
    xd = x.astype(np.float64)
    for j, f in enumerate(("sin", "cos", "tan")):
        g, w = out[f], ref[f]
        gd = g.astype(np.float64)
        st["max_ulp"][j] = int(np.max(np.abs(g.view(np.int32).astype(np.int64) - w.view(np.int32).astype(np.int64))))
        st["n_inf"][j] = int(np.isinf(gd).sum())
        st["n_nan"][j] = int(np.isnan(gd).sum())
        st["checksum"][j] = int(g.view(np.uint32).astype(np.uint64).sum(dtype=np.uint64))
        lib = getattr(np, f)(xd)
        fin = np.isfinite(gd) & np.isfinite(lib)
        e = np.abs(gd[fin] - lib[fin])
        r = np.where(np.abs(lib[fin]) > 1e-12, e / np.abs(lib[fin]), 0.0)
        st["n_finite_libm"][j] = int(fin.sum())
        st["max_abs_vs_libm"][j] = float(e.max())
        st["max_rel_vs_libm"][j] = float(r.max())
        st["sum_abs_vs_libm"][j] = float(e.sum())
        st["sum_rel_vs_libm"][j] = float(r.sum())
    return st


def shard_stats(rank: int, world: int) -> dict:
    w = CONFIGS["cfg5"]
    lo, hi = shard(N, rank, world)
    x = O.gen_uniform(hi - lo, w.lo, w.hi, w.seed, lo, np.float32)
    r = O.proposed(x, 7, threads=1)
    return host_stats(x, r, r)


def _worker(rank: int, world: int, port: int, q) -> None:
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        red = reduce_stats(shard_stats(rank, world))
        q.put((rank, red))
    finally:
        dist.destroy_process_group()


def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [2])
def test_sharded_stats_equal_unsharded(world):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    whole = shard_stats(0, 1)
    for rank in range(world):
        red = results[rank]
        for k in ("n_checked", "max_ulp", "n_inf", "n_nan", "n_finite_libm", "checksum",
                  "max_abs_vs_libm", "max_rel_vs_libm"):
            assert red[k] == whole[k], (rank, k)
        for k in ("sum_abs_vs_libm", "sum_rel_vs_libm"):
            assert np.allclose(red[k], whole[k], rtol=1e-9), k
    # sanity: the checksum is a wrap-around uint64 sum (order independent)
    assert all(0 <= c < (1 << 64) for c in whole["checksum"])
    assert whole["n_checked"] == N and math.isfinite(whole["max_abs_vs_libm"][0])


def test_shard_ranges_cover_exactly():
    for n in (0, 1, 7, 1 << 33):
        for world in (1, 2, 3, 4, 8):
            spans = [shard(n, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
            assert max(b - a for a, b in spans) - min(b - a for a, b in spans) <= 1


def test_reduce_stats_single_process_is_identity():
    st = shard_stats(0, 1)
    red = reduce_stats(st)
    for k in st:
        assert red[k] == st[k] or np.allclose(red[k], st[k]), k


def test_reduce_stats_clamps_nan_ulp_and_sums_bit_mismatches():
    """max_ulp of a NaN-vs-number pair (K3 reports 2^64-1) stays huge after the
    int64 reduction; n_bit_mismatch is summed like the other counters."""
    st = shard_stats(0, 1)
    st["max_ulp"] = [(1 << 64) - 1, 3, 0]
    st["n_bit_mismatch"] = [5, 0, 1]
    red = reduce_stats(st)
    assert red["max_ulp"] == [(1 << 63) - 1, 3, 0]
    assert red["n_bit_mismatch"] == [5, 0, 1]


def _bench_json(cmd: list[str], timeout: int = 900) -> dict:
    import json
    import subprocess
    import sys

    from conftest import ROOT

    r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, cwd=ROOT,
                       env={**os.environ, "PYTHONPATH": ROOT})
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


@pytest.mark.gpu
def test_bench_two_ranks_real_k3_stats_equal_one_rank():
    """bench.py under torchrun with 2 ranks (gloo, both on the one GPU of the
    lease): every rank runs K1 + K3 on its contiguous shard of one cfg5-recipe
    array and the ranks all-reduce the real K3 statistics; the reduced checksums,
    counts and maxima equal a single rank's pass over the whole array, and the
    full 2^33-element array reproduces round 1's bit-exact checksums."""
    import sys

    from conftest import ROOT

    common = ["--config", "cfg5", "--elements", str(1 << 30), "--configs", "none", "--no-e2e", "--no-cpu",
              "--steps", "3", "--warmup", "3", "--f32-policy", "bitwise", "--sustained-seconds", "0"]
    two = _bench_json([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                       "--master-addr", "127.0.0.1", "--master-port", str(free_port()),
                       os.path.join(ROOT, "bench.py"), "--gpus", "2", "--backend", "gloo", *common])
    one = _bench_json([sys.executable, os.path.join(ROOT, "bench.py"), *common])
    assert two["n_gpus"] == 2 and two["scaling"] == "strong"
    assert two["config"]["elements_per_gpu"] == 1 << 29 and one["config"]["elements_per_gpu"] == 1 << 30
    a2, a1 = two["accuracy"], one["accuracy"]
    for k in ("checked", "checksum", "inf_count", "nan_count", "max_ulp_vs_oracle", "max_abs_err_vs_libm",
              "max_rel_err_vs_libm", "bit_mismatch_vs_oracle"):
        assert a2[k] == a1[k], k
    assert a1["checked"] == 1 << 30 and a1["max_ulp_vs_oracle"] == [0, 0, 0]
    full = _bench_json([sys.executable, os.path.join(ROOT, "bench.py"), "--config", "cfg5", "--configs", "none",
                        "--no-e2e", "--no-cpu", "--steps", "2", "--warmup", "3", "--f32-policy", "bitwise",
                        "--sustained-seconds", "0"])
    assert full["accuracy"]["checked"] == 1 << 33
    # profiles/r01e_cfg5_full.json (round 1, bit-exact kernel)
    assert full["accuracy"]["checksum"] == [18298921530744543647, 18299087910619986952, 18375888137372184031]
