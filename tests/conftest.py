"""pytest configuration: `gpu` marker, repo root on sys.path, shared fixtures."""
from __future__ import annotations

import os
import sys

import numpy as np
import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "golden_v1.npz")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


@pytest.fixture(scope="session")
def golden():
    return dict(np.load(GOLDEN))


@pytest.fixture(scope="session")
def ft():
    """The product package with its CUDA library loaded (fails loudly if missing)."""
    import paper_2502_10831_b200 as pkg
    from paper_2502_10831_b200 import _lib

    if not os.path.exists(_lib.LIB_PATH):
        _lib.build()
    _lib.lib()
    return pkg


def golden_cases(g: dict):
    """Yield (case, mode, x, {'sin','cos','tan','seg_sc','seg_t'}) from the fixture."""
    keys = sorted({k.rsplit("__", 1)[0] for k in g if k.count("__") == 2 and not k.startswith("taylor")})
    for key in keys:
        case, mode = key.split("__")
        yield case, mode, g[key + "__x"], {f: g[key + "__" + f] for f in ("sin", "cos", "tan", "seg_sc", "seg_t")}


MODES = {"fisr1": (1, 1), "exact": (0, 0), "fisr2": (1, 2), "fisr0": (1, 0)}


def same_bits(a: np.ndarray, b: np.ndarray) -> bool:
    """Bitwise equality with all NaNs treated as equal."""
    if a.shape != b.shape:
        return False
    na, nb = np.isnan(a), np.isnan(b)
    if not np.array_equal(na, nb):
        return False
    ua = a.view(np.uint32 if a.dtype == np.float32 else np.uint64)
    ub = b.view(np.uint32 if b.dtype == np.float32 else np.uint64)
    return bool(np.array_equal(ua[~na], ub[~nb]))


def ulp_dist(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """|ordered(a) - ordered(b)| in units of the dtype; NaN==NaN is 0, NaN vs number is huge."""
    it = np.int32 if a.dtype == np.float32 else np.int64
    mask = np.iinfo(it).max

    def ordered(v):
        b_ = v.view(it).astype(np.int64)
        return np.where(b_ < 0, -(b_ & mask), b_)

    d = np.abs(ordered(a) - ordered(b)).astype(np.float64)
    na, nb = np.isnan(a), np.isnan(b)
    d[na & nb] = 0
    d[na ^ nb] = np.inf
    return d
