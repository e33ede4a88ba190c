"""ctypes front-end for the CPU checkers (TEST INFRASTRUCTURE ONLY).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's ``cpu_baseline`` /
``--impl reference`` legs import this module, and only as the checker or the
timed CPU baseline.  The product path (paper_2502_10831_b200) never does.

Two libraries:
  * ``port()``  -- oracle/build/liboracle.so, the C restatement ft_oracle.c;
  * ``ref()``   -- oracle/_ref/libfasttrig_ref.so, the unmodified reference
                   headers (R:proj/include/fasttrig/*.hpp) behind ref_shim.cpp.
                   Present only if it was built where /root/reference exists.
Missing libraries are (re)built with ``make -C oracle`` on first use; the
reference shim can only be built where the reference headers exist.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from functools import lru_cache

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "build", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libfasttrig_ref.so")

F32, F64 = 0, 1
SIN, COS, TAN = 1, 2, 4
EXACT, FISR = 0, 1


def _make():
    subprocess.run(["make", "-s", "-C", HERE], check=True, stdout=subprocess.DEVNULL)


@lru_cache(None)
def port() -> C.CDLL:
    if not os.path.exists(PORT_SO) or os.path.getmtime(PORT_SO) < os.path.getmtime(
        os.path.join(HERE, "ft_oracle.c")
    ):
        _make()
    lib = C.CDLL(PORT_SO)
    d, i, u64, vp, sz = C.c_double, C.c_int, C.c_uint64, C.c_void_p, C.c_size_t
    for name in ("ora_proposed_sin", "ora_proposed_cos", "ora_proposed_tan"):
        getattr(lib, name).restype = d
        getattr(lib, name).argtypes = [d, i, i]
    for name in ("ora_taylor_sin", "ora_taylor_cos", "ora_taylor_tan"):
        getattr(lib, name).restype = d
        getattr(lib, name).argtypes = [d, i]
    lib.ora_fast_inverse_sqrt.restype = d
    lib.ora_fast_inverse_sqrt.argtypes = [d, i, i]
    lib.ora_segment_index.restype = i
    lib.ora_segment_index.argtypes = [d]
    for name in ("ora_reduce_sin", "ora_reduce_cos", "ora_reduce_tan"):
        getattr(lib, name).argtypes = [d, C.POINTER(d), C.POINTER(d)]
    lib.ora_segment_table.argtypes = [vp]
    lib.ora_taylor_coeffs.argtypes = [vp, vp, vp]
    lib.ora_proposed_batch.restype = i
    lib.ora_proposed_batch.argtypes = [i, vp, sz, C.c_uint, i, i, vp, vp, vp, vp, vp, i]
    lib.ora_taylor_batch.restype = i
    lib.ora_taylor_batch.argtypes = [i, vp, sz, C.c_uint, i, vp, vp, vp, i]
    lib.ora_splitmix64.restype = u64
    lib.ora_splitmix64.argtypes = [u64, u64]
    lib.ora_gen_uniform.argtypes = [i, d, d, u64, u64, sz, vp]
    return lib


def ref_available() -> bool:
    if os.path.exists(REF_SO):
        return True
    try:
        _make()
    except Exception:
        return False
    return os.path.exists(REF_SO)


@lru_cache(None)
def ref() -> C.CDLL:
    if not ref_available():
        raise RuntimeError("oracle/_ref/libfasttrig_ref.so not built (needs /root/reference)")
    lib = C.CDLL(REF_SO)
    d, i, vp, sz = C.c_double, C.c_int, C.c_void_p, C.c_size_t
    lib.ref_proposed_batch.restype = i
    lib.ref_proposed_batch.argtypes = [i, vp, sz, C.c_uint, i, i, vp, vp, vp, vp, vp, i]
    lib.ref_api_batch.restype = i
    lib.ref_api_batch.argtypes = [i, vp, sz, i, i, vp]
    lib.ref_segment_table.argtypes = [vp]
    lib.ref_segment_index.restype = i
    lib.ref_segment_index.argtypes = [d]
    lib.ref_fast_inverse_sqrt.restype = d
    lib.ref_fast_inverse_sqrt.argtypes = [d, i, i]
    lib.ref_reduce.argtypes = [i, d, C.POINTER(d), C.POINTER(d)]
    lib.ref_scalar.restype = d
    lib.ref_scalar.argtypes = [i, d, i, i]
    lib.ref_check_f32_range.restype = i
    lib.ref_check_f32_range.argtypes = [C.c_uint32, sz, i, i, vp, vp, vp, vp, vp, vp, i]
    return lib


def ref_check_f32_range(start: int, got: dict, method: int = FISR, steps: int = 1,
                        threads: int | None = None) -> dict:
    """The unmodified reference on the float inputs with bit patterns start ..
    start+n-1 (n = len of the given arrays), compared with got['sin'/'cos'/'tan']
    (float32 host arrays) and optionally got['seg_sc'/'seg_t'] (uint8)."""
    arrs = [got.get(k) for k in ("sin", "cos", "tan", "seg_sc", "seg_t")]
    n = next(a.size for a in arrs if a is not None)
    for a in arrs:
        assert a is None or (a.size == n and a.flags.c_contiguous)
    out = np.zeros(11, np.uint64)
    rc = ref().ref_check_f32_range(start & 0xFFFFFFFF, n, method, steps, *[_p(a) for a in arrs],
                                   out.ctypes.data, threads or ncpu())
    assert rc == 0
    o = [int(v) for v in out]
    return {"max_ulp": o[0:3], "n_bit_mismatch": o[3:6], "n_over_2ulp": o[6:9], "seg_mismatch": o[9:11]}


def _p(a):
    return None if a is None else a.ctypes.data


def ncpu() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def proposed(x: np.ndarray, mask: int = 7, method: int = FISR, steps: int = 1, seg: bool = False,
             threads: int | None = None, impl: str = "port"):
    """Evaluate the proposed functions on a host array with the port or the reference.

    Returns dict with keys among 'sin','cos','tan','seg_sc','seg_t'."""
    x = np.ascontiguousarray(x)
    dtype = F32 if x.dtype == np.float32 else F64
    assert x.dtype in (np.float32, np.float64)
    n = x.size
    out = {}
    names = [("sin", SIN), ("cos", COS), ("tan", TAN)]
    arrs = []
    for nm, bit in names:
        a = np.empty(n, x.dtype) if mask & bit else None
        if a is not None:
            out[nm] = a
        arrs.append(a)
    seg_sc = np.empty(n, np.uint8) if seg else None
    seg_t = np.empty(n, np.uint8) if seg else None
    lib = port() if impl == "port" else ref()
    fn = lib.ora_proposed_batch if impl == "port" else lib.ref_proposed_batch
    rc = fn(dtype, _p(x), n, mask, method, steps, _p(arrs[0]), _p(arrs[1]), _p(arrs[2]),
            _p(seg_sc), _p(seg_t), threads or ncpu())
    assert rc == 0
    if seg:
        out["seg_sc"], out["seg_t"] = seg_sc, seg_t
    return out


def taylor(x: np.ndarray, n_terms: int = 5, mask: int = 3, threads: int | None = None):
    x = np.ascontiguousarray(x)
    dtype = F32 if x.dtype == np.float32 else F64
    n = x.size
    out, arrs = {}, []
    for nm, bit in (("sin", SIN), ("cos", COS), ("tan", TAN)):
        a = np.empty(n, x.dtype) if mask & bit else None
        if a is not None:
            out[nm] = a
        arrs.append(a)
    rc = port().ora_taylor_batch(dtype, _p(x), n, mask, n_terms, _p(arrs[0]), _p(arrs[1]),
                                 _p(arrs[2]), threads or ncpu())
    assert rc == 0
    return out


def gen_uniform(n: int, lo: float, hi: float, seed: int, offset: int = 0, dtype=np.float64):
    out = np.empty(n, dtype)
    port().ora_gen_uniform(F32 if dtype == np.float32 else F64, lo, hi, seed, offset, n, out.ctypes.data)
    return out


def segment_table(impl: str = "port") -> np.ndarray:
    out = np.empty(49, np.float64)
    if impl == "port":
        port().ora_segment_table(out.ctypes.data)
    else:
        ref().ref_segment_table(out.ctypes.data)
    return out
