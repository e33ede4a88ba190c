"""ctypes binding of lib/libfasttrig_b200.so (the C ABI in include/fasttrig_b200.h).

The shared library is built in-tree (``make -C paper_2502_10831_b200`` or
``__graft_entry__.build()``).  There is no fallback: if the library is missing
or cannot be loaded, every entry point raises.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FASTTRIG_B200_LIB") or os.path.join(PKG, "lib", "libfasttrig_b200.so")

FT_OK, FT_ERR_INVALID_ARG, FT_ERR_CUDA, FT_ERR_OOM, FT_ERR_NO_DEVICE = 0, 1, 2, 3, 4
FT_F32, FT_F64 = 0, 1
FT_OUT_SIN, FT_OUT_COS, FT_OUT_TAN = 1, 2, 4
FT_SQRT_EXACT, FT_SQRT_FISR = 0, 1
FT_DIST_UNIFORM, FT_DIST_TAN_STRESS = 0, 1
FT_F32_ULP2, FT_F32_BITWISE = 0, 1

# Every symbol include/fasttrig_b200.h declares (checked by
# tests/test_capi_host.py::test_exports_every_declared_symbol).
EXPORTS = (
    "ft_proposed_sin_batch", "ft_proposed_cos_batch", "ft_proposed_tan_batch",
    "ft_proposed_batch_host", "ft_taylor_batch_host", "ft_proposed_eval", "ft_proposed_eval_seg",
    "ft_taylor_eval", "ft_mirror_eval", "ft_parity_reduce", "ft_stats_reset", "ft_gen_inputs",
    "ft_l2_flush", "ft_host_alloc", "ft_host_free", "ft_segment_table", "ft_taylor_coeffs",
    "ft_thresholds", "ft_launch_count", "ft_last_error_string", "ft_abi_version",
    "ft_set_host_devices", "ft_get_host_devices", "ft_set_f32_policy", "ft_get_f32_policy",
    "ft_device_const_table", "ft_device_rows", "ft_release",
)


class SqrtModeC(C.Structure):
    """ft_sqrt_mode == fasttrig::SqrtMode (R:proj/include/fasttrig/fisr.hpp:14-24)."""
    _fields_ = [("method", C.c_int32), ("newton_steps", C.c_int32)]


class StatsC(C.Structure):
    """ft_stats (include/fasttrig_b200.h)."""
    _fields_ = [
        ("n_checked", C.c_uint64),
        ("max_ulp", C.c_uint64 * 3),
        ("n_over_tol", C.c_uint64 * 3),
        ("seg_mismatch", C.c_uint64 * 2),
        ("n_inf", C.c_uint64 * 3),
        ("n_nan", C.c_uint64 * 3),
        ("n_finite_libm", C.c_uint64 * 3),
        ("checksum", C.c_uint64 * 3),
        ("max_abs_vs_oracle", C.c_double * 3),
        ("max_abs_vs_libm", C.c_double * 3),
        ("max_rel_vs_libm", C.c_double * 3),
        ("sum_abs_vs_libm", C.c_double * 3),
        ("sum_rel_vs_libm", C.c_double * 3),
        ("n_bit_mismatch", C.c_uint64 * 3),
    ]


class FasttrigError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"fasttrig_b200 error {code}: {msg}")
        self.code = code


_lock = threading.Lock()
_lib = None


def build() -> None:
    """Compile the CUDA library in-tree (sm_100a)."""
    subprocess.run(["make", "-s", "-C", PKG, "-j4"], check=True)


def lib() -> C.CDLL:
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise FasttrigError(
                FT_ERR_INVALID_ARG,
                f"{LIB_PATH} is missing: build it with `make -C {PKG}` (no CPU fallback exists)",
            )
        L = C.CDLL(LIB_PATH)
        vp, sz, u, i32, u64, d = C.c_void_p, C.c_size_t, C.c_uint, C.c_int, C.c_uint64, C.c_double
        sm = SqrtModeC
        sig = {
            "ft_proposed_sin_batch": [vp, sz, sm, vp],
            "ft_proposed_cos_batch": [vp, sz, sm, vp],
            "ft_proposed_tan_batch": [vp, sz, sm, vp],
            "ft_proposed_batch_host": [i32, vp, sz, u, sm, vp, vp, vp],
            "ft_taylor_batch_host": [i32, vp, sz, u, i32, vp, vp, vp],
            "ft_proposed_eval": [i32, vp, sz, u, sm, vp, vp, vp, vp],
            "ft_proposed_eval_seg": [i32, vp, sz, u, sm, vp, vp, vp, vp, vp, vp],
            "ft_taylor_eval": [i32, vp, sz, u, i32, vp, vp, vp, vp],
            "ft_mirror_eval": [i32, vp, sz, u, i32, sm, i32, vp, vp, vp, vp, vp, vp],
            "ft_parity_reduce": [i32, vp, sz, u, i32, sm, i32, vp, vp, vp, vp, vp, vp, vp, vp,
                                 u64, vp, vp],
            "ft_stats_reset": [vp, vp],
            "ft_gen_inputs": [i32, i32, d, d, u64, u64, sz, vp, vp],
            "ft_l2_flush": [vp],
            "ft_host_alloc": [C.POINTER(C.c_void_p), sz],
            "ft_host_free": [vp],
            "ft_segment_table": [vp],
            "ft_taylor_coeffs": [vp, vp, vp],
            "ft_thresholds": [vp],
            "ft_set_host_devices": [i32],
            "ft_set_f32_policy": [i32],
            "ft_device_const_table": [i32, vp],
            "ft_device_rows": [i32, vp],
            "ft_release": [i32],
        }
        for name, args in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = C.c_int
        L.ft_launch_count.restype = C.c_uint64
        L.ft_launch_count.argtypes = []
        L.ft_last_error_string.restype = C.c_char_p
        L.ft_last_error_string.argtypes = []
        L.ft_abi_version.restype = C.c_int
        L.ft_abi_version.argtypes = []
        L.ft_get_host_devices.restype = C.c_int
        L.ft_get_host_devices.argtypes = []
        L.ft_get_f32_policy.restype = C.c_int
        L.ft_get_f32_policy.argtypes = []
        _lib = L
        return L


def check(rc: int) -> None:
    if rc != FT_OK:
        raise FasttrigError(rc, lib().ft_last_error_string().decode())
