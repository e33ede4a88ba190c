"""B200-native batched piecewise sin/cos/tan (+ Taylor) -- arXiv 2502.10831.

The product is lib/libfasttrig_b200.so (sm_100a kernels behind the C ABI in
include/fasttrig_b200.h).  This package is its Python host mirror; see
``fasttrig`` for the API that follows R:proj/include/fasttrig/kernels.hpp.
"""
from . import _lib
from .fasttrig import (  # noqa: F401
    COS,
    SIN,
    TAN,
    SqrtMode,
    device_const_table,
    device_rows,
    gen_inputs,
    f32_policy,
    get_f32_policy,
    get_host_devices,
    l2_flush,
    launch_count,
    mirror_eval,
    parity_reduce,
    proposed_batch,
    proposed_cos_batch,
    proposed_eval,
    proposed_sin_batch,
    proposed_tan_batch,
    release,
    segment_table,
    set_f32_policy,
    set_host_devices,
    taylor_batch,
    taylor_coeffs,
    taylor_eval,
    thresholds,
)

LIB_PATH = _lib.LIB_PATH
build = _lib.build
