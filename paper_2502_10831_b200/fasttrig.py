"""Host-side mirror of the reference ``fasttrig`` API over the B200 C ABI.

The reference (R:proj/include/fasttrig/) is a header-only C++ library; its hot
path is the batch API

    std::vector<double> proposed_{sin,cos,tan}_batch(std::span<const double>, SqrtMode = {})
                                                              -- kernels.hpp:84-94

This module keeps those names, argument meanings and error behaviour for
Python callers (tests, bench, harness) -- the C++ drop-in is
include/fasttrig/gpu.hpp.  Host arrays go through the host-pointer entry points
(``ft_proposed_*_batch``); torch CUDA tensors go through the asynchronous
device-pointer entry points on the current torch stream.  Every call runs the
sm_100a kernels in lib/libfasttrig_b200.so; there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib as L

SIN, COS, TAN = L.FT_OUT_SIN, L.FT_OUT_COS, L.FT_OUT_TAN
NAMES = ("sin", "cos", "tan")


@dataclass(frozen=True)
class SqrtMode:
    """fasttrig::SqrtMode (fisr.hpp:14-24): method 0 exact / 1 fisr, newton_steps."""

    method: int = L.FT_SQRT_FISR
    newton_steps: int = 1

    @staticmethod
    def exact() -> "SqrtMode":  # fisr.hpp:20
        return SqrtMode(L.FT_SQRT_EXACT, 0)

    @staticmethod
    def fisr(steps: int = 1) -> "SqrtMode":  # fisr.hpp:21-23 (steps < 1 -> 1)
        return SqrtMode(L.FT_SQRT_FISR, 1 if steps < 1 else steps)

    def c(self) -> L.SqrtModeC:
        return L.SqrtModeC(self.method, self.newton_steps)


def _dtype_code(dt) -> int:
    if dt in (np.float32, "float32"):
        return L.FT_F32
    if dt in (np.float64, "float64"):
        return L.FT_F64
    s = str(dt)
    if s.endswith("float32"):
        return L.FT_F32
    if s.endswith("float64"):
        return L.FT_F64
    raise TypeError(f"fasttrig_b200 supports float32 / float64 inputs, got {dt}")


# --------------------------------------------------------------------------
# Host-pointer API (reference semantics: host in, host out, blocking)
# --------------------------------------------------------------------------
def _host_batch(fn_name: str, xs, mode: SqrtMode) -> np.ndarray:
    x = np.ascontiguousarray(xs, dtype=np.float64)
    out = np.empty_like(x)
    L.check(getattr(L.lib(), fn_name)(x.ctypes.data, x.size, mode.c(), out.ctypes.data))
    return out


def proposed_sin_batch(xs, mode: SqrtMode = SqrtMode()) -> np.ndarray:
    """kernels.hpp:84-86 -- out[i] = proposed_sin(xs[i], mode), bitwise."""
    return _host_batch("ft_proposed_sin_batch", xs, mode)


def proposed_cos_batch(xs, mode: SqrtMode = SqrtMode()) -> np.ndarray:
    """kernels.hpp:88-90."""
    return _host_batch("ft_proposed_cos_batch", xs, mode)


def proposed_tan_batch(xs, mode: SqrtMode = SqrtMode()) -> np.ndarray:
    """kernels.hpp:92-94."""
    return _host_batch("ft_proposed_tan_batch", xs, mode)


def proposed_batch(xs: np.ndarray, mask: int = 7, mode: SqrtMode = SqrtMode(), out=None) -> dict:
    """Fused host-pointer form (f32 or f64): one read of x, the masked outputs."""
    x = np.ascontiguousarray(xs)
    dt = _dtype_code(x.dtype)
    outs = out or {nm: np.empty_like(x) for j, nm in enumerate(NAMES) if mask & (1 << j)}
    ptr = [outs[nm].ctypes.data if nm in outs else None for nm in NAMES]
    L.check(L.lib().ft_proposed_batch_host(dt, x.ctypes.data, x.size, mask, mode.c(), *ptr))
    return outs


def taylor_batch(xs: np.ndarray, n_terms: int = 5, mask: int = 3, out=None) -> dict:
    x = np.ascontiguousarray(xs)
    dt = _dtype_code(x.dtype)
    outs = out or {nm: np.empty_like(x) for j, nm in enumerate(NAMES) if mask & (1 << j)}
    ptr = [outs[nm].ctypes.data if nm in outs else None for nm in NAMES]
    L.check(L.lib().ft_taylor_batch_host(dt, x.ctypes.data, x.size, mask, n_terms, *ptr))
    return outs


# --------------------------------------------------------------------------
# Device API (torch CUDA tensors, asynchronous on the current torch stream)
# --------------------------------------------------------------------------
def _stream(stream):
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def _outs(x, mask, out):
    import torch

    if out is not None:
        return out
    return {nm: torch.empty_like(x) for j, nm in enumerate(NAMES) if mask & (1 << j)}


def _ptrs(outs):
    return [outs[nm].data_ptr() if nm in outs else None for nm in NAMES]


def proposed_eval(x, mask: int = 7, mode: SqrtMode = SqrtMode(), out: dict | None = None,
                  seg: bool = False, stream=None) -> dict:
    """K1 on a CUDA tensor: returns {'sin','cos','tan'} (per mask) [+ 'seg_sc','seg_t']."""
    import torch

    assert x.is_cuda and x.is_contiguous()
    outs = _outs(x, mask, out)
    if seg:
        outs["seg_sc"] = torch.empty(x.numel(), dtype=torch.uint8, device=x.device)
        outs["seg_t"] = torch.empty(x.numel(), dtype=torch.uint8, device=x.device)
        L.check(L.lib().ft_proposed_eval_seg(
            _dtype_code(x.dtype), x.data_ptr(), x.numel(), mask, mode.c(), *_ptrs(outs),
            outs["seg_sc"].data_ptr(), outs["seg_t"].data_ptr(), _stream(stream)))
    else:
        L.check(L.lib().ft_proposed_eval(_dtype_code(x.dtype), x.data_ptr(), x.numel(), mask,
                                         mode.c(), *_ptrs(outs), _stream(stream)))
    return outs


def taylor_eval(x, n_terms: int = 5, mask: int = 3, out: dict | None = None, stream=None) -> dict:
    """K2 on a CUDA tensor."""
    assert x.is_cuda and x.is_contiguous()
    outs = _outs(x, mask, out)
    L.check(L.lib().ft_taylor_eval(_dtype_code(x.dtype), x.data_ptr(), x.numel(), mask, n_terms,
                                   *_ptrs(outs), _stream(stream)))
    return outs


def mirror_eval(x, mask: int = 7, kind: int = 0, mode: SqrtMode = SqrtMode(), n_terms: int = 5,
                seg: bool = False, stream=None) -> dict:
    """Device restatement of the reference (the device-side oracle of K3)."""
    import torch

    assert x.is_cuda and x.is_contiguous()
    outs = _outs(x, mask, None)
    sp = [None, None]
    if seg:
        outs["seg_sc"] = torch.empty(x.numel(), dtype=torch.uint8, device=x.device)
        outs["seg_t"] = torch.empty(x.numel(), dtype=torch.uint8, device=x.device)
        sp = [outs["seg_sc"].data_ptr(), outs["seg_t"].data_ptr()]
    L.check(L.lib().ft_mirror_eval(_dtype_code(x.dtype), x.data_ptr(), x.numel(), mask, kind,
                                   mode.c(), n_terms, *_ptrs(outs), *sp, _stream(stream)))
    return outs


def stats_to_dict(st: L.StatsC) -> dict:
    d = {}
    for name, _ in L.StatsC._fields_:
        v = getattr(st, name)
        d[name] = list(v) if hasattr(v, "__len__") else v
    return d


def parity_reduce(x, outs: dict, mask: int, kind: int = 0, mode: SqrtMode = SqrtMode(),
                  n_terms: int = 5, refs: dict | None = None, ulp_tol: int = 2,
                  check_seg: bool = False, stats_buf=None, reset: bool = True, stream=None) -> dict:
    """K3: parity + error statistics of `outs` against `refs` (device arrays) or the
    device restatement.  Returns the ft_stats fields as a dict (synchronises)."""
    import torch

    refs = refs or {}
    buf = stats_buf if stats_buf is not None else torch.zeros(
        C.sizeof(L.StatsC), dtype=torch.uint8, device=x.device)
    s = _stream(stream)
    if reset:
        L.check(L.lib().ft_stats_reset(buf.data_ptr(), s))
    rp = [refs[nm].data_ptr() if nm in refs else None for nm in NAMES]
    sp = [outs["seg_sc"].data_ptr() if check_seg else None,
          outs["seg_t"].data_ptr() if check_seg else None]
    L.check(L.lib().ft_parity_reduce(_dtype_code(x.dtype), x.data_ptr(), x.numel(), mask, kind,
                                     mode.c(), n_terms, *_ptrs(outs), *rp, *sp, ulp_tol,
                                     buf.data_ptr(), s))
    host = buf.cpu().numpy().tobytes()
    return stats_to_dict(L.StatsC.from_buffer_copy(host))


def gen_inputs(n: int, dtype, dist: int = L.FT_DIST_UNIFORM, lo: float = 0.0, hi: float = 1.0,
               seed: int = 2024873, offset: int = 0, device=None, out=None, stream=None):
    """K4: seeded inputs in place on the device (element i = global element offset+i)."""
    import torch

    x = out if out is not None else torch.empty(n, dtype=dtype, device=device or "cuda")
    L.check(L.lib().ft_gen_inputs(_dtype_code(x.dtype), dist, lo, hi, seed, offset, n,
                                  x.data_ptr(), _stream(stream)))
    return x


def l2_flush(stream=None) -> None:
    L.check(L.lib().ft_l2_flush(_stream(stream)))


def segment_table() -> np.ndarray:
    out = np.empty(49, np.float64)
    L.check(L.lib().ft_segment_table(out.ctypes.data))
    return out


def taylor_coeffs() -> tuple[np.ndarray, np.ndarray, np.ndarray]:
    s, c, t = (np.empty(9, np.float64) for _ in range(3))
    L.check(L.lib().ft_taylor_coeffs(s.ctypes.data, c.ctypes.data, t.ctypes.data))
    return s, c, t


def thresholds() -> np.ndarray:
    """[quad1, quad2, quad3, guard] by host bisection, then the compiled-in copies."""
    out = np.empty(8, np.float64)
    L.check(L.lib().ft_thresholds(out.ctypes.data))
    return out


def set_host_devices(n: int) -> None:
    """How many GPUs one host-pointer call spreads over (n <= 0: all visible)."""
    L.check(L.lib().ft_set_host_devices(n))


def get_host_devices() -> int:
    return int(L.lib().ft_get_host_devices())


def launch_count() -> int:
    return int(L.lib().ft_launch_count())
