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


def _check_mask(mask: int) -> None:
    if not isinstance(mask, (int, np.integer)) or not 1 <= int(mask) <= 7:
        raise ValueError(f"mask must select 1..3 of sin/cos/tan (1..7), got {mask!r}")


def _host_outs(x: np.ndarray, mask: int, out) -> dict:
    """Caller-supplied host outputs must match x exactly: the C ABI writes
    x.size * itemsize bytes through each pointer."""
    _check_mask(mask)
    if out is None:
        return {nm: np.empty_like(x) for j, nm in enumerate(NAMES) if mask & (1 << j)}
    for j, nm in enumerate(NAMES):
        if not mask & (1 << j):
            continue
        o = out.get(nm)
        if not isinstance(o, np.ndarray):
            raise TypeError(f"out[{nm!r}] must be a numpy array")
        if o.dtype != x.dtype:
            raise TypeError(f"out[{nm!r}] has dtype {o.dtype}, x has {x.dtype}")
        if o.size != x.size:
            raise ValueError(f"out[{nm!r}] has {o.size} elements, x has {x.size}")
        if not o.flags.c_contiguous or not o.flags.writeable:
            raise ValueError(f"out[{nm!r}] must be C-contiguous and writeable")
    return out


def proposed_batch(xs: np.ndarray, mask: int = 7, mode: SqrtMode = SqrtMode(), out=None) -> dict:
    """Fused host-pointer form (f32 or f64): one read of x, the masked outputs."""
    x = np.ascontiguousarray(xs)
    dt = _dtype_code(x.dtype)
    outs = _host_outs(x, mask, out)
    ptr = [outs[nm].ctypes.data if nm in outs else None for nm in NAMES]
    L.check(L.lib().ft_proposed_batch_host(dt, x.ctypes.data, x.size, mask, mode.c(), *ptr))
    return outs


def taylor_batch(xs: np.ndarray, n_terms: int = 5, mask: int = 3, out=None) -> dict:
    x = np.ascontiguousarray(xs)
    dt = _dtype_code(x.dtype)
    outs = _host_outs(x, mask, out)
    ptr = [outs[nm].ctypes.data if nm in outs else None for nm in NAMES]
    L.check(L.lib().ft_taylor_batch_host(dt, x.ctypes.data, x.size, mask, n_terms, *ptr))
    return outs


# --------------------------------------------------------------------------
# Device API (torch CUDA tensors, asynchronous on the current torch stream)
# --------------------------------------------------------------------------
def _stream(stream, device=None):
    import torch

    s = stream if stream is not None else torch.cuda.current_stream(device)
    return C.c_void_p(s.cuda_stream)


def _check_x(x) -> None:
    if not (getattr(x, "is_cuda", False) and x.is_contiguous()):
        raise ValueError("x must be a contiguous CUDA tensor")


def _outs(x, mask, out):
    """Caller-supplied device outputs must match x (dtype, element count, device)
    and be contiguous: the C ABI writes x.numel() * itemsize bytes through each."""
    import torch

    _check_mask(mask)
    if out is None:
        return {nm: torch.empty_like(x) for j, nm in enumerate(NAMES) if mask & (1 << j)}
    for j, nm in enumerate(NAMES):
        if not mask & (1 << j):
            continue
        o = out.get(nm)
        if not isinstance(o, torch.Tensor):
            raise TypeError(f"out[{nm!r}] must be a torch tensor")
        if o.dtype != x.dtype:
            raise TypeError(f"out[{nm!r}] has dtype {o.dtype}, x has {x.dtype}")
        if o.numel() != x.numel():
            raise ValueError(f"out[{nm!r}] has {o.numel()} elements, x has {x.numel()}")
        if o.device != x.device:
            raise ValueError(f"out[{nm!r}] is on {o.device}, x on {x.device}")
        if not o.is_contiguous():
            raise ValueError(f"out[{nm!r}] must be contiguous")
    return out


def _ptrs(outs):
    return [outs[nm].data_ptr() if nm in outs else None for nm in NAMES]


def proposed_eval(x, mask: int = 7, mode: SqrtMode = SqrtMode(), out: dict | None = None,
                  seg: bool = False, stream=None) -> dict:
    """K1 on a CUDA tensor: returns {'sin','cos','tan'} (per mask) [+ 'seg_sc','seg_t']."""
    import torch

    _check_x(x)
    outs = _outs(x, mask, out)
    with torch.cuda.device(x.device):  # the C ABI launches on the current device
        s = _stream(stream, x.device)
        if seg:
            outs["seg_sc"] = torch.empty(x.numel(), dtype=torch.uint8, device=x.device)
            outs["seg_t"] = torch.empty(x.numel(), dtype=torch.uint8, device=x.device)
            L.check(L.lib().ft_proposed_eval_seg(
                _dtype_code(x.dtype), x.data_ptr(), x.numel(), mask, mode.c(), *_ptrs(outs),
                outs["seg_sc"].data_ptr(), outs["seg_t"].data_ptr(), s))
        else:
            L.check(L.lib().ft_proposed_eval(_dtype_code(x.dtype), x.data_ptr(), x.numel(), mask,
                                             mode.c(), *_ptrs(outs), s))
    return outs


def taylor_eval(x, n_terms: int = 5, mask: int = 3, out: dict | None = None, stream=None) -> dict:
    """K2 on a CUDA tensor."""
    import torch

    _check_x(x)
    outs = _outs(x, mask, out)
    with torch.cuda.device(x.device):
        L.check(L.lib().ft_taylor_eval(_dtype_code(x.dtype), x.data_ptr(), x.numel(), mask, n_terms,
                                       *_ptrs(outs), _stream(stream, x.device)))
    return outs


def mirror_eval(x, mask: int = 7, kind: int = 0, mode: SqrtMode = SqrtMode(), n_terms: int = 5,
                seg: bool = False, stream=None) -> dict:
    """Device restatement of the reference (the device-side oracle of K3)."""
    import torch

    _check_x(x)
    outs = _outs(x, mask, None)
    sp = [None, None]
    if seg:
        outs["seg_sc"] = torch.empty(x.numel(), dtype=torch.uint8, device=x.device)
        outs["seg_t"] = torch.empty(x.numel(), dtype=torch.uint8, device=x.device)
        sp = [outs["seg_sc"].data_ptr(), outs["seg_t"].data_ptr()]
    with torch.cuda.device(x.device):
        L.check(L.lib().ft_mirror_eval(_dtype_code(x.dtype), x.data_ptr(), x.numel(), mask, kind,
                                       mode.c(), n_terms, *_ptrs(outs), *sp, _stream(stream, x.device)))
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

    _check_x(x)
    _outs(x, mask, {nm: outs[nm] for nm in NAMES if nm in outs})  # same checks as the outputs
    refs = refs or {}
    for nm, r in refs.items():
        if r.dtype != x.dtype or r.numel() != x.numel() or r.device != x.device or not r.is_contiguous():
            raise ValueError(f"refs[{nm!r}] must match x (dtype, size, device) and be contiguous")
    if check_seg:
        for nm in ("seg_sc", "seg_t"):
            sg = outs[nm]
            if sg.dtype != torch.uint8 or sg.numel() != x.numel() or sg.device != x.device or not sg.is_contiguous():
                raise ValueError(f"outs[{nm!r}] must be a contiguous uint8 tensor with one byte per element")
    buf = stats_buf if stats_buf is not None else torch.zeros(
        C.sizeof(L.StatsC), dtype=torch.uint8, device=x.device)
    if buf.numel() * buf.element_size() < C.sizeof(L.StatsC) or buf.device != x.device:
        raise ValueError(f"stats_buf must hold {C.sizeof(L.StatsC)} bytes on {x.device}")
    with torch.cuda.device(x.device):
        s = _stream(stream, x.device)
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
    _check_x(x)
    if x.numel() < n:
        raise ValueError(f"out holds {x.numel()} elements, {n} requested")
    with torch.cuda.device(x.device):
        L.check(L.lib().ft_gen_inputs(_dtype_code(x.dtype), dist, lo, hi, seed, offset, n,
                                      x.data_ptr(), _stream(stream, x.device)))
    return x


def l2_flush(stream=None) -> None:
    L.check(L.lib().ft_l2_flush(_stream(stream)))


def segment_table() -> np.ndarray:
    out = np.empty(49, np.float64)
    L.check(L.lib().ft_segment_table(out.ctypes.data))
    return out


def device_const_table(unit: int = 0) -> np.ndarray:
    """The 49 table doubles read back from a translation unit's __constant__ bank
    (0 K1/K2, 1 K3, 2 K4/K5, 3 C-ABI)."""
    out = np.empty(49, np.float64)
    L.check(L.lib().ft_device_const_table(unit, out.ctypes.data))
    return out


ROW_DTYPE = np.dtype([("a", "<f8"), ("b", "<f8"), ("c", "<f8"), ("d", "<f8"), ("X", "<f8"),
                      ("Y", "<f8"), ("Z", "<f8"), ("klo_hi", "<i4"), ("khi_hi", "<i4"),
                      ("klo", "<f8"), ("khi", "<f8")])


RELAX_ROW_DTYPE = np.dtype([("a", "<f8"), ("b", "<f8"), ("c", "<f8"), ("d", "<f8"),
                            ("klo_hi", "<i4"), ("khi_hi", "<i4"), ("pad", "<i4", (2,))])


def device_rows(kind: int = 0) -> np.ndarray:
    """The 8 shared-memory rows a K1 block stages (kind 0: bit-exact 80-byte rows;
    1..7: the relaxed f32 48-byte rows for that mask), copied out by a kernel."""
    buf = np.zeros(640, np.uint8)
    L.check(L.lib().ft_device_rows(kind, buf.ctypes.data))
    dt = ROW_DTYPE if kind == 0 else RELAX_ROW_DTYPE
    return buf[: 8 * dt.itemsize].view(dt).copy()


def release(device: int = -1) -> None:
    """Free the host-pointer pipeline / staging / L2-flush buffers (-1: all devices)."""
    L.check(L.lib().ft_release(device))


def taylor_coeffs() -> tuple[np.ndarray, np.ndarray, np.ndarray]:
    s, c, t = (np.empty(9, np.float64) for _ in range(3))
    L.check(L.lib().ft_taylor_coeffs(s.ctypes.data, c.ctypes.data, t.ctypes.data))
    return s, c, t


def thresholds() -> np.ndarray:
    """[quad1, quad2, quad3, guard] by host bisection, then the compiled-in copies."""
    out = np.empty(8, np.float64)
    L.check(L.lib().ft_thresholds(out.ctypes.data))
    return out


F32_POLICIES = {"ulp2": L.FT_F32_ULP2, "bitwise": L.FT_F32_BITWISE}


def set_f32_policy(policy: str) -> None:
    """'ulp2' (default): f32 outputs within 2 ulp of (float)proposed((double)x) with
    the identical segment choice; 'bitwise': bit-identical to it."""
    L.check(L.lib().ft_set_f32_policy(F32_POLICIES[policy]))


def get_f32_policy() -> str:
    code = int(L.lib().ft_get_f32_policy())
    return next(k for k, v in F32_POLICIES.items() if v == code)


class f32_policy:
    """Context manager: ``with f32_policy('bitwise'): ...`` (restores the previous one)."""

    def __init__(self, policy: str):
        self.policy = policy

    def __enter__(self):
        self.prev = get_f32_policy()
        set_f32_policy(self.policy)
        return self

    def __exit__(self, *exc):
        set_f32_policy(self.prev)
        return False


def set_host_devices(n: int) -> None:
    """How many GPUs one host-pointer call spreads over (n <= 0: all visible)."""
    L.check(L.lib().ft_set_host_devices(n))


def get_host_devices() -> int:
    return int(L.lib().ft_get_host_devices())


def launch_count() -> int:
    return int(L.lib().ft_launch_count())
