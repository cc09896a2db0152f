"""Python binding of libisprime.so (arXiv 2108.04791 "isprime_fast" hot path on
B200).  Argument marshalling only: every step of the path runs in the CUDA
kernels behind the C-ABI of ``include/isprime.h``.  There is no CPU fallback:
if the library cannot be loaded, or there is no CUDA device, calls raise.

Names follow the C-ABI:
    isprime(N) -> uint8 mask                 host arrays (numpy), synchronous
    isprime_device(dN, dout, n, stream)      device pointers / tensors
    isprime_count_device(dN, dout, n, dcount, stream)
    isprime_popcount_device(dout, n, dcount, stream)
    isprime_sprp_device / isprime_mulmod_device   diagnostics over the same code
    set_option / get_option / get_stats / reset_stats / shutdown
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

from . import _build

_HERE = os.path.dirname(os.path.abspath(__file__))
# ISPRIME_LIB: load another build of the same library (A/B timing of kernel variants)
LIB_PATH = os.environ.get("ISPRIME_LIB") or os.path.join(_HERE, "libisprime.so")

ISP_OK, ISP_EINVAL, ISP_ENOMEM, ISP_ECUDA, ISP_ENODEV = 0, -1, -2, -3, -4

EXPORTED_SYMBOLS = (
    "isprime", "isprime_device", "isprime_count_device", "isprime_popcount_device",
    "isprime_strerror", "isprime_shutdown", "isprime_set_option", "isprime_get_option",
    "isprime_get_stats", "isprime_reset_stats", "isprime_sprp_device", "isprime_mulmod_device",
    "isprime_get_kernel_times", "isprime_reset_kernel_times",
)


class IsPrimeError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"isprime status {status}: {msg}")
        self.status = status


class Stats(ctypes.Structure):
    _fields_ = [(name, ctypes.c_uint64) for name in (
        "window_lo", "window_hi", "sieve_runs", "sieved_integers", "queued32", "queued64",
        "passed32", "passed64", "chunks", "kernel_launches")] + [
        ("mulmods", ctypes.c_uint64 * 4), ("mulmods_fp64", ctypes.c_uint64 * 2),
        ("mulmods_fused", ctypes.c_uint64 * 2)]

    def as_dict(self) -> dict:
        d = {name: int(getattr(self, name)) for name, _ in self._fields_ if not name.startswith("mulmods")}
        d["mulmods"] = [int(x) for x in self.mulmods]
        d["mulmods_fp64"] = [int(x) for x in self.mulmods_fp64]
        d["mulmods_fused"] = [int(x) for x in self.mulmods_fused]
        return d


class KernelTime(ctypes.Structure):
    _fields_ = [("name", ctypes.c_char * 16), ("launches", ctypes.c_uint64), ("ms_total", ctypes.c_double)]


_lib = None


def load(build_if_missing: bool = True) -> ctypes.CDLL:
    """Load libisprime.so (building it with nvcc first if it is absent)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        if not build_if_missing:
            raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build()")
        _build.build()
    lib = ctypes.CDLL(LIB_PATH)
    vp, sz, i32, ll = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_longlong
    lib.isprime.argtypes = [vp, vp, sz]
    lib.isprime_device.argtypes = [vp, vp, sz, vp]
    lib.isprime_count_device.argtypes = [vp, vp, sz, vp, vp]
    lib.isprime_popcount_device.argtypes = [vp, sz, vp, vp]
    lib.isprime_sprp_device.argtypes = [vp, vp, vp, sz, vp]
    lib.isprime_mulmod_device.argtypes = [vp, vp, vp, vp, sz, vp]
    for f in ("isprime", "isprime_device", "isprime_count_device", "isprime_popcount_device",
              "isprime_sprp_device", "isprime_mulmod_device"):
        getattr(lib, f).restype = i32
    lib.isprime_strerror.argtypes = [i32]
    lib.isprime_strerror.restype = ctypes.c_char_p
    lib.isprime_shutdown.argtypes = []
    lib.isprime_shutdown.restype = None
    lib.isprime_set_option.argtypes = [ctypes.c_char_p, ll]
    lib.isprime_set_option.restype = i32
    lib.isprime_get_option.argtypes = [ctypes.c_char_p]
    lib.isprime_get_option.restype = ll
    lib.isprime_get_stats.argtypes = [ctypes.POINTER(Stats)]
    lib.isprime_get_stats.restype = i32
    lib.isprime_reset_stats.argtypes = []
    lib.isprime_reset_stats.restype = i32
    lib.isprime_get_kernel_times.argtypes = [ctypes.POINTER(KernelTime), i32, ctypes.POINTER(i32)]
    lib.isprime_get_kernel_times.restype = i32
    lib.isprime_reset_kernel_times.argtypes = []
    lib.isprime_reset_kernel_times.restype = i32
    _lib = lib
    return lib


def _check(status: int) -> None:
    if status != ISP_OK:
        raise IsPrimeError(status, load().isprime_strerror(status).decode())


def _ptr(x) -> int | None:
    """Device/host address of a torch tensor, numpy array or integer."""
    if x is None:
        return None
    if isinstance(x, int):
        return x
    if hasattr(x, "data_ptr"):
        return x.data_ptr()
    if isinstance(x, np.ndarray):
        return x.ctypes.data
    raise TypeError(f"cannot take the address of {type(x)!r}")


def _stream(stream) -> int | None:
    if stream is None:
        try:
            import torch
            if torch.cuda.is_available():
                return torch.cuda.current_stream().cuda_stream
        except ImportError:
            pass
        return None
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream  # torch.cuda.Stream


# ---------------------------------------------------------------- C-ABI calls
def isprime(N) -> np.ndarray:
    """Host front door: uint8 0/1 mask, same length as N (flattened)."""
    N = np.ascontiguousarray(np.asarray(N, dtype=np.uint64)).ravel()
    out = np.empty(N.shape[0], dtype=np.uint8)
    _check(load().isprime(N.ctypes.data if N.size else None, out.ctypes.data if N.size else None, N.shape[0]))
    return out


def isprime_into(N, out) -> None:
    """Host front door writing into a caller buffer (numpy arrays or pinned
    torch CPU tensors; element counts must match)."""
    n = N.numel() if hasattr(N, "numel") else N.shape[0]
    _check(load().isprime(_ptr(N), _ptr(out), n))


def isprime_device(dN, dout, n: int | None = None, stream=None) -> None:
    """Device front door on tensors / device pointers (stream-ordered)."""
    if n is None:
        n = dN.numel()
    _check(load().isprime_device(_ptr(dN), _ptr(dout), n, _stream(stream)))


def isprime_count_device(dN, dout, dcount, n: int | None = None, stream=None) -> None:
    if n is None:
        n = dN.numel()
    _check(load().isprime_count_device(_ptr(dN), _ptr(dout), n, _ptr(dcount), _stream(stream)))


def isprime_popcount_device(dout, dcount, n: int | None = None, stream=None) -> None:
    if n is None:
        n = dout.numel()
    _check(load().isprime_popcount_device(_ptr(dout), n, _ptr(dcount), _stream(stream)))


def isprime_sprp_device(dn, da, dout, count: int | None = None, stream=None) -> None:
    if count is None:
        count = dn.numel()
    _check(load().isprime_sprp_device(_ptr(dn), _ptr(da), _ptr(dout), count, _stream(stream)))


def isprime_mulmod_device(da, db, dm, dout, count: int | None = None, stream=None) -> None:
    if count is None:
        count = da.numel()
    _check(load().isprime_mulmod_device(_ptr(da), _ptr(db), _ptr(dm), _ptr(dout), count, _stream(stream)))


def set_option(key: str, value: int) -> None:
    _check(load().isprime_set_option(key.encode(), int(value)))


def get_option(key: str) -> int:
    return int(load().isprime_get_option(key.encode()))


def get_stats() -> dict:
    st = Stats()
    _check(load().isprime_get_stats(ctypes.byref(st)))
    return st.as_dict()


def reset_stats() -> None:
    _check(load().isprime_reset_stats())


def get_kernel_times() -> dict:
    """{kernel name: (launches, total ms)} accumulated with option kernel_timing=1."""
    arr = (KernelTime * 16)()
    cnt = ctypes.c_int(0)
    _check(load().isprime_get_kernel_times(arr, 16, ctypes.byref(cnt)))
    return {arr[k].name.decode(): (int(arr[k].launches), float(arr[k].ms_total)) for k in range(min(cnt.value, 16))}


def reset_kernel_times() -> None:
    _check(load().isprime_reset_kernel_times())


def shutdown() -> None:
    load().isprime_shutdown()


# ---------------------------------------------------------------- torch helpers
def isprime_tensor(dN, stream=None):
    """uint8 mask tensor for a uint64 (or int64) CUDA tensor dN."""
    import torch
    if not dN.is_cuda:
        raise ValueError("isprime_tensor needs a CUDA tensor (use isprime() for host arrays)")
    dN = dN.contiguous()
    dout = torch.empty(dN.numel(), dtype=torch.uint8, device=dN.device)
    isprime_device(dN, dout, dN.numel(), stream)
    return dout.view(dN.shape)
