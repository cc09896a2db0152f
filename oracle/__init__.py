"""CPU oracle for elementwise primality (arXiv 2108.04791) -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The
product path (``paper_2108_04791_b200``) never imports it and shares no code
with it; see ``oracle/oracle.c`` for what each function computes and the
passage of PAPER.md it follows.

This module is argument marshalling over ``liboracle.so`` (plain C, built by
``__graft_entry__.build()`` or on first import with gcc).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

BASES = (2, 325, 9375, 28178, 450775, 9780504, 1795265022)  # PAPER.md:54-56 (Eq 4)


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (-O2, pthreads).  Returns its path."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(
            ["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-pthread", _SRC, "-o", tmp]
        )
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        u64, i32, sz = ctypes.c_uint64, ctypes.c_int, ctypes.c_size_t
        p = ctypes.c_void_p
        lib.oracle_mulmod.argtypes = [u64, u64, u64]
        lib.oracle_mulmod.restype = u64
        lib.oracle_powmod.argtypes = [u64, u64, u64]
        lib.oracle_powmod.restype = u64
        lib.oracle_sprp.argtypes = [u64, u64]
        lib.oracle_sprp.restype = i32
        lib.oracle_trial_division.argtypes = [u64]
        lib.oracle_trial_division.restype = i32
        lib.oracle_miller_rabin.argtypes = [u64]
        lib.oracle_miller_rabin.restype = i32
        lib.oracle_isprime_u64.argtypes = [u64]
        lib.oracle_isprime_u64.restype = i32
        lib.oracle_isprime_array.argtypes = [p, p, sz, i32]
        lib.oracle_isprime_array.restype = u64
        lib.oracle_sieve.argtypes = [u64, p]
        lib.oracle_sieve.restype = u64
        lib.oracle_dense_range.argtypes = [u64, sz, p]
        lib.oracle_dense_range.restype = u64
        lib.oracle_sprp_array.argtypes = [p, p, p, sz]
        lib.oracle_sprp_array.restype = None
        lib.oracle_mulmod_array.argtypes = [p, p, p, p, sz]
        lib.oracle_mulmod_array.restype = None
        lib.oracle_powmod_array.argtypes = [p, p, p, p, sz]
        lib.oracle_powmod_array.restype = None
        _lib = lib
    return _lib


def _u64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint64))


def default_threads() -> int:
    return os.cpu_count() or 1


# ---- scalar entry points -------------------------------------------------
def mulmod(a: int, b: int, m: int) -> int:
    return int(_load().oracle_mulmod(a, b, m))


def powmod(a: int, e: int, m: int) -> int:
    return int(_load().oracle_powmod(a, e, m))


def sprp(n: int, a: int) -> bool:
    """Strong probable-prime test of odd n >= 3 to base a."""
    return bool(_load().oracle_sprp(n, a))


def trial_division(n: int) -> bool:
    return bool(_load().oracle_trial_division(n))


def miller_rabin(n: int) -> bool:
    """7-base deterministic Miller-Rabin."""
    return bool(_load().oracle_miller_rabin(n))


def isprime_u64(n: int) -> bool:
    return bool(_load().oracle_isprime_u64(n))


# ---- array entry points ----------------------------------------------------
def isprime(N, threads: int | None = None) -> np.ndarray:
    """out[i] = 1 iff N[i] is prime (uint8 0/1, same length as N)."""
    N = _u64(N).ravel()
    out = np.zeros(N.shape[0], dtype=np.uint8)
    if N.shape[0]:
        _load().oracle_isprime_array(
            N.ctypes.data, out.ctypes.data, N.shape[0], threads or default_threads()
        )
    return out


def sieve(limit: int) -> np.ndarray:
    """Byte mask is_prime[k] for 0 <= k < limit (plain Eratosthenes)."""
    out = np.empty(limit, dtype=np.uint8)
    if limit:
        _load().oracle_sieve(limit, out.ctypes.data)
    return out


def dense_range(lo: int, n: int) -> np.ndarray:
    """isprime(lo + i) for i < n, lo + n <= 2^32, through the plain sieve."""
    out = np.empty(n, dtype=np.uint8)
    if n:
        r = _load().oracle_dense_range(lo, n, out.ctypes.data)
        if r == (1 << 64) - 1:
            raise ValueError("dense_range: lo + n must be <= 2^32 (or out of memory)")
    return out


def sprp_array(n, a) -> np.ndarray:
    n, a = _u64(n), _u64(a)
    out = np.empty(n.shape[0], dtype=np.uint8)
    _load().oracle_sprp_array(n.ctypes.data, a.ctypes.data, out.ctypes.data, n.shape[0])
    return out


def mulmod_array(a, b, m) -> np.ndarray:
    a, b, m = _u64(a), _u64(b), _u64(m)
    out = np.empty(a.shape[0], dtype=np.uint64)
    _load().oracle_mulmod_array(a.ctypes.data, b.ctypes.data, m.ctypes.data,
                                out.ctypes.data, a.shape[0])
    return out


def powmod_array(a, e, m) -> np.ndarray:
    a, e, m = _u64(a), _u64(e), _u64(m)
    out = np.empty(a.shape[0], dtype=np.uint64)
    _load().oracle_powmod_array(a.ctypes.data, e.ctypes.data, m.ctypes.data,
                                out.ctypes.data, a.shape[0])
    return out
