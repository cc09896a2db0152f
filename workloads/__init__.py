"""Seeded synthetic inputs for the five BASELINE.json configurations.

The generator definition is SURVEY.md section 8(d) (counter-based splitmix64,
so any shard can produce its own slice).  This package holds no primality or
modular arithmetic: it serves both the oracle tests and the CUDA path.  The
one number-theoretic input, ``chernick_k.txt`` (the k in [1, 242347] with
6k+1, 12k+1, 18k+1 all prime), was written by ``make_chernick_table.py``,
which calls ``oracle/`` only.

The paper's own workloads are synthetic too (random k-bit primes / odds /
randoms, incrementing sequences, normal distributions: PAPER.md:308, 349,
Tables 3 and 5); no dataset is involved.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "gen.c")
_LIB = os.path.join(_HERE, "libgen.so")
_KFILE = os.path.join(_HERE, "chernick_k.txt")

P64M59 = (1 << 64) - 59  # largest 64-bit prime

# name -> (config index, n, description); BASELINE.json "configs"
CONFIGS = {
    "C1": (1, 100_000, "uniform [0, 2^20): small-integer array path (sieve 2^20 + gather)"),
    "C2": (2, 1 << 24, "uniform [2^20, 2^32): medium scalars (prefilter + 32-bit MR)"),
    "C3": (3, 1 << 26, "uniform [2^49, 2^64) forced odd: large integers (64-bit MR)"),
    "C4": (4, 1 << 32, "dense range 0 .. 2^32-1 (sieve + gather, pi(2^32) = 203280221)"),
    "C5": (5, 1 << 28, "log-uniform bit length 1-64 + Chernick every 1024th + 2^64-59 every 4096th"),
}


def build(force: bool = False) -> str:
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
        u64, sz, i32, p = ctypes.c_uint64, ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p
        lib.gen_mix64.argtypes = [u64]
        lib.gen_mix64.restype = u64
        lib.gen_U.argtypes = [u64, u64]
        lib.gen_U.restype = u64
        lib.gen_RNG.argtypes = [u64, u64, u64]
        lib.gen_RNG.restype = u64
        lib.gen_carmichael_stream.argtypes = [p, sz, p, sz]
        lib.gen_carmichael_stream.restype = u64
        lib.gen_config.argtypes = [i32, u64, sz, p, p, sz, i32]
        lib.gen_config.restype = i32
        lib.gen_uniform.argtypes = [u64, u64, sz, u64, u64, i32, p]
        lib.gen_uniform.restype = None
        lib.gen_loguniform.argtypes = [u64, u64, sz, i32, i32, p]
        lib.gen_loguniform.restype = None
        _lib = lib
    return _lib


_valid_k = None


def chernick_valid_k() -> np.ndarray:
    """k in [1, 242347] with 6k+1, 12k+1, 18k+1 all prime (1675 values)."""
    global _valid_k
    if _valid_k is None:
        ks = []
        with open(_KFILE) as f:
            for line in f:
                line = line.split("#", 1)[0].strip()
                if line:
                    ks.append(int(line))
        _valid_k = np.array(ks, dtype=np.uint32)
    return _valid_k


def chernick_numbers() -> list[int]:
    """Every Chernick number (6k+1)(12k+1)(18k+1) < 2^64 with prime factors."""
    return [(6 * k + 1) * (12 * k + 1) * (18 * k + 1) for k in chernick_valid_k().tolist()]


def carmichael_stream(count: int) -> tuple[np.ndarray, int]:
    """Carm[0..count) of config C5 and the number of draws consumed."""
    ks = chernick_valid_k()
    out = np.empty(count, dtype=np.uint64)
    draws = _load().gen_carmichael_stream(ks.ctypes.data, ks.shape[0], out.ctypes.data, count)
    return out, int(draws)


def generate(cfg: str | int, start: int = 0, count: int | None = None,
             threads: int | None = None, out: np.ndarray | None = None) -> np.ndarray:
    """N[start : start+count] of config ``cfg`` ("C1".."C5" or 1..5) as uint64."""
    if isinstance(cfg, str):
        idx, n, _ = CONFIGS[cfg]
    else:
        idx = int(cfg)
        n = CONFIGS[f"C{idx}"][1]
    if count is None:
        count = n - start
    if out is None:
        out = np.empty(count, dtype=np.uint64)
    assert out.dtype == np.uint64 and out.flags.c_contiguous and out.shape[0] >= count
    ks = chernick_valid_k()
    rc = _load().gen_config(idx, start, count, out.ctypes.data, ks.ctypes.data,
                            ks.shape[0], threads or (os.cpu_count() or 1))
    if rc != 0:
        raise RuntimeError(f"gen_config failed: {rc}")
    return out[:count]


def uniform(seed: int, count: int, lo: int, hi: int, force_odd: bool = False,
            start: int = 0) -> np.ndarray:
    """Seeded uniform draws in [lo, hi) (hi = 2^64 allowed)."""
    out = np.empty(count, dtype=np.uint64)
    _load().gen_uniform(seed & (2**64 - 1), start, count, lo, hi & (2**64 - 1),
                        int(force_odd), out.ctypes.data)
    return out


def loguniform(seed: int, count: int, bmin: int = 1, bmax: int = 64, start: int = 0) -> np.ndarray:
    """Seeded values with bit length uniform in [bmin, bmax]."""
    out = np.empty(count, dtype=np.uint64)
    _load().gen_loguniform(seed & (2**64 - 1), start, count, bmin, bmax, out.ctypes.data)
    return out
