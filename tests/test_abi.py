"""Host-side checks that need no GPU: the C-ABI library builds, loads and
exports every symbol include/isprime.h declares; argument validation happens
before any device work; options validate their ranges; the product package
never imports the oracle."""
import ast
import ctypes
import os
import re

import pytest

import paper_2108_04791_b200 as isp
from paper_2108_04791_b200 import _build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "isprime.h")


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[\w ]+?\*?\s*\b(isprime\w*)\s*\(", src, flags=re.M)))


def test_header_declares_the_boundary():
    names = _declared()
    for must in ("isprime", "isprime_device", "isprime_count_device", "isprime_strerror", "isprime_shutdown"):
        assert must in names
    assert set(names) == set(isp.EXPORTED_SYMBOLS)


def test_library_builds_and_exports_every_symbol():
    path = _build.build()
    lib = ctypes.CDLL(path)
    for name in _declared():
        assert hasattr(lib, name), name
    out = os.popen(f"nm -D --defined-only {path}").read()
    for name in _declared():
        assert re.search(rf"\bT {name}\b", out), name


def test_sm100a_code_in_library():
    path = _build.build()
    out = os.popen(f"cuobjdump --list-elf {path} 2>&1").read()
    assert "sm_100a" in out


def test_argument_validation_without_device_work():
    lib = isp.load()
    assert lib.isprime(None, None, 0) == isp.ISP_OK
    assert lib.isprime_device(None, None, 0, None) == isp.ISP_OK
    assert lib.isprime(None, None, 5) == isp.ISP_EINVAL
    assert lib.isprime_device(None, None, 5, None) == isp.ISP_EINVAL
    buf = ctypes.create_string_buffer(64)
    base = ctypes.addressof(buf)
    # out overlapping N
    assert lib.isprime(base, base + 8, 4) == isp.ISP_EINVAL
    assert lib.isprime_device(base, base + 3, 4, None) == isp.ISP_EINVAL
    assert lib.isprime_strerror(isp.ISP_EINVAL).decode().startswith("invalid")


def test_options_validate():
    assert isp.get_option("force_path") in (0, 1, 2)
    with pytest.raises(isp.IsPrimeError):
        isp.set_option("force_path", 3)
    with pytest.raises(isp.IsPrimeError):
        isp.set_option("td_primes32", 1000)
    with pytest.raises(isp.IsPrimeError):
        isp.set_option("no_such_key", 1)
    old = isp.get_option("win64")
    isp.set_option("win64", 3)
    assert isp.get_option("win64") == 3
    isp.set_option("win64", old)
    # trial-division counts: 0..ISP_MAX_TD accepted (rounded down to a compiled variant when used)
    for key in ("td_primes32", "td_primes64"):
        saved = isp.get_option(key)
        for bad in (-1, 129):
            with pytest.raises(isp.IsPrimeError):
                isp.set_option(key, bad)
        isp.set_option(key, 128)
        assert isp.get_option(key) == 128
        isp.set_option(key, saved)
    for key, bad, good in (("witness", 3, 2), ("small_max", -1, 0), ("small_max", 1 << 32, (1 << 32) - 1),
                           ("warp_max", -1, 64), ("fuse_bits", 33, 51), ("fuse_bits", -1, 0), ("small_sieve", 2, 0),
                           ("count_work", 2, 0), ("graph", 2, 0), ("graph", -1, 1)):
        saved = isp.get_option(key)
        with pytest.raises(isp.IsPrimeError):
            isp.set_option(key, bad)
        isp.set_option(key, good)
        assert isp.get_option(key) == good
        isp.set_option(key, saved)


def test_no_cpu_fallback_without_device():
    """Without a CUDA device the compute calls fail loudly (ENODEV)."""
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a GPU is present")
    except ImportError:
        pass
    lib = isp.load()
    a = (ctypes.c_uint64 * 4)(1, 2, 3, 4)
    o = (ctypes.c_uint8 * 4)()
    assert lib.isprime(a, o, 4) == isp.ISP_ENODEV
    with pytest.raises(isp.IsPrimeError):
        isp.isprime([1, 2, 3])


def test_product_package_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2108_04791_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            p = os.path.join(dirpath, f)
            if f.endswith(".py"):
                tree = ast.parse(open(p).read())
                for node in ast.walk(tree):
                    if isinstance(node, ast.Import):
                        assert all(not a.name.startswith("oracle") for a in node.names), p
                    if isinstance(node, ast.ImportFrom):
                        assert not (node.module or "").startswith("oracle"), p
            if f.endswith((".cu", ".cuh", ".h")):
                assert "oracle" not in open(p).read().lower(), p
