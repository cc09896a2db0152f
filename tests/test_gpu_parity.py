"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle,
bit-exact (integer output: SURVEY.md 8(c), no tolerance), on the seeded
workloads of BASELINE.json, the number-theory pin lists and the edge cases of
the boundary (include/isprime.h)."""
import os

import numpy as np
import pytest

import oracle
import workloads

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # collected on CPU boxes, skipped there
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2108_04791_b200 as isp  # noqa: E402

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
DEV = torch.device("cuda:0")


def _rows(name):
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.split("#", 1)[0].strip()
            if line:
                yield line.split()


def gpu(N: np.ndarray) -> np.ndarray:
    N = np.ascontiguousarray(N, dtype=np.uint64)
    dN = torch.from_numpy(N.view(np.int64)).to(DEV)
    dout = torch.full((N.shape[0],), 7, dtype=torch.uint8, device=DEV)  # poison
    isp.isprime_device(dN, dout, N.shape[0])
    torch.cuda.synchronize()
    return dout.cpu().numpy()


def assert_same(got, exp, N=None):
    bad = np.nonzero(got != exp)[0]
    if bad.size:
        first = bad[:8].tolist()
        vals = N[first].tolist() if N is not None else None
        pytest.fail(f"{bad.size} mismatches; first idx {first} values {vals} got {got[first].tolist()} "
                    f"expected {exp[first].tolist()}")


@pytest.fixture(autouse=True)
def _default_options():
    saved = {k: isp.get_option(k) for k in ("force_path", "bases32", "td_primes32", "td_primes64",
                                             "chunk_log2", "win64", "warp_p", "small_max", "warp_max",
                                             "witness", "sieve_cache", "sched", "fuse_bits", "count_work",
                                             "small_sieve", "graph")}
    yield
    for k, v in saved.items():
        isp.set_option(k, v)


# ------------------------------------------------------------------ pins
def test_paper_worked_example():
    """isprime([1,2,3,4,5]) = [0 1 1 0 1]."""
    assert gpu(np.array([1, 2, 3, 4, 5], dtype=np.uint64)).tolist() == [0, 1, 1, 0, 1]


def test_special_values_all_paths():
    vals = np.array([int(r[0]) for r in _rows("special_values.txt")], dtype=np.uint64)
    exp = np.array([int(r[1]) for r in _rows("special_values.txt")], dtype=np.uint8)
    assert np.array_equal(oracle.isprime(vals), exp)
    for fp in (0, 1, 2):
        isp.set_option("force_path", fp)
        assert_same(gpu(vals), exp, vals)
        # repeated so the values fill whole tiles, warps and queues
        rep = np.tile(vals, 257)
        assert_same(gpu(rep), np.tile(exp, 257), rep)


def test_chernick_and_pseudoprimes():
    cs = np.array(workloads.chernick_numbers(), dtype=np.uint64)
    sp2 = np.array([2047, 3277, 4033, 4681, 8321, 15841, 29341, 42799, 49141, 52633, 65281, 74665,
                    80581, 85489, 88357, 90751, 3215031751, 2152302898747, 3474749660383,
                    341550071728321, 3825123056546413051], dtype=np.uint64)
    N = np.concatenate([cs, sp2])
    for small_max in (0, 1 << 17):  # pipeline and short-array path
        isp.set_option("small_max", small_max)
        got = gpu(N)
        assert got.sum() == 0
        assert_same(got, oracle.isprime(N), N)


def test_boundary_primes_and_neighbours():
    centres = [2**18, 2**20, 2**31, 2**32, 2**33, 2**49, 2**50, 2**51, 2**52, 2**53, 2**61, 2**62, 2**63, 2**64 - 1]
    vals = []
    for c in centres:
        lo = max(0, c - 3000)
        hi = min(2**64, c + 3000)
        vals.extend(range(lo, hi))
    N = np.array(vals, dtype=np.uint64)
    exp = oracle.isprime(N)
    for small_max in (0, 1 << 17):  # pipeline and short-array path
        isp.set_option("small_max", small_max)
        assert_same(gpu(N), exp, N)


@pytest.mark.parametrize("witness", [0, 1, 2])
def test_fp64_class_top_bit_exact(witness):
    """The FP64 class reaches 2^51 (modmath.cuh fmul_lazy: |q - ab/n| < 1, so
    |r| < n, at the top of the range; the base-2 ladder doubles separately at
    bit length 51): random odd values of bit length 49, 50 and 51, the odd
    values just below 2^50 and 2^51, products of two primes near 2^25 and
    2^25.5, through the pipeline (every witness mode) and the short-array path."""
    isp.set_option("witness", witness)
    rng = np.random.default_rng(50 + witness)
    vals = [rng.integers(1 << (b - 1), 1 << b, size=1 << 18, dtype=np.uint64) | np.uint64(1) for b in (49, 50, 51)]
    below = [np.arange((1 << b) - 100_001, 1 << b, 2, dtype=np.uint64) for b in (50, 51)]
    ps = [33554393, 33554383, 33554371, 33554347, 33554341, 33554317]  # primes below 2^25
    qs = [47453111, 47453099, 47453053, 47453039]  # primes below 2^25.5
    semi = np.array([p * q for p in ps + qs for q in ps + qs], dtype=np.uint64)
    N = np.concatenate(vals + below + [semi])
    exp = oracle.isprime(N)
    for small_max in (0, 1 << 17):
        isp.set_option("small_max", small_max)
        assert_same(gpu(N), exp, N)
        assert_same(gpu(N[: 1 << 16]), exp[: 1 << 16], N[: 1 << 16])
        assert_same(gpu(N[-(1 << 12):]), exp[-(1 << 12):], N[-(1 << 12):])


def test_all_below_2_20_every_path():
    N = np.arange(1 << 20, dtype=np.uint64)
    exp = oracle.sieve(1 << 20)
    for fp in (0, 1, 2):
        isp.set_option("force_path", fp)
        assert_same(gpu(N), exp, N)
    assert exp.sum() == 82025


@pytest.mark.parametrize("small_max,warp_max,small_sieve", [(0, 4096, 1), (1 << 17, 0, 1), (1 << 17, 0, 0),
                                                             (1 << 17, 4096, 1), (1 << 17, 1 << 17, 1)])
def test_short_array_path_vs_pipeline(small_max, warp_max, small_sieve):
    """Short arrays (n <= small_max) take one fused launch -- one warp per
    element with one base per lane up to warp_max elements (small_warp_kernel),
    one thread per element above (small_kernel); longer ones the plan / sieve /
    classify / Miller-Rabin pipeline.  The pin lists and seeded prefixes of
    every magnitude class through each must equal the oracle."""
    isp.set_option("small_max", small_max)
    isp.set_option("warp_max", warp_max)
    isp.set_option("small_sieve", small_sieve)
    vals = np.array([int(r[0]) for r in _rows("special_values.txt")], dtype=np.uint64)
    cs = np.array(workloads.chernick_numbers(), dtype=np.uint64)
    near = np.concatenate([np.arange(max(0, c - 500), c + 500, dtype=np.uint64)
                           for c in (2**32, 2**49, 2**63)] + [np.arange(2**64 - 1000, 2**64 - 1, dtype=np.uint64)])
    for N in (vals, cs, near, workloads.generate("C1", count=100_000), workloads.generate("C5", count=100_000),
              workloads.generate("C3", count=30_000), workloads.generate("C2", count=50_000)):
        exp = oracle.isprime(N)
        assert_same(gpu(N), exp, N)
        for n in (1, 31, 257):
            assert_same(gpu(N[:n]), exp[:n], N[:n])


@pytest.mark.parametrize("bases32", [3, 7])
def test_cluster_sieve_short_arrays(bases32):
    """Short arrays through the cluster-sieve launch (small_sieve_kernel: 8
    blocks sieve [0, 2^20) in their shared memory, elements read their byte
    through distributed shared memory): every element of [0, 2^20) in shuffled
    order, the values around the 2^20 limit and around each block's segment
    boundary (multiples of 2^17), lengths that end mid-block and mid-cluster,
    and clusters with no small odd value (the vote skips the sieve) beside
    clusters with some."""
    isp.set_option("small_max", 1 << 17)
    isp.set_option("warp_max", 0)
    isp.set_option("small_sieve", 1)  # an option (default 0: small_kernel)
    isp.set_option("bases32", bases32)
    rng = np.random.default_rng(2020 + bases32)
    allv = rng.permutation(np.arange(1 << 20, dtype=np.uint64))
    s20 = oracle.sieve(1 << 20)
    for lo in range(0, 1 << 20, 1 << 17):
        seg = allv[lo:lo + (1 << 17)]
        assert_same(gpu(seg), s20[seg.astype(np.int64)], seg)
    edges = np.concatenate([np.arange(max(0, b - 300), b + 300, dtype=np.uint64)
                            for b in [k << 17 for k in range(1, 9)]])
    for n in (1, 2047, 2048, 2049, 16383, 16384, 16385, 100_000):
        N = np.resize(np.concatenate([edges, workloads.generate("C1", count=4096)]), n)
        assert_same(gpu(N), oracle.isprime(N), N)
    # 64-bit values only in the first clusters, small ones only in the last
    big = workloads.generate("C3", count=40_000)
    small = workloads.generate("C1", count=60_000)
    N = np.concatenate([big, small])
    assert_same(gpu(N), oracle.isprime(N), N)
    N = np.concatenate([small[:20_000], big[:20_000] | np.uint64(1), np.array([2, 4, 1, 0], dtype=np.uint64)])
    assert_same(gpu(N), oracle.isprime(N), N)


def test_bpsw_witness_option():
    """Option witness = 1 replaces the six remaining Eq 4 bases of the 64-bit
    Montgomery class by a strong Lucas test (Baillie-PSW, the paper's proposed
    next step).  The Chernick numbers include 251 strong
    base-2 pseudoprimes, which only the Lucas part can
    reject; with them the pins, boundary neighbours and seeded 64-bit data must
    equal the oracle, and the full C3 count must hold."""
    saved = isp.get_option("witness")
    try:
        isp.set_option("witness", 1)
        isp.set_option("small_max", 0)
        cs = np.array(workloads.chernick_numbers(), dtype=np.uint64)
        vals = np.array([int(r[0]) for r in _rows("special_values.txt")], dtype=np.uint64)
        near = np.concatenate([np.arange(c - 3000, c + 3000, dtype=np.uint64) for c in (2**49, 2**56, 2**63)]
                              + [np.arange(2**64 - 6000, 2**64 - 1, dtype=np.uint64)])
        sq = np.array([p * p for p in (4294967291, 4294967279, 65521 * 65519, 2147483647)], dtype=np.uint64)
        for N in (cs, np.tile(vals, 64), near, sq, workloads.generate("C3", count=(1 << 18) + 3),
                  workloads.generate("C5", count=(1 << 20) + 4097)):
            assert_same(gpu(N), oracle.isprime(N), N)
        N = workloads.generate("C3")
        dN = torch.from_numpy(N.view(np.int64)).to(DEV)
        dout = torch.empty(N.shape[0], dtype=torch.uint8, device=DEV)
        dcount = torch.zeros(1, dtype=torch.int64, device=DEV)
        isp.isprime_count_device(dN, dout, dcount)
        torch.cuda.synchronize()
        assert int(dcount.item()) == _counts()["C3"]
    finally:
        isp.set_option("witness", saved)


def test_reduced_witness_option():
    """Option witness = 2: below 2^32 base 2 plus one
    hashed base, below 1,122,004,669,633 the Jaeschke set {2, 13, 23,
    1662803}, above the Eq 4 set.  Every strong base-2 pseudoprime below 2^32
    (the oracle's list) must come out composite, the Jaeschke bound itself and
    the odd values around it must equal the oracle, and so must seeded data of
    every magnitude and the full C2 / C5 counts."""
    isp.set_option("witness", 2)
    isp.set_option("small_max", 0)
    spsp = np.array([int(r[0]) for r in _rows("spsp2_below_2p32.txt")], dtype=np.uint64)
    assert spsp.shape[0] == 2314
    assert not gpu(spsp).any()
    B = 1122004669633
    rng = np.random.default_rng(11)
    near = np.concatenate([np.arange(B - 200_001, B + 200_001, 2, dtype=np.uint64),
                           np.array([B], dtype=np.uint64),
                           rng.integers(1 << 32, 1 << 42, size=1 << 20, dtype=np.uint64) | np.uint64(1)])
    cs = np.array(workloads.chernick_numbers(), dtype=np.uint64)
    vals = np.array([int(r[0]) for r in _rows("special_values.txt")], dtype=np.uint64)
    for N in (near, cs, np.tile(vals, 64), workloads.generate("C2", count=(1 << 20) + 5),
              workloads.generate("C5", count=(1 << 20) + 4097)):
        assert_same(gpu(N), oracle.isprime(N), N)
    assert gpu(np.array([B], dtype=np.uint64))[0] == 0
    for cfg in ("C2", "C5"):
        N = workloads.generate(cfg)
        dN = torch.from_numpy(N.view(np.int64)).to(DEV)
        dout = torch.empty(N.shape[0], dtype=torch.uint8, device=DEV)
        dcount = torch.zeros(1, dtype=torch.int64, device=DEV)
        isp.isprime_count_device(dN, dout, dcount)
        torch.cuda.synchronize()
        assert int(dcount.item()) == _counts()[cfg], cfg


@pytest.mark.parametrize("count", [3000, 300_000])
def test_base2_ladder_around_2_63(count):
    """The base-2 ladder fuses its doubling into the reduction below 2^63 and
    uses the separate conditional doubling at or above it, chosen per warp.
    Odd values on both sides of 2^63 -- warps entirely below, entirely above
    and mixed (interleaved), in short arrays (queue left unsorted) and long
    ones (queue sorted by bit length) -- plus primes found by the oracle next
    to 2^62, 2^63 and 2^64, must equal the oracle bit for bit."""
    rng = np.random.default_rng(63)
    lo = rng.integers(1 << 62, 1 << 63, size=count, dtype=np.uint64) | np.uint64(1)
    hi = (rng.integers(0, 1 << 63, size=count, dtype=np.uint64) | np.uint64(1 << 63)) | np.uint64(1)
    mixed = np.empty(2 * count, dtype=np.uint64)
    mixed[0::2], mixed[1::2] = lo, hi
    near = []
    for c in ((1 << 62), (1 << 63), (1 << 64) - 1):
        cand = np.array([c - k for k in range(1, 4000, 2)] + [c + k for k in range(1, 4000, 2) if c + k < (1 << 64)],
                        dtype=np.uint64)
        near.append(cand[oracle.isprime(cand) == 1])
    N = np.concatenate([lo, hi, mixed] + near)
    isp.set_option("small_max", 0)  # through the pipeline's witness kernels
    assert_same(gpu(N), oracle.isprime(N), N)


# ------------------------------------------------------------------ configs, reduced sizes (bit-exact)
@pytest.mark.parametrize("cfg,count", [("C1", 100_000), ("C2", (1 << 20) + 777), ("C3", (1 << 18) + 3),
                                       ("C5", (1 << 20) + 4097)])
def test_config_prefix_bit_exact(cfg, count):
    N = workloads.generate(cfg, count=count)
    assert_same(gpu(N), oracle.isprime(N), N)


def test_c4_prefix_bit_exact():
    n = (1 << 24) + 13
    N = np.arange(n, dtype=np.uint64)
    assert_same(gpu(N), oracle.dense_range(0, n), N)


def test_dense_range_path_and_fallback():
    """Chunks the plan samples as a dense range N[i] = N0 + i below 2^32 are
    sieved and classified in one pass (dense_kernel, no global bitmap).  Odd
    and even starting points, ragged lengths, multiple chunks, a range ending
    at 2^32, and ranges with a few foreign elements the sampling cannot see
    (the kernel detects them and the classify pass redoes the chunk without
    the window) must all equal the oracle."""
    cases = [(0, (1 << 21) + 5), (1_000_001, (1 << 20) + 999), ((1 << 32) - (1 << 21) - 3, (1 << 21) + 3),
             (123_456_788, 3 << 20)]
    for lo, n in cases:
        N = np.arange(lo, lo + n, dtype=np.uint64)
        exp = oracle.dense_range(lo, n)
        assert_same(gpu(N), exp, N)
        isp.set_option("chunk_log2", 20)  # several chunks, each its own dense window
        assert_same(gpu(N), exp, N)
        isp.set_option("chunk_log2", 28)
    rng = np.random.default_rng(4)
    N = np.arange(7_000_000, 7_000_000 + (1 << 21), dtype=np.uint64)
    hit = rng.choice(N.shape[0], size=37, replace=False)
    N[hit] = rng.integers(0, 2**64 - 1, size=37, dtype=np.uint64, endpoint=True)
    N[hit[:5]] = np.array([2, 1, 0, (1 << 64) - 59, 4294967291], dtype=np.uint64)
    assert_same(gpu(N), oracle.isprime(N), N)


@pytest.mark.parametrize("lo,n", [(1, 1 << 28), (3, (1 << 20) + 5), ((1 << 31) + 7, (1 << 26) + 3),
                                  ((1 << 32) - (1 << 22) - 1, 1 << 21), (0, (1 << 20) + 1), (2, 1 << 21)])
def test_stride2_range_every_element(lo, n):
    """Arithmetic progressions of stride 2 -- odd numbers in a restricted
    range and the even ones -- go to dense_kernel (no global
    bitmap): N[i] = lo + 2 i, every element compared with the oracle's sieve."""
    isp.set_option("small_max", 0)
    dN = torch.arange(lo, lo + 2 * n, 2, dtype=torch.int64, device=DEV)
    dout = torch.full((n,), 7, dtype=torch.uint8, device=DEV)
    isp.reset_stats()
    isp.isprime_device(dN, dout, n)
    torch.cuda.synchronize()
    del dN
    st = isp.get_stats()
    assert st["queued32"] == 0 and st["queued64"] == 0  # no element left for the witness kernels
    exp = _sieve32()[lo:lo + 2 * n:2]
    got = dout.cpu().numpy()
    assert_same(got, exp, np.arange(lo, lo + 2 * n, 2, dtype=np.uint64))
    del dout
    torch.cuda.empty_cache()


def test_stride2_range_with_foreign_elements():
    """A stride-2 range with a few planted foreign values: dense_kernel sees
    the mismatch and the classify pass redoes the chunk without the window."""
    rng = np.random.default_rng(22)
    N = np.arange(9_000_001, 9_000_001 + 2 * (1 << 21), 2, dtype=np.uint64)
    hit = rng.choice(N.shape[0], size=41, replace=False)
    N[hit] = rng.integers(0, 2**64 - 1, size=41, dtype=np.uint64, endpoint=True)
    N[hit[:4]] = np.array([2, 9, (1 << 64) - 59, 4294967291], dtype=np.uint64)
    isp.set_option("small_max", 0)
    assert_same(gpu(N), oracle.isprime(N), N)


def test_sieve_cache_reuses_held_window():
    """Option sieve_cache = 1 lets a call reuse the bitmap an earlier call
    sieved; a later window inside the held one must index the bitmap from
    the held window's start (plan_kernel publishes the held range)."""
    isp.set_option("sieve_cache", 1)
    isp.set_option("small_max", 0)
    rng = np.random.default_rng(12)
    first = rng.integers(0, 1 << 22, size=1 << 21, dtype=np.uint64)
    assert_same(gpu(first), oracle.isprime(first), first)
    for lo, hi in ((700_000, 710_000), (3_000_001, 3_100_000), (1 << 21, 1 << 22)):
        N = rng.integers(lo, hi, size=1 << 20, dtype=np.uint64)
        assert_same(gpu(N), oracle.isprime(N), N)


def test_c4_shard_window_bit_exact():
    lo = (1 << 32) - (1 << 22) - 99
    N = np.arange(lo, 1 << 32, dtype=np.uint64)
    assert_same(gpu(N), oracle.dense_range(lo, N.shape[0]), N)


@pytest.mark.parametrize("witness", [0, 1, 2])
def test_random_all_magnitudes_bit_exact(witness):
    """2^22 values drawn three ways -- uniform over all of [0, 2^64), uniform
    bit length 1..64, and odd values just above/below powers of two -- through
    the full pipeline, every element compared with the oracle (beyond the
    seeded BASELINE.json configurations)."""
    isp.set_option("small_max", 0)
    saved = isp.get_option("witness")
    try:
        isp.set_option("witness", witness)
        rng = np.random.default_rng(2108 + witness)
        n = 1 << 20
        uni = rng.integers(0, 2**64 - 1, size=n, dtype=np.uint64, endpoint=True)
        bl = rng.integers(1, 65, size=n)
        lo = rng.integers(0, 2**63, size=n, dtype=np.uint64)
        logu = np.array([(1 << (b - 1)) | (int(x) & ((1 << (b - 1)) - 1)) for b, x in zip(bl.tolist(), lo.tolist())],
                        dtype=np.uint64)
        k = rng.integers(1, 64, size=n)
        off = rng.integers(0, 1 << 12, size=n)
        edge = np.array([((1 << int(a)) + int(o)) | 1 if (i & 1) else max(3, ((1 << int(a)) - int(o)) | 1)
                         for i, (a, o) in enumerate(zip(k.tolist(), off.tolist()))], dtype=np.uint64)
        N = np.concatenate([uni, logu, edge, rng.permutation(np.concatenate([uni[: n // 2], logu[: n // 2]]))])
        assert_same(gpu(N), oracle.isprime(N), N)
    finally:
        isp.set_option("witness", saved)


# ------------------------------------------------------------------ full sizes (count + sampled elements)
def _counts():
    return {r[0]: int(r[2]) for r in _rows("config_counts.txt")}


@pytest.mark.parametrize("cfg", ["C1", "C2", "C3", "C5"])
def test_config_full_size(cfg):
    """Full BASELINE.json size through isprime_count_device (the launch
    configuration bench.py times): EVERY element equals the oracle's
    (PAPER.md:11-20 output definition; the oracle runs on all host cores), and
    the device count equals the oracle's count stored by
    tests/golden/make_golden.py."""
    N = workloads.generate(cfg)
    dN = torch.from_numpy(N.view(np.int64)).to(DEV)
    dout = torch.full((N.shape[0],), 7, dtype=torch.uint8, device=DEV)  # poison
    dcount = torch.zeros(1, dtype=torch.int64, device=DEV)
    isp.isprime_count_device(dN, dout, dcount)
    torch.cuda.synchronize()
    assert int(dcount.item()) == _counts()[cfg]
    got = dout.cpu().numpy()
    del dN, dout
    exp = oracle.isprime(N)
    assert_same(got, exp, N)
    assert int(exp.sum()) == _counts()[cfg]
    if cfg == "C5":
        assert np.all(got[4095::4096] == 1)          # 2^64 - 59
        assert np.all(got[1023::1024][(np.arange(1023, N.shape[0], 1024) & 4095) != 4095] == 0)  # Chernick
    torch.cuda.empty_cache()


_SIEVE32 = []


def _sieve32():
    """The oracle's plain sieve of [0, 2^32) (one ~1 min single-thread run),
    kept for every dense-range comparison of this module."""
    if not _SIEVE32:
        _SIEVE32.append(oracle.sieve(1 << 32))
    return _SIEVE32[0]


def _compare_dense(dout, lo, n, step=1 << 28):
    """dout (device) against the oracle's sieve over [lo, lo + n) (lo + n <=
    2^32), element by element, copied back in slices."""
    exp = _sieve32()[lo:lo + n]
    for s0 in range(0, n, step):
        s1 = min(n, s0 + step)
        got = dout[s0:s1].cpu().numpy()
        bad = np.nonzero(got != exp[s0:s1])[0]
        if bad.size:
            first = (bad[:8] + s0).tolist()
            pytest.fail(f"{bad.size} mismatches in [{s0}, {s1}); first idx {first} "
                        f"values {[lo + i for i in first]} got {got[bad[:8]].tolist()} "
                        f"expected {exp[first].tolist()}")


def test_c4_full_dense_range_every_element():
    """Config C4: N = 0 .. 2^32-1 in the launch configuration bench.py times.
    All 2^32 output bytes equal the oracle's plain sieve of [0, 2^32)
    (PAPER.md:22), and the count is pi(2^32) = 203,280,221."""
    n = 1 << 32
    dN = torch.arange(n, dtype=torch.int64, device=DEV)
    dout = torch.full((n,), 7, dtype=torch.uint8, device=DEV)
    dcount = torch.zeros(1, dtype=torch.int64, device=DEV)
    isp.isprime_count_device(dN, dout, dcount)
    torch.cuda.synchronize()
    assert int(dcount.item()) == 203280221
    del dN
    torch.cuda.empty_cache()
    assert int(_sieve32().sum(dtype=np.int64)) == 203280221
    _compare_dense(dout, 0, n)
    del dout
    torch.cuda.empty_cache()


@pytest.mark.parametrize("lo,n", [(0, 1 << 28), (1, (1 << 28) + 7), (3, 553356671), (0, 552977921),
                                  (1, (1 << 20) + 3), ((1 << 31) + 1, (1 << 28) + 31)])
def test_dense_kernel_multi_segment_every_element(lo, n):
    """dense_kernel over many segments per block (2^28 values = ~1366 odd
    segments, ~9 per block: both shared buffers, the "buffer empty" hand-over
    at k >= 2), odd and even starts (the pair path's even element is the high
    byte when lo is odd: lo = 1 makes out[1] the prime 2), and the lengths
    whose last segment overlaps the range in one or two elements (the tail
    loop), written into a poisoned buffer and compared element by element."""
    dN = torch.arange(lo, lo + n, dtype=torch.int64, device=DEV)
    dout = torch.full((n,), 7, dtype=torch.uint8, device=DEV)
    isp.set_option("small_max", 0)
    isp.isprime_device(dN, dout, n)
    torch.cuda.synchronize()
    del dN
    _compare_dense(dout, lo, n)
    del dout
    torch.cuda.empty_cache()


def test_more_than_2_32_elements():
    """n > 2^32 elements (include/isprime.h: "n may exceed 2^32"): N[i] = i mod
    2^32 for i < 2^32 + 2^20, so the count is pi(2^32) + pi(2^20) = 203,280,221
    + 82,025, and every element equals the oracle (the first 2^32 the sieve of
    [0, 2^32), the rest the sieve of [0, 2^20))."""
    n = (1 << 32) + (1 << 20)
    # filled 2^30 elements at a time: one torch kernel over more than 2^32
    # elements wrote zeros past 2^32 here (torch 2.11 arange / bitwise_and)
    dN = torch.empty(n, dtype=torch.int64, device=DEV)
    for s0 in range(0, n, 1 << 30):
        m = min(1 << 30, n - s0)
        torch.arange(s0, s0 + m, dtype=torch.int64, device=DEV, out=dN[s0:s0 + m])
        dN[s0:s0 + m].bitwise_and_(0xFFFFFFFF)
    assert dN[1 << 32: (1 << 32) + 3].tolist() == [0, 1, 2]
    dout = torch.empty(n, dtype=torch.uint8, device=DEV)
    dcount = torch.zeros(1, dtype=torch.int64, device=DEV)
    isp.isprime_count_device(dN, dout, dcount)
    torch.cuda.synchronize()
    assert int(dcount.item()) == 203280221 + 82025
    tail = dout[1 << 32:].cpu().numpy()
    assert_same(tail, oracle.sieve(1 << 20), np.arange(1 << 20, dtype=np.uint64))
    del dN
    _compare_dense(dout, 0, 1 << 32)
    del dout
    torch.cuda.empty_cache()


def test_force_path_equivalence_all_32bit():
    """SPEC.md:392 analogue over the ENTIRE 32-bit domain: sieve path vs
    trial-division + Miller-Rabin path ({2,7,61}) vs Miller-Rabin with the full
    Eq 4 base set vs base 2 + one hashed base (option witness = 2).
    Every path's output equals the oracle's sieve of [0, 2^32) element by
    element."""
    step = 1 << 28
    outs = {}
    dN = torch.empty(step, dtype=torch.int64, device=DEV)
    o = {k: torch.empty(step, dtype=torch.uint8, device=DEV) for k in ("sieve", "mr3", "mr7", "mrh")}
    total = 0
    for base in range(0, 1 << 32, step):
        torch.arange(base, base + step, dtype=torch.int64, device=DEV, out=dN)
        isp.set_option("force_path", 1); isp.set_option("bases32", 3)
        isp.isprime_device(dN, o["sieve"])
        isp.set_option("force_path", 2); isp.set_option("bases32", 3)
        isp.isprime_device(dN, o["mr3"])
        isp.set_option("bases32", 7)
        isp.isprime_device(dN, o["mr7"])
        isp.set_option("bases32", 3); isp.set_option("witness", 2)  # base 2 + hashed base
        isp.isprime_device(dN, o["mrh"])
        isp.set_option("witness", 0)
        torch.cuda.synchronize()
        assert torch.equal(o["sieve"], o["mr3"]), base
        assert torch.equal(o["sieve"], o["mr7"]), base
        assert torch.equal(o["sieve"], o["mrh"]), base
        _compare_dense(o["sieve"], base, step)
        total += int(o["sieve"].sum(dtype=torch.int64).item())
    assert total == 203280221


# ------------------------------------------------------------------ scratch memory
@pytest.mark.parametrize("cfg", ["C5", "C4"])
def test_scratch_memory_bound(cfg):
    """The library's device scratch (queues: 8 bytes per element of a chunk,
    kernels.cuh Queues; the sieve bitmap; tables) stays below 2x the input's
    bytes on the headline configurations, measured as the drop in free device
    memory across a first call after isprime_shutdown()."""
    n = workloads.CONFIGS[cfg][1]
    if cfg == "C4":
        dN = torch.arange(n, dtype=torch.int64, device=DEV)
    else:
        dN = torch.from_numpy(workloads.generate(cfg).view(np.int64)).to(DEV)
    dout = torch.empty(n, dtype=torch.uint8, device=DEV)
    torch.cuda.synchronize()
    isp.shutdown()
    free0 = torch.cuda.mem_get_info()[0]
    isp.isprime_device(dN, dout)
    torch.cuda.synchronize()
    used = free0 - torch.cuda.mem_get_info()[0]
    assert used <= 2 * 8 * n, (cfg, used, 8 * n)
    if cfg == "C5":
        assert used <= 1.25 * 8 * n, (cfg, used, 8 * n)
    del dN, dout
    torch.cuda.empty_cache()


# ------------------------------------------------------------------ streams and threads
def test_calls_on_two_streams_and_threads():
    """The library keeps one set of queues per device: a call on another
    stream waits for the previous call's completion event (isprime.cu
    last_done), so back-to-back calls on two streams with no host sync in
    between, and host-API calls from two threads at once, all stay exact."""
    import threading
    A = np.concatenate([workloads.generate("C5", count=1 << 20), workloads.generate("C2", count=1 << 19)])
    B = np.concatenate([workloads.generate("C3", count=1 << 20), workloads.generate("C1", count=50_000)])
    expA, expB = oracle.isprime(A), oracle.isprime(B)
    isp.set_option("small_max", 0)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    dA = torch.from_numpy(A.view(np.int64)).to(DEV)
    dB = torch.from_numpy(B.view(np.int64)).to(DEV)
    torch.cuda.synchronize()
    outs = []
    for k in range(3):
        oA = torch.full((A.shape[0],), 7, dtype=torch.uint8, device=DEV)
        oB = torch.full((B.shape[0],), 7, dtype=torch.uint8, device=DEV)
        torch.cuda.synchronize()
        isp.isprime_device(dA, oA, stream=s1)
        isp.isprime_device(dB, oB, stream=s2)
        isp.isprime_device(dA, oA, stream=s2 if k == 2 else s1)
        outs.append((oA, oB))
    torch.cuda.synchronize()
    for oA, oB in outs:
        assert_same(oA.cpu().numpy(), expA, A)
        assert_same(oB.cpu().numpy(), expB, B)
    res = {}

    def host_call(name, N):
        res[name] = isp.isprime(N)

    th = [threading.Thread(target=host_call, args=(nm, N)) for nm, N in (("A", A), ("B", B), ("A2", A))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert_same(res["A"], expA, A)
    assert_same(res["A2"], expA, A)
    assert_same(res["B"], expB, B)


# ------------------------------------------------------------------ options never change a bit
def test_options_do_not_change_results():
    N = np.concatenate([workloads.generate("C5", count=300_000), workloads.generate("C2", count=100_000),
                        workloads.generate("C1", count=50_000)])
    exp = oracle.isprime(N)
    for key, vals in (("td_primes32", (0, 1, 5, 128)), ("td_primes64", (0, 3, 128)), ("win64", (1, 2, 3)),
                      ("force_path", (0, 1, 2)), ("chunk_log2", (16, 17, 28)), ("warp_p", (17, 600, 65536)),
                      ("witness", (1, 2, 0)), ("sched", (0, 1, 2)), ("fuse_bits", (0, 51, 32)),
                      ("graph", (0, 1))):
        saved = isp.get_option(key)
        for v in vals:
            isp.set_option(key, v)
            assert_same(gpu(N), exp, N)
        isp.set_option(key, saved)


# ------------------------------------------------------------------ fused witness tests in classify
@pytest.mark.parametrize("fuse_bits", [0, 32, 51])
@pytest.mark.parametrize("witness,bases32", [(0, 3), (0, 7), (1, 3), (2, 3), (2, 7)])
def test_fused_classes_every_witness_mode(fuse_bits, witness, bases32):
    """Option fuse_bits: classify runs base 2 and the remaining bases itself
    for trial-division survivors below 2^fuse_bits (per-warp lists, rounds of
    32, kernels.cuh FzWarp).  Every element against the oracle on a C5 / C2
    mix, the class boundaries 2^32 and 2^51, the strong pseudoprimes and
    Chernick numbers (base-2 passers that must fail a later base), and runs of
    consecutive primes -- every list slot a survivor, so a warp-tile carries
    more survivors than one round and rounds straddle tiles."""
    isp.set_option("small_max", 0)
    isp.set_option("fuse_bits", fuse_bits)
    isp.set_option("witness", witness)
    isp.set_option("bases32", bases32)
    sp2 = np.array([int(r[0]) for r in _rows("special_values.txt")], dtype=np.uint64)
    cs = np.array(workloads.chernick_numbers(), dtype=np.uint64)
    s32 = oracle.sieve(1 << 22)
    primes_small = np.nonzero(s32)[0].astype(np.uint64)[-40_000:]  # consecutive primes below 2^22
    near = np.concatenate([np.arange(c - 20_001, c + 20_001, 2, dtype=np.uint64) for c in (2**32, 2**51)])
    N = np.concatenate([workloads.generate("C5", count=200_003), workloads.generate("C2", count=100_000),
                        np.tile(np.concatenate([sp2, cs]), 9), primes_small, near])
    exp = oracle.isprime(N)
    assert_same(gpu(N), exp, N)
    st0 = isp.get_stats()
    assert st0["passed32"] <= st0["queued32"] and st0["passed64"] <= st0["queued64"]
    # every element a prime below 2^32 (no window for the tail: force the MR path)
    isp.set_option("force_path", 2)
    P = np.tile(primes_small, 3)
    assert_same(gpu(P), np.ones(P.shape[0], dtype=np.uint8), P)


def test_fused_stats_count_like_the_queues():
    """fuse_bits moves the witness tests, not the counts: trial-division
    survivors and base-2 passes per class are the same numbers with the lists
    in classify as with the queues and witness kernels."""
    isp.set_option("small_max", 0)
    N = np.concatenate([workloads.generate("C5", count=1 << 20), workloads.generate("C2", count=1 << 18)])
    res = {}
    for fb in (0, 32, 51):
        isp.set_option("fuse_bits", fb)
        isp.reset_stats()
        gpu(N)
        st = isp.get_stats()
        res[fb] = tuple(st[k] for k in ("queued32", "queued64", "passed32", "passed64"))
    assert res[0] == res[32] == res[51], res


def test_count_work_instantiations_change_nothing():
    """Option count_work runs separate kernel instantiations that count the
    algorithmic products; the result stays bit-exact and every class reports
    work (fused 32-bit tests in classify, FP64 and Montgomery classes in the
    witness kernels)."""
    isp.set_option("small_max", 0)
    N = np.concatenate([workloads.generate("C5", count=1 << 19), workloads.generate("C2", count=1 << 18)])
    exp = oracle.isprime(N)
    isp.set_option("count_work", 1)
    isp.reset_stats()
    assert_same(gpu(N), exp, N)
    st = isp.get_stats()
    isp.set_option("count_work", 0)
    assert st["mulmods_fused"][0] > 0 and st["mulmods_fused"][1] > 0
    assert st["mulmods"][1] > 0 and st["mulmods"][3] > 0 and st["mulmods_fp64"][0] > 0
    isp.reset_stats()
    assert_same(gpu(N), exp, N)
    assert sum(isp.get_stats()["mulmods_fused"]) == 0  # counting off: nothing counted


# ------------------------------------------------------------------ boundary edge cases
@pytest.mark.parametrize("small_max", [0, 1 << 17])
def test_edge_sizes_and_alignment(small_max):
    isp.set_option("small_max", small_max)
    N = workloads.generate("C5", count=70_001)
    exp = oracle.isprime(N)
    for n in (0, 1, 2, 3, 7, 8, 31, 2047, 2048, 2049, 4097, 70_001):
        if n == 0:
            isp.isprime_device(0, 0, 0)
            continue
        assert_same(gpu(N[:n]), exp[:n], N[:n])
    # misaligned input (8-B but not 16-B) and odd output offsets
    dN = torch.from_numpy(N.view(np.int64)).to(DEV)
    dout = torch.zeros(N.shape[0] + 16, dtype=torch.uint8, device=DEV)
    for off_in, off_out in ((1, 0), (0, 1), (1, 3), (3, 5)):
        n = N.shape[0] - off_in
        isp.isprime_device(dN.data_ptr() + 8 * off_in, dout.data_ptr() + off_out, n)
        torch.cuda.synchronize()
        got = dout[off_out:off_out + n].cpu().numpy()
        assert_same(got, exp[off_in:off_in + n], N[off_in:])


def test_errors():
    lib = isp.load()
    assert lib.isprime_device(None, None, 4, None) == isp.ISP_EINVAL
    buf = torch.zeros(64, dtype=torch.uint8, device=DEV)
    assert lib.isprime_device(buf.data_ptr(), buf.data_ptr() + 8, 4, None) == isp.ISP_EINVAL


def test_host_api_pageable_and_pinned():
    N = np.concatenate([workloads.generate("C5", count=(1 << 24) + 1001), workloads.generate("C1", count=5000)])
    exp = oracle.isprime(N[::97])
    got = isp.isprime(N)
    assert_same(got[::97], exp, N[::97])
    tN = torch.from_numpy(N.view(np.int64)).pin_memory()
    tout = torch.empty(N.shape[0], dtype=torch.uint8).pin_memory()
    isp.isprime_into(tN, tout)
    assert np.array_equal(tout.numpy(), got)
    gpu_ref = gpu(N)
    assert np.array_equal(gpu_ref, got)


def test_count_and_popcount():
    N = workloads.generate("C2", count=1 << 20)
    dN = torch.from_numpy(N.view(np.int64)).to(DEV)
    dout = torch.empty(N.shape[0], dtype=torch.uint8, device=DEV)
    dcount = torch.zeros(1, dtype=torch.int64, device=DEV)
    isp.isprime_count_device(dN, dout, dcount)
    torch.cuda.synchronize()
    assert int(dcount.item()) == int(oracle.isprime(N).sum())
    dc2 = torch.zeros(1, dtype=torch.int64, device=DEV)
    isp.isprime_popcount_device(dout[3:], dc2, N.shape[0] - 3)  # unaligned
    torch.cuda.synchronize()
    assert int(dc2.item()) == int(dout[3:].sum(dtype=torch.int64).item())


def test_stats_reflect_plan():
    isp.reset_stats()
    N = np.arange(1 << 22, dtype=np.uint64)
    gpu(N)
    st = isp.get_stats()
    assert st["window_hi"] > st["window_lo"] and st["sieve_runs"] >= 1
    isp.reset_stats()
    isp.set_option("force_path", 2)
    gpu(workloads.generate("C3", count=1 << 16))
    st = isp.get_stats()
    assert st["sieve_runs"] == 0 and st["queued64"] > 0 and st["passed64"] > 0
    assert st["passed64"] <= st["queued64"]


# ------------------------------------------------------------------ device modmath and witness step
def test_mulmod_device_vs_oracle():
    rng = np.random.default_rng(1)
    n = 1 << 20
    m = rng.integers(0, 2**64 - 1, size=n, dtype=np.uint64, endpoint=True) | np.uint64(1)
    small = rng.integers(3, 2**32 - 1, size=n // 4, dtype=np.uint64) | np.uint64(1)
    edge = np.array([3, 5, 2**32 - 5, 2**32 + 1, 2**32 - 1, 2**63 - 25, 2**63 + 1, 2**64 - 59, 2**64 - 1],
                    dtype=np.uint64)
    logu = workloads.loguniform(91, n // 2, 2, 64) | np.uint64(1)  # every class: FP64, lazy and full REDC
    edge = np.concatenate([edge, np.array([2**51 - 129, 2**51 + 1, 2**62 - 57, 2**62 + 1, 2**50 + 1, 2**49 - 81,
                                           2**39 + 1, 2**40 - 1, 2**60 - 1, 2**60 + 1, 3 * 2**58 + 1],
                                          dtype=np.uint64)])  # + the R mod n quotient-estimate range (bit length 40..60)
    m = np.concatenate([m, small, logu, np.repeat(edge, 1000)])
    a = rng.integers(0, 2**64 - 1, size=m.shape[0], dtype=np.uint64, endpoint=True)
    b = rng.integers(0, 2**64 - 1, size=m.shape[0], dtype=np.uint64, endpoint=True)
    a[-edge.shape[0] * 1000:] = m[-edge.shape[0] * 1000:] - np.uint64(1)
    t = [torch.from_numpy(x.view(np.int64)).to(DEV) for x in (a, b, m)]
    out = torch.empty_like(t[0])
    isp.isprime_mulmod_device(*t, out)
    torch.cuda.synchronize()
    got = out.cpu().numpy().view(np.uint64)
    exp = oracle.mulmod_array(a % m, b % m, m)
    assert np.array_equal(got, exp)


@pytest.mark.parametrize("win", [1, 2, 3])
def test_sprp_device_vs_oracle(win):
    """The witness step base by base, in the arithmetic of each class (FP64
    below 2^51, 64-bit Montgomery above; window width 1..3)."""
    isp.set_option("win64", win)
    rng = np.random.default_rng(2 + win)
    n32 = rng.integers(3, 2**32 - 1, size=40000, dtype=np.uint64) | np.uint64(1)
    n64 = workloads.loguniform(77 + win, 40000, 33, 64) | np.uint64(1)
    primes = np.array([2**64 - 59, 2**63 - 25, 2**61 - 1, 4294967291, 2**49 - 81], dtype=np.uint64)
    psp = np.array([2047, 3215031751, 3825123056546413051] + workloads.chernick_numbers()[:200], dtype=np.uint64)
    ns = np.concatenate([n32, n64, primes, psp])
    bases = list(oracle.BASES) + [3, 5, 7, 61, 2**63 + 5, 2**64 - 1]
    for a in bases:
        av = np.full(ns.shape[0], a, dtype=np.uint64)
        dn = torch.from_numpy(ns.view(np.int64)).to(DEV)
        da = torch.from_numpy(av.view(np.int64)).to(DEV)
        out = torch.empty(ns.shape[0], dtype=torch.uint8, device=DEV)
        isp.isprime_sprp_device(dn, da, out)
        torch.cuda.synchronize()
        assert_same(out.cpu().numpy(), oracle.sprp_array(ns, av), ns)


# ------------------------------------------------------------------ graph replay (option "graph")
def test_graph_replay_reads_current_inputs():
    """Option graph: a call's pipeline is captured once per (pointers, n,
    options, scratch) and replayed; conditional nodes set on the device skip
    the stages a chunk does not need.  The same device buffers refilled with
    inputs that need different stages -- witness kernels (C5), fused tests only
    (C2), a dense range (dense_kernel), a stride-2 range (dense2_kernel), a
    sieve window only (C1 values) -- must each equal the oracle on replay, and
    equal the plain-launch path (graph = 0); so must several chunks of one call
    whose stages differ (chunk_log2 = 20: a dense chunk beside random ones)."""
    n = 3 << 20
    lo = 1_000_001
    inputs = [workloads.generate("C5", count=n), workloads.generate("C2", count=n),
              np.arange(lo, lo + n, dtype=np.uint64), np.arange(lo, lo + 2 * n, 2, dtype=np.uint64),
              workloads.generate("C1", count=n)]
    dN = torch.empty(n, dtype=torch.int64, device=DEV)
    dout = torch.empty(n, dtype=torch.uint8, device=DEV)
    for graph in (1, 0):
        isp.set_option("graph", graph)
        for rep in range(2):
            for N in inputs:
                dN.copy_(torch.from_numpy(np.ascontiguousarray(N).view(np.int64)))
                dout.fill_(7)
                isp.isprime_device(dN, dout, n)
                torch.cuda.synchronize()
                assert_same(dout.cpu().numpy(), oracle.isprime(N), N)
    isp.set_option("graph", 1)
    isp.set_option("chunk_log2", 20)
    N = np.concatenate([workloads.generate("C5", count=1 << 20), np.arange(lo, lo + (1 << 20), dtype=np.uint64),
                        workloads.generate("C2", count=1 << 20), workloads.generate("C1", count=(1 << 20) - 5)])
    exp = oracle.isprime(N)
    for _ in range(3):
        assert_same(gpu(N), exp, N)


# ------------------------------------------------------------------ tiny windows
@pytest.mark.parametrize("vals", [(3,), (3, 5, 7), (2, 3, 61), (31,), (61, 59, 63)])
@pytest.mark.parametrize("with_big", [False, True])
def test_window_below_64_values(vals, with_big):
    """Found by tools/fuzz_gpu.py: when every small odd value sampled by the plan
    lies below 64 (a long run of 3s), the chosen window [0, 2^b) with b < 6 held
    no whole 64-value bitmap word, the sieve wrote nothing, and classify read a
    stale word.  The plan widens such a window to [0, 64)."""
    rng = np.random.default_rng(64)
    n = 400_468
    N = np.array(vals, dtype=np.uint64)[rng.integers(0, len(vals), size=n)]
    if with_big:
        big = workloads.generate("C3", count=n)
        N = np.where(rng.integers(0, 2, size=n) == 0, N, big)
    exp = oracle.isprime(N)
    for sieve_cache in (0, 1):
        isp.set_option("sieve_cache", sieve_cache)
        assert_same(gpu(N), exp, N)
        # a wider window right after (and the held bitmap, when cached)
        M = workloads.generate("C1", count=n)
        assert_same(gpu(M), oracle.isprime(M), M)
        assert_same(gpu(N), exp, N)
