"""Pins of the CPU oracle (oracle/oracle.c) against facts fixed by the paper
and by number theory -- never against the oracle itself or the CUDA path.

Each test names what it pins.  A plausible mistake in the oracle (dropped
base, wrong s-chain bound, off-by-one sqrt bound, wrong sign in the -1 check,
non-reduced base) fails at least one of these.
"""
import math
import os

import numpy as np
import pytest
import sympy
from sympy.ntheory.primetest import is_strong_bpsw_prp, mr as sympy_mr

import oracle
import workloads

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _rows(name):
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.split("#", 1)[0].strip()
            if line:
                yield line.split()


# --- the paper's own worked example and table --------------------------------
def test_paper_worked_example():
    """isprime([1,2,3,4,5]) = [0 1 1 0 1]."""
    rows = list(_rows("paper_example.txt"))
    inp = [int(x) for x in rows[0]]
    exp = [int(x) for x in rows[1]]
    assert oracle.isprime(inp).tolist() == exp


def test_table1_division_counts_pin_sieve():
    """PAPER.md:231-246 (Table 1) via the paper's counting rule at PAPER.md:226-229:
    each prime q <= floor(sqrt(N)) is divided into every n in 1..N with q < n,
    i.e. contributes N - q.  Pins oracle.sieve (the primes up to 10^4)."""
    for n_s, div_s in _rows("table1_divisions.txt"):
        N, expected = int(n_s), int(div_s)
        r = math.isqrt(N)
        mask = oracle.sieve(r + 1)
        primes = np.nonzero(mask)[0].astype(np.int64)
        assert int((N - primes).sum()) == expected, N


# --- definition-level pins ----------------------------------------------------
def test_zero_and_one_not_prime():
    """0 and 1 are not prime."""
    assert oracle.isprime([0, 1]).tolist() == [0, 0]
    assert not oracle.trial_division(0) and not oracle.trial_division(1)
    assert not oracle.miller_rabin(0) and not oracle.miller_rabin(1)


def test_brute_force_below_1e6_vs_sympy_sieve():
    """Every n < 10^6 against sympy's own sieve (an independent library), and
    pi(10^6) = 78498."""
    N = np.arange(10**6, dtype=np.uint64)
    got = oracle.isprime(N)
    ref = np.zeros(10**6, dtype=np.uint8)
    ref[np.fromiter(sympy.sieve.primerange(2, 10**6), dtype=np.int64)] = 1
    assert np.array_equal(got, ref)
    assert int(got.sum()) == 78498


def test_sieve_equals_trial_division_and_mr_small():
    """Three different oracle algorithms agree on [0, 2^17): the sieve, trial
    division and 7-base MR (with base reduction, reading G3)."""
    n = 1 << 17
    s = oracle.sieve(n)
    td = oracle.isprime(np.arange(n, dtype=np.uint64))
    assert np.array_equal(s, td)
    mr = np.array([oracle.miller_rabin(k) for k in range(0, n, 7)], dtype=np.uint8)
    assert np.array_equal(mr, s[::7])


def test_pi_1e9():
    """pi(10^9) = 50847534 (closed count; BASELINE.json north_star)."""
    assert oracle.dense_range(0, 10**9 + 1).sum() == 50847534


@pytest.mark.slow
def test_pi_2_32():
    """pi(2^32) = 203280221 (config C4's validation count)."""
    assert oracle.dense_range(0, 1 << 32).sum() == 203280221


def test_dense_range_offsets():
    """dense_range(lo, n) is the slice [lo, lo+n) of the sieve."""
    s = oracle.sieve(3_000_000)
    assert np.array_equal(oracle.dense_range(1_234_567, 1_000_000), s[1_234_567:2_234_567])
    with pytest.raises(ValueError):
        oracle.dense_range((1 << 32) - 5, 10)


# --- special values -------------------------------------------------------------
def test_special_values():
    """tests/golden/special_values.txt: 2^64-59 prime, 2^64-1 composite, strong
    pseudoprimes, boundary primes.  Composites carry a factorisation that the
    test multiplies out; primes are confirmed by sympy's strong BPSW test (a
    different algorithm: strong Lucas, not Miller-Rabin with Eq 4 bases)."""
    for row in _rows("special_values.txt"):
        v, exp, fac = int(row[0]), int(row[1]), row[2]
        if fac != "-":
            fs = [int(x) for x in fac.split("*")]
            assert math.prod(fs) == v and all(f > 1 for f in fs)
            assert exp == 0
        elif v >= 2:
            assert is_strong_bpsw_prp(v) == bool(exp)
        assert oracle.isprime_u64(v) == bool(exp), v
        assert oracle.isprime([v]).tolist() == [exp]


@pytest.mark.parametrize("n,bases", [
    (2047, [2]), (3277, [2]), (4033, [2]), (4681, [2]), (8321, [2]),
    (3215031751, [2, 3, 5, 7]),
    (3825123056546413051, [2, 3, 5, 7, 11, 13, 17, 19, 23]),
])
def test_strong_pseudoprimes_pass_their_bases(n, bases):
    """Known strong pseudoprimes (Jaeschke) must PASS
    the strong test to their bases -- pins that oracle_sprp is the strong test
    of Eq 1-3 (reading G2), not something stricter -- and still be composite."""
    for a in bases:
        assert oracle.sprp(n, a), (n, a)
    assert not oracle.isprime_u64(n)


def test_sprp_witnesses():
    """2047 is not a strong probable prime to base 3; the Eq 4
    set rejects 3825123056546413051 (sympy's mr agrees base by base)."""
    assert not oracle.sprp(2047, 3)
    n = 3825123056546413051
    for a in oracle.BASES:
        assert oracle.sprp(n, a) == sympy_mr(n, [a]), a
    assert not all(oracle.sprp(n, a) for a in oracle.BASES)


def test_sprp_base_reduction_reading_g3():
    """Reading G3: a base that is 0 mod n passes; otherwise reduce mod n."""
    assert oracle.sprp(5, 325)   # 325 = 0 mod 5
    assert oracle.sprp(13, 9375 + 13 * 0) == oracle.sprp(13, 9375 % 13)
    for n in range(3, 2000, 2):
        for a in oracle.BASES:
            if a % n:
                assert oracle.sprp(n, a) == oracle.sprp(n, a % n)


def test_fermat_invariant_primes_pass_every_base():
    """Textbook invariant: every prime p passes the strong test to
    every base a with a mod p != 0.  All primes < 10^4 and the boundary primes."""
    primes = list(sympy.sieve.primerange(3, 10**4)) + [
        262139, 1048573, 4294967291, 562949953421231, 4503599627370449,
        9007199254740881, (1 << 64) - 59]
    for p in primes:
        for a in oracle.BASES:
            if a % p:
                assert oracle.sprp(p, a), (p, a)


def test_chernick_carmichael_all_composite():
    """All 1675 Chernick numbers (6k+1)(12k+1)(18k+1) < 2^64 are composite
    (their factorisation is the construction).  sympy's strong test agrees base
    by base; the number of leading Eq 4 bases passed before the first witness
    is 0 for 1424, 1 for 243 and 2 for 8 of them."""
    cs = workloads.chernick_numbers()
    assert len(cs) == 1675
    got = oracle.isprime(np.array(cs, dtype=np.uint64))
    assert got.sum() == 0
    pass2 = [c for c in cs if oracle.sprp(c, 2)]
    assert pass2 == [c for c in cs if sympy_mr(c, [2])]
    lead = []
    for c in cs:
        k = 0
        while k < 7 and oracle.sprp(c, oracle.BASES[k]):
            k += 1
        lead.append(k)
    assert {k: lead.count(k) for k in set(lead)} == {0: 1424, 1: 243, 2: 8}


# --- library cross-checks ----------------------------------------------------------
def test_mulmod_powmod_vs_python_bigint():
    """oracle_mulmod / oracle_powmod against Python's exact big integers."""
    a = workloads.uniform(11, 5000, 0, 0)
    b = workloads.uniform(12, 5000, 0, 0)
    m = workloads.uniform(13, 5000, 1, 0)
    edge = [1, 2, 3, 2**32 - 1, 2**32 + 1, 2**63 - 1, 2**63, 2**63 + 1, 2**64 - 59, 2**64 - 1]
    m = np.concatenate([m, np.array(edge, dtype=np.uint64)])
    a = np.concatenate([a, np.array(edge, dtype=np.uint64) - 1])
    b = np.concatenate([b, np.array(edge, dtype=np.uint64) // 2])
    mm = oracle.mulmod_array(a, b, m)
    pm = oracle.powmod_array(a, b, m)
    for x, y, z, r1, r2 in zip(a.tolist(), b.tolist(), m.tolist(), mm.tolist(), pm.tolist()):
        assert r1 == (x * y) % z
        assert r2 == pow(x, y, z)


def test_isprime_vs_sympy_bpsw_random_64bit():
    """20,000 seeded 64-bit values (log-uniform bit length 33..64, forced odd)
    and the 3,000 odd values just below 2^64 against sympy's strong BPSW test
    (an independent primality algorithm, exact below 2^64)."""
    vals = workloads.loguniform(0xB0B, 20000, 33, 64) | np.uint64(1)
    top = np.arange((1 << 64) - 6001, (1 << 64), 2, dtype=np.uint64)
    vals = np.concatenate([vals, top])
    got = oracle.isprime(vals)
    ref = np.array([is_strong_bpsw_prp(int(v)) for v in vals.tolist()], dtype=np.uint8)
    assert np.array_equal(got, ref)
    assert got.sum() > 300


def test_isprime_vs_sympy_32bit_random():
    """Trial-division half of the oracle against sympy.isprime on 20,000 seeded
    values in [2^20, 2^32) (sympy uses hashed MR bases there: independent)."""
    vals = workloads.uniform(0xC0C, 20000, 1 << 20, 1 << 32)
    got = oracle.isprime(vals)
    ref = np.array([sympy.isprime(int(v)) for v in vals.tolist()], dtype=np.uint8)
    assert np.array_equal(got, ref)


# --- generator golden values ------------------------------------------
def test_generator_golden():
    for row in _rows("generator.txt"):
        name = row[0]
        if name == "CARM":
            carm, draws = workloads.carmichael_stream(262144)
            assert draws == int(row[1])
            assert carm[0] == int(row[2]) and carm[1] == int(row[3])
            continue
        first = [int(x) for x in row[1].split(",")]
        assert workloads.generate(name, count=4).tolist() == first
        if name in ("C1", "C2"):
            x = workloads.generate(name)
            i = np.arange(x.shape[0], dtype=np.uint64)
            assert int(np.bitwise_xor.reduce(x * (2 * i + 1))) == int(row[2], 16)


def test_generator_shards_concatenate():
    """Counter-based: any slice equals the same slice of the whole (shards)."""
    for cfg in ("C3", "C5"):
        whole = workloads.generate(cfg, count=50_000)
        parts = [workloads.generate(cfg, start=s, count=c)
                 for s, c in ((0, 12_345), (12_345, 20_000), (32_345, 17_655))]
        assert np.array_equal(np.concatenate(parts), whole)
    assert workloads.generate("C4", start=1 << 31, count=3).tolist() == [2**31, 2**31 + 1, 2**31 + 2]


def test_c1_prime_count():
    """Config C1's prime count (SURVEY.md 8(d) golden table: 7937)."""
    row = [r for r in _rows("generator.txt") if r[0] == "C1"][0]
    assert oracle.isprime(workloads.generate("C1")).sum() == int(row[3])


# ---- reduced witness sets (option witness = 2) ----------
_CSRC = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2108_04791_b200", "csrc")


def _hash_table():
    """The product's hashed-base table, read from its generated header (the
    numbers only; nothing of the product is imported)."""
    txt = open(os.path.join(_CSRC, "witness32_table.h")).read()
    mul = int(txt.split("#define ISP_HASH_MUL32", 1)[1].split()[0].rstrip("u"), 16)
    body = txt.split("#define ISP_HASH_BASE32_LIST", 1)[1]
    bases = [int(x) for x in body.replace("\\", " ").replace(",", " ").split()]
    assert len(bases) == 256
    return mul, bases


def test_spsp2_golden_list():
    """tests/golden/spsp2_below_2p32.txt (tests/golden/make_spsp2.py, oracle/
    only): 2314 entries = the survey's independent count (SURVEY.md Appendix
    A), starting 2047, 3277, 4033, 4681, 8321; each entry is
    composite (sympy) and a strong probable prime to base 2 (oracle)."""
    spsp = [int(r[0]) for r in _rows("spsp2_below_2p32.txt")]
    assert len(spsp) == 2314 and spsp == sorted(set(spsp))
    assert spsp[:5] == [2047, 3277, 4033, 4681, 8321] and spsp[-1] < 2**32
    rng = np.random.default_rng(3)
    for n in rng.choice(spsp, size=200, replace=False).tolist() + spsp[:20] + spsp[-20:]:
        assert not sympy.isprime(n) and oracle.sprp(n, 2), n
    ok = oracle.sprp_array(np.array(spsp, dtype=np.uint64), np.full(len(spsp), 2, dtype=np.uint64))
    assert ok.all()


def test_hash32_table_rejects_every_spsp2():
    """Exactness of "base 2 + hashed base" below 2^32: a composite n < 2^32
    that passes base 2 is in the oracle's list, and the product's table base
    for n's bucket must reject it (oracle strong test).  Bases are < 2047, so a
    base is never 0 mod such n (reading G3 cannot let one through)."""
    mul, bases = _hash_table()
    assert all(3 <= a < 2047 for a in bases)
    spsp = np.array([int(r[0]) for r in _rows("spsp2_below_2p32.txt")], dtype=np.uint64)
    h = ((spsp * np.uint64(mul)) & np.uint64(0xFFFFFFFF)) >> np.uint64(24)
    a = np.array(bases, dtype=np.uint64)[h.astype(np.int64)]
    assert not oracle.sprp_array(spsp, a).any()


def test_jaeschke_set_bound_is_tight():
    """{2, 13, 23, 1662803} is exact below 1,122,004,669,633 (Jaeschke 1993);
    the bound is the smallest composite passing all four, so it must be
    composite and pass each of them -- a misremembered base or bound fails
    here.  The product's constants (csrc/kernels.cuh) must be these numbers."""
    B = 1122004669633
    assert not sympy.isprime(B) and not oracle.isprime_u64(B)
    for a in (2, 13, 23, 1662803):
        assert oracle.sprp(B, a), a
    assert not all(oracle.sprp(B, a) for a in oracle.BASES)
    src = open(os.path.join(_CSRC, "kernels.cuh")).read()
    assert "c_bases_j4[3] = {13ull, 23ull, 1662803ull}" in src
    assert f"kJaeschkeBound4 = {B}ull" in src
    # below the bound the four bases agree with the oracle on seeded odd values
    rng = np.random.default_rng(7)
    n = rng.integers(1 << 32, B, size=20000, dtype=np.uint64) | np.uint64(1)
    passed = np.ones(n.shape[0], dtype=bool)
    for a in (2, 13, 23, 1662803):
        passed &= oracle.sprp_array(n, np.full(n.shape[0], a, dtype=np.uint64)).astype(bool)
    assert np.array_equal(passed, oracle.isprime(n).astype(bool))


@pytest.mark.slow
def test_definition_level_64bit_trial_division():
    """The plain definition above 2^32 ("scale this up in the
    builder's slow tests"): trial division by every prime below 2^32 -- which
    decides primality of any n < 2^64 -- against the oracle's Eq 4
    Miller-Rabin, on the first 64 C3 values (primes exactly at indices 29, 32
    and 40), 2^64-59, 2^52-47, 3825123056546413051, Chernick
    numbers and 64-bit C5 values."""
    sieve = oracle.sieve(1 << 32)
    primes = np.nonzero(sieve)[0].astype(np.uint64)
    del sieve
    c3 = workloads.generate("C3", count=64)
    c5 = workloads.generate("C5", count=4096)
    c5 = c5[c5 >= np.uint64(1 << 40)][:24]
    extra = np.array([2**64 - 59, 2**52 - 47, 3825123056546413051] + workloads.chernick_numbers()[:8], dtype=np.uint64)
    vals = np.concatenate([c3, c5, extra])
    by_definition = []
    for v in vals.tolist():
        lim = int(np.sqrt(float(v))) + 2
        p = primes[: np.searchsorted(primes, np.uint64(min(lim, 2**32 - 1)), side="right")]
        by_definition.append(int(not np.any(np.uint64(v) % p == 0)))
    assert by_definition == oracle.isprime(vals).tolist()
    assert [i for i in range(64) if by_definition[i]] == [29, 32, 40]
    assert by_definition[-11:-8] == [1, 1, 0]
