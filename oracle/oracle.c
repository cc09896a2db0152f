/*
 * oracle.c -- plain, slow, obviously-correct CPU oracle for elementwise
 * primality classification (arXiv 2108.04791, "isprime_fast").
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product path (the CUDA library
 * under paper_2108_04791_b200/) may include, link or call this file.  Only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference leg may load liboracle.so.  It shares no code, header, table or
 * constant generator with the CUDA path.
 *
 * What it computes (section 1): isprime(N) returns a logical
 * array of the same size as N, 1 where N[i] is prime; 0 and 1 are not prime.
 *
 * Definition used: out[i] = 1 iff N[i] >= 2 and no
 * d with 2 <= d <= floor(sqrt(N[i])) divides N[i].
 *   - N[i] < 2^32: that definition written out (trial division by every odd
 *     d with d*d <= n).
 *   - N[i] >= 2^32: the paper's deterministic Miller-Rabin (PAPER.md:37-56,
 *     section 2.1, Eq 1-4) with the Eq 4 bases {2, 325, 9375, 28178, 450775,
 *     9780504, 1795265022}, which PAPER.md:53 (citing Sinclair) states is
 *     exact for every 64-bit input.  Products are exact 128-bit
 *     (unsigned __int128), so no saturation-avoidance trick (section 2.2-2.3)
 *     is needed; ModExp is exponentiation by squaring.
 *   - Bulk dense ranges: a plain sieve of Eratosthenes (the
 *     "crosses-off multiples of primes" description), byte per integer.
 *
 * Readings of the paper:
 *   G1/G2  Eq 1-3 are read as the standard strong-probable-prime condition:
 *          a^d == 1 (mod n) or a^(2^r d) == n-1 (mod n) for some 0 <= r < s.
 *   G3     A base is reduced mod n first; a reduced base of 0 passes.
 *   G10    Domain is 0 .. 2^64-1.
 *
 * Parity pins: see tests/test_oracle.py (every function here is pinned; none
 * is "parity unpinned").
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

typedef unsigned __int128 u128;

/* Eq 4. */
static const uint64_t ORACLE_BASES[7] = {2ull, 325ull, 9375ull, 28178ull,
                                         450775ull, 9780504ull, 1795265022ull};

/* (a * b) mod m with an exact 128-bit product. */
uint64_t oracle_mulmod(uint64_t a, uint64_t b, uint64_t m) {
    if (m == 0) return 0;
    return (uint64_t)(((u128)a * (u128)b) % (u128)m);
}

/* ModExp: a^e mod m by exponentiation by squaring,
 * right-to-left over the bits of e. */
uint64_t oracle_powmod(uint64_t a, uint64_t e, uint64_t m) {
    if (m == 1) return 0;
    uint64_t result = 1;
    uint64_t base = a % m;
    while (e > 0) {
        if (e & 1) result = oracle_mulmod(result, base, m);
        base = oracle_mulmod(base, base, m);
        e >>= 1;
    }
    return result;
}

/* Strong probable-prime test of odd n >= 3 to base a (PAPER.md:37-51,
 * Eq 1-3, reading G1/G2; base reduction reading G3).  Returns 1 if n passes
 * (is a strong probable prime to base a), 0 if a is a witness of
 * compositeness. */
int oracle_sprp(uint64_t n, uint64_t a) {
    if (n < 3 || (n & 1) == 0) return 0;
    uint64_t ar = a % n;
    if (ar == 0) return 1;                 /* reading G3 */
    /* n - 1 = 2^s * d with d odd */
    uint64_t d = n - 1;
    int s = 0;
    while ((d & 1) == 0) { d >>= 1; s++; }
    uint64_t x = oracle_powmod(ar, d, n);  /* a^d, the last term of Eq 3 */
    if (x == 1 || x == n - 1) return 1;
    for (int r = 1; r < s; r++) {          /* a^(2^r d), r = 1 .. s-1 */
        x = oracle_mulmod(x, x, n);
        if (x == n - 1) return 1;
    }
    return 0;
}

/* Trial division by the plain definition: n >= 2, no d in [2, sqrt(n)]
 * divides n.  Only even d = 2 and odd d are tried (an even d > 2 divides n
 * only if 2 does).  Used for n < 2^32 where d*d cannot overflow. */
int oracle_trial_division(uint64_t n) {
    if (n < 2) return 0;
    if (n < 4) return 1;
    if ((n & 1) == 0) return 0;
    for (uint64_t d = 3; d * d <= n; d += 2)
        if (n % d == 0) return 0;
    return 1;
}

/* Deterministic Miller-Rabin with the 7 bases of Eq 4:
 * prime iff every base passes (composite on the first witness). */
int oracle_miller_rabin(uint64_t n) {
    if (n < 2) return 0;
    if (n == 2) return 1;
    if ((n & 1) == 0) return 0;
    for (int i = 0; i < 7; i++)
        if (!oracle_sprp(n, ORACLE_BASES[i])) return 0;
    return 1;
}

/* One element, as isprime would classify it. */
int oracle_isprime_u64(uint64_t n) {
    if (n < (1ull << 32)) return oracle_trial_division(n);
    return oracle_miller_rabin(n);
}

/* ---- array front door, threaded over contiguous chunks ---- */
typedef struct {
    const uint64_t* N;
    uint8_t* out;
    size_t lo, hi;
} oracle_job;

static void* oracle_worker(void* arg) {
    oracle_job* j = (oracle_job*)arg;
    for (size_t i = j->lo; i < j->hi; i++)
        j->out[i] = (uint8_t)oracle_isprime_u64(j->N[i]);
    return NULL;
}

/* out[i] = isprime(N[i]) for i < n, using `threads` POSIX threads over
 * contiguous chunks (threads <= 1: the calling thread only).  Returns the
 * number of primes found. */
uint64_t oracle_isprime_array(const uint64_t* N, uint8_t* out, size_t n,
                              int threads) {
    if (threads < 1) threads = 1;
    if ((size_t)threads > n) threads = n > 0 ? (int)n : 1;
    oracle_job* jobs = (oracle_job*)calloc((size_t)threads, sizeof(oracle_job));
    pthread_t* tids = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
    for (int t = 0; t < threads; t++) {
        jobs[t].N = N;
        jobs[t].out = out;
        jobs[t].lo = n * (size_t)t / (size_t)threads;
        jobs[t].hi = n * (size_t)(t + 1) / (size_t)threads;
    }
    for (int t = 1; t < threads; t++)
        pthread_create(&tids[t], NULL, oracle_worker, &jobs[t]);
    oracle_worker(&jobs[0]);
    for (int t = 1; t < threads; t++) pthread_join(tids[t], NULL);
    uint64_t count = 0;
    for (size_t i = 0; i < n; i++) count += out[i];
    free(jobs);
    free(tids);
    return count;
}

/* Plain sieve of Eratosthenes: is_prime[k] = 1 iff k is prime,
 * for 0 <= k < limit.  Starts from "all marked", clears 0 and 1, and for
 * every p with p*p < limit that is still marked crosses off p*p, p*p+p, ...
 * `is_prime` must hold `limit` bytes.  Returns the prime count pi(limit-1). */
uint64_t oracle_sieve(uint64_t limit, uint8_t* is_prime) {
    if (limit == 0) return 0;
    memset(is_prime, 1, (size_t)limit);
    is_prime[0] = 0;
    if (limit > 1) is_prime[1] = 0;
    for (uint64_t p = 2; p * p < limit; p++) {
        if (!is_prime[p]) continue;
        for (uint64_t m = p * p; m < limit; m += p) is_prime[m] = 0;
    }
    uint64_t count = 0;
    for (uint64_t k = 0; k < limit; k++) count += is_prime[k];
    return count;
}

/* Dense-range classification out[i] = isprime(lo + i), i < n, through the
 * plain sieve above (for the contiguous configuration C4 and its shards).
 * Requires lo + n <= 2^32 (the sieve is byte-per-integer).  Returns the
 * number of primes in the range, or UINT64_MAX on bad arguments. */
uint64_t oracle_dense_range(uint64_t lo, size_t n, uint8_t* out) {
    if (n == 0) return 0;
    if (lo + n > (1ull << 32) || lo + n < lo) return UINT64_MAX;
    uint64_t limit = lo + n;
    uint8_t* s = (uint8_t*)malloc((size_t)limit);
    if (!s) return UINT64_MAX;
    oracle_sieve(limit, s);
    memcpy(out, s + lo, n);
    free(s);
    uint64_t count = 0;
    for (size_t i = 0; i < n; i++) count += out[i];
    return count;
}

/* Strong probable-prime verdicts for a list of (n, base) pairs (used to pin
 * the device witness kernels base by base).  n must be odd >= 3. */
void oracle_sprp_array(const uint64_t* n, const uint64_t* a, uint8_t* out,
                       size_t count) {
    for (size_t i = 0; i < count; i++) out[i] = (uint8_t)oracle_sprp(n[i], a[i]);
}

/* (a*b) mod m for arrays (pins the device Montgomery library). */
void oracle_mulmod_array(const uint64_t* a, const uint64_t* b,
                         const uint64_t* m, uint64_t* out, size_t count) {
    for (size_t i = 0; i < count; i++) out[i] = oracle_mulmod(a[i], b[i], m[i]);
}

/* a^e mod m for arrays. */
void oracle_powmod_array(const uint64_t* a, const uint64_t* e,
                         const uint64_t* m, uint64_t* out, size_t count) {
    for (size_t i = 0; i < count; i++) out[i] = oracle_powmod(a[i], e[i], m[i]);
}
