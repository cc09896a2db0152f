/*
 * isprime.h -- C-ABI of libisprime.so, the B200 (sm_100a) elementwise
 * primality classifier of arXiv 2108.04791 ("isprime_fast").
 *
 * Operation (section 1): "MATLAB's isprime function accepts
 * an input array, N, then returns which elements in the array are prime";
 * isprime([1,2,3,4,5]) = [0 1 1 0 1].  isprime_fast's "inputs and outputs are
 * identical"; its domain is 0 .. 2^64-1 (reading
 * G10).  Arrays of any shape are allowed: this library takes
 * the flattened array, preserves element order, and leaves shape to the
 * caller.
 *
 * Result: out[i] = 1 if N[i] is prime, else 0 (0 and 1 are not prime).  The
 * result is exact for every uint64 value: the large-integer class uses the
 * deterministic Miller-Rabin bases of Eq 4, the array path
 * uses a sieve of Eratosthenes when the values are small,
 * and small-prime trial division ("shrinking") in front of
 * both.  The path chosen for an element never changes its result.
 *
 * Every call returns ISP_OK (0) or a negative isp_status.  Calls are
 * thread-safe (serialised internally).  No call keeps a reference to a
 * caller buffer after it returns (host API) or after the work it enqueued
 * completes (device API).  There is no CPU fallback: without a CUDA device
 * every compute call returns ISP_ENODEV.
 */
#ifndef ISPRIME_H
#define ISPRIME_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    ISP_OK = 0,
    ISP_EINVAL = -1, /* NULL pointer with n > 0, out overlapping N, bad option */
    ISP_ENOMEM = -2, /* device or pinned-host allocation failed */
    ISP_ECUDA = -3,  /* a CUDA runtime call or kernel failed; out is undefined */
    ISP_ENODEV = -4  /* no CUDA device */
} isp_status;

/* Host-pointer front door: out[i] = isprime(N[i]) for i < n.
 *   N    host array of n uint64 values (pinned or pageable; any 8-B alignment)
 *   out  host array of n bytes, written with 0/1; must not overlap N
 * Synchronous: returns after out is complete.  Internally stages chunks to the
 * current CUDA device with overlapped H2D / compute / D2H.
 * n == 0 returns ISP_OK and may pass NULL pointers. */
int isprime(const uint64_t* N, uint8_t* out, size_t n);

/* Device-pointer front door, stream-ordered (asynchronous w.r.t. the host):
 *   dN     device array of n uint64 values on the current device
 *   dout   device array of n bytes (0/1 written for every i); must not overlap dN
 *   stream a cudaStream_t (NULL = legacy default stream)
 * Uses internal per-device scratch (plan, bitmap, queues) ordered on `stream`;
 * concurrent calls on different streams are serialised by the library. */
int isprime_device(const uint64_t* dN, uint8_t* dout, size_t n, void* stream);

/* As isprime_device, then *dcount (device pointer, one uint64) = number of
 * primes in dout (used for the multi-GPU validation reduce). */
int isprime_count_device(const uint64_t* dN, uint8_t* dout, size_t n,
                         uint64_t* dcount, void* stream);

/* *dcount = sum of dout[0..n) (device pointers, stream-ordered). */
int isprime_popcount_device(const uint8_t* dout, size_t n, uint64_t* dcount,
                            void* stream);

/* Human-readable text for a status (includes the last CUDA error string for
 * ISP_ECUDA).  Never NULL; the pointer stays valid until the next call. */
const char* isprime_strerror(int status);

/* Frees all cached per-device scratch (queues, bitmap, tables, streams). */
void isprime_shutdown(void);

/* ---- options (process-wide; for tests and tuning) --------------------------
 * key                value
 * "force_path"       0 auto (cost model), 1 sieve (window [0, 2^32) for every
 *                    value below 2^32), 2 mr (no sieve window: trial division +
 *                    Miller-Rabin for everything).  Default from env
 *                    ISPRIME_FORCE_PATH=auto|sieve|mr.  Never changes a bit of
 *                    out ("--force-path never changes any mask bit").
 * "bases32"          3: bases {2, 7, 61} for 2^32 > n (exact below 4,759,123,141,
 *                    Jaeschke; verified over all n < 2^32); 7: the full Eq 4 set.
 * "td_primes32"      number of odd primes (from 3) trial-divided into values
 *                    below 2^32 before Miller-Rabin (0..ISP_MAX_TD)
 * "td_primes64"      same for values >= 2^32.  Both are accepted in 0..ISP_MAX_TD
 *                    and rounded down to the compiled variants 0, 8, 16, 24, 32
 *                    (defaults 24 / 32: the round-2 re-sweep on the fused classify,
 *                    C2 8 / 16 / 24 primes 0.169 / 0.159 / 0.154 ms; C5 flat).
 * "chunk_log2"       device chunk size (elements) = 2^value, 16..31 (default 30;
 *                    halved while the queues of a chunk do not fit in memory)
 * "win64"            exponent window width for the 64-bit multi-base phase (1..3,
 *                    default 3; the window tables live in shared memory)
 * "sieve_cache"      0 (default): every call sieves its own window; 1: a call may
 *                    reuse the bitmap an earlier call on this device produced
 * "mr2_group"        3 or 6: 64-bit phase-2 bases run in lockstep groups of this size
 * "witness"          0 (default): the Eq 4 bases after base 2 for every
 *                    class; 1: Baillie-PSW for n >= 2^51 -- a strong Lucas test
 *                    (Selfridge parameters) after the base-2 strong test, the
 *                    paper's proposed next step; exact below
 *                    2^64 like Eq 4, so it never changes a bit of out;
 *                    2: reduced witness sets by magnitude:
 *                    n < 2^32 base 2 + one base picked by a hash of n (table
 *                    from tools/gen_witness32.c, checked against every strong
 *                    base-2 pseudoprime below 2^32); n < 1,122,004,669,633 the
 *                    Jaeschke set {2, 13, 23, 1662803}; above, Eq 4.  Exact, so
 *                    it never changes a bit of out.  Applies to the pipeline's
 *                    witness kernels (the short-array path keeps Eq 4)
 * "fuse_bits"        0, 32 (default) or 51: trial-division survivors below
 *                    2^fuse_bits are not queued; the classify kernel runs the
 *                    strong tests (base 2, then the remaining bases of the
 *                    selected witness set) itself, per warp on rounds of 32, on
 *                    the FP64 pipe.  0 queues every survivor for the witness
 *                    kernels.  Same tests, same bases: never changes a bit of out
 * "graph"            0 (default) or 1: the pipeline of a call is captured once into a
 *                    CUDA graph (cached per device, keyed by the call's pointers,
 *                    n, the options and the scratch buffers; 8 kept, least recently
 *                    used evicted) and replayed; conditional nodes that the plan and
 *                    classify kernels set on the device skip the sieve, the dense-range
 *                    kernels and the sort + witness kernels when they have nothing to
 *                    do.  Each replay reads the current contents of N, so a graph
 *                    never caches a result.  0: one stream launch per stage, chained
 *                    by programmatic dependent launch (measured faster on B200: a
 *                    conditional node costs more than the early-exit launch it
 *                    skips).  Never changes a bit of out
 * "small_max"        arrays with n <= small_max (default 131072) and force_path 0
 *                    take one fused launch (trial division + Miller-Rabin per
 *                    element) instead of the plan / sieve / queue pipeline;
 *                    0 disables it; accepted in 0..2^32-1.  Never changes a bit of out.
 * "small_sieve"      0 (default) or 1: within the short-array path, arrays longer
 *                    than warp_max run as 8-block thread-block clusters that sieve
 *                    [0, 2^20) in their shared memory and read each small element's
 *                    byte through distributed shared memory (north_star (c),
 *                    PAPER.md:279); larger elements keep trial division + strong
 *                    tests.  Never changes a bit of out
 * "warp_max"         within the short-array path, n <= warp_max (default 4096)
 *                    runs one warp per element with one Eq 4 base per lane
 *                    (latency of one exponentiation instead of seven)
 * "sieve_fs_per_int", "sieve_fixed_ns", "mr32_fs_per_bit", "mr_fixed_ns"
 *                    the plan's cost model (femtoseconds per integer of sieve
 *                    window, nanoseconds per sieve pass, femtoseconds per odd
 *                    element-bit of trial division + Miller-Rabin, nanoseconds of
 *                    witness-kernel latency floor); defaults fitted on a B200 by
 *                    tools/costfit.py (the Fig BestFit analogue).
 *                    Path choice only: never changes a bit of out
 * "warp_p"           sieve: primes below this cross off warp-cooperatively
 * "sched"            witness-kernel work distribution: 0 dynamic guided claims
 *                    from an atomic cursor per class; 1 static interleaved
 *                    rounds of 32 queue entries per warp, no atomics; 2
 *                    (default) static for the 32-bit class, dynamic for the
 *                    64-bit classes.  Never changes a bit of out
 * "kernel_timing"    1: bracket every launch with CUDA events on its stream and
 *                    accumulate per-kernel device time (isprime_get_kernel_times)
 * "count_work"       1: the witness tests count their algorithmic modular
 *                    multiplications (isprime_stats.mulmods*); separate
 *                    instantiations, so timings are taken with it off
 * Returns ISP_OK or ISP_EINVAL. */
#define ISP_MAX_TD 128
int isprime_set_option(const char* key, long long value);
long long isprime_get_option(const char* key);

/* ---- diagnostics (test hooks over the same device code as the path) ---- */
typedef struct {
    uint64_t window_lo, window_hi;   /* last chunk's sieve window [lo, hi) */
    uint64_t sieve_runs;             /* segmented-sieve passes since last reset */
    uint64_t sieved_integers;        /* integers covered by those passes */
    uint64_t queued32, queued64;     /* survivors of trial division (all chunks) */
    uint64_t passed32, passed64;     /* of those, strong probable primes to base 2 */
    uint64_t chunks;                 /* device chunks processed */
    uint64_t kernel_launches;        /* kernels launched by the library (host count) */
    uint64_t mulmods[4];             /* algorithmic modular multiplications counted while
                                        "count_work" is 1: mr1 32-bit, mr1 64-bit,
                                        mr2 32-bit, mr2 64-bit (square-and-multiply count);
                                        the 64-bit entries count the Montgomery class only */
    uint64_t mulmods_fp64[2];        /* same for the FP64 class (odd 2^32 <= n < 2^51): mr1, mr2 */
    uint64_t mulmods_fused[2];       /* same for the strong tests classify runs itself (option
                                        "fuse_bits"): base 2, remaining bases (FP64 pipe) */
} isprime_stats;

/* Synchronises the current device, copies the accumulated statistics. */
int isprime_get_stats(isprime_stats* st);
int isprime_reset_stats(void);

/* Per-kernel device time accumulated while option "kernel_timing" is 1
 * (synchronises the device).  Fills up to `max` entries; *count = entries
 * available.  Names: plan, sieve, classify, sort, mr1, mr2, popcount. */
typedef struct {
    char name[16];
    uint64_t launches;
    double ms_total;
} isprime_kernel_time;
int isprime_get_kernel_times(isprime_kernel_time* out, int max, int* count);
int isprime_reset_kernel_times(void);

/* out[i] = 1 iff n[i] (odd, >= 3) is a strong probable prime to base a[i]
 * (Eq 1-3; a reduced mod n, 0 passes), computed with the
 * device arithmetic of the witness kernels for n's class (FP64 lazy residues
 * below 2^51, 64-bit Montgomery above; window width from option "win64").
 * Device pointers, stream-ordered.  Elements with n even or < 3 give 0. */
int isprime_sprp_device(const uint64_t* dn, const uint64_t* da, uint8_t* dout,
                        size_t count, void* stream);

/* out[i] = a[i] * b[i] mod m[i] (odd m >= 3; a, b are reduced mod m first) with
 * the product the witness kernels use for m's class: FP64 lazy residues below
 * 2^51, the lazy additive Montgomery REDC below 2^62, the subtraction REDC
 * above.  Device pointers, stream-ordered.  m even -> 0. */
int isprime_mulmod_device(const uint64_t* da, const uint64_t* db,
                          const uint64_t* dm, uint64_t* dout, size_t count,
                          void* stream);

#ifdef __cplusplus
}
#endif
#endif /* ISPRIME_H */
