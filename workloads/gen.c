/*
 * gen.c -- seeded, counter-based synthetic input generators for the five
 * BASELINE.json configurations ("Generator
 * definition").  Shared by the oracle tests and the CUDA-path tests/bench;
 * holds none of the method's arithmetic (no primality, no modular
 * arithmetic): the only number-theoretic input, the list of k for which
 * (6k+1), (12k+1), (18k+1) are all prime, is passed in from
 * workloads/chernick_k.txt, which workloads/make_chernick_table.py wrote by
 * calling oracle/ only.
 *
 *   mix64(z)      splitmix64 finaliser (mod 2^64)
 *   U(s, i)       mix64(s + (i+1) * 0x9E3779B97F4A7C15)
 *   RNG(u,lo,hi)  lo + floor(u * (hi - lo) / 2^64)   (hi = 2^64 written as 0)
 *   SEED(c)       0x210804791 + c
 *
 *   C1  N[i] = RNG(U(SEED1,i), 0, 2^20)            i < 100000
 *   C2  N[i] = RNG(U(SEED2,i), 2^20, 2^32)         i < 2^24
 *   C3  N[i] = RNG(U(SEED3,i), 2^49, 2^64) | 1     i < 2^26
 *   C4  N[i] = i                                   i < 2^32
 *   C5  i < 2^28; (i & 4095) == 4095 -> 2^64 - 59
 *                 (i & 1023) == 1023 -> Carm[i >> 10]
 *                 else L = 1 + RNG(U(SEED5 ^ 0x5555..., i), 0, 64),
 *                      N[i] = 2^(L-1) | (U(SEED5, i) & (2^(L-1) - 1))
 *       Carm[j] = (6k+1)(12k+1)(18k+1) for the j-th accepted draw
 *       k_t = 1 + RNG(U(SEED5 ^ 0xAAAA..., t), 0, 242347), t = 0, 1, ...
 *       accepted iff k_t is in the supplied valid-k list.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

#define SEED(c) (0x210804791ull + (uint64_t)(c))
#define GOLDEN 0x9E3779B97F4A7C15ull
#define CHERNICK_KMAX 242347u

static inline uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

static inline uint64_t U(uint64_t s, uint64_t i) { return mix64(s + (i + 1) * GOLDEN); }

static inline uint64_t RNG(uint64_t u, uint64_t lo, uint64_t hi) {
    uint64_t w = hi - lo; /* hi = 2^64 passed as 0 wraps correctly */
    return lo + (uint64_t)(((unsigned __int128)u * w) >> 64);
}

uint64_t gen_mix64(uint64_t z) { return mix64(z); }
uint64_t gen_U(uint64_t s, uint64_t i) { return U(s, i); }
uint64_t gen_RNG(uint64_t u, uint64_t lo, uint64_t hi) { return RNG(u, lo, hi); }

/* Carm[0 .. count) for config C5.  `valid_k` lists the admissible k in
 * [1, 242347].  Returns the number of draws consumed, 0 on bad input. */
uint64_t gen_carmichael_stream(const uint32_t* valid_k, size_t nvalid,
                               uint64_t* carm, size_t count) {
    uint8_t* ok = (uint8_t*)calloc(CHERNICK_KMAX + 1, 1);
    if (!ok) return 0;
    for (size_t j = 0; j < nvalid; j++)
        if (valid_k[j] >= 1 && valid_k[j] <= CHERNICK_KMAX) ok[valid_k[j]] = 1;
    uint64_t s = SEED(5) ^ 0xAAAAAAAAAAAAAAAAull;
    uint64_t t = 0;
    size_t j = 0;
    if (nvalid == 0) { free(ok); return 0; }
    while (j < count) {
        uint64_t k = 1 + RNG(U(s, t), 0, CHERNICK_KMAX);
        t++;
        if (ok[k])
            carm[j++] = (6 * k + 1) * (12 * k + 1) * (18 * k + 1);
    }
    free(ok);
    return t;
}

typedef struct {
    int cfg;
    uint64_t start;
    uint64_t* out;
    size_t lo, hi;
    const uint64_t* carm;
} gen_job;

static void* gen_worker(void* arg) {
    gen_job* g = (gen_job*)arg;
    for (size_t k = g->lo; k < g->hi; k++) {
        uint64_t i = g->start + k;
        uint64_t v;
        switch (g->cfg) {
        case 1: v = RNG(U(SEED(1), i), 0, 1ull << 20); break;
        case 2: v = RNG(U(SEED(2), i), 1ull << 20, 1ull << 32); break;
        case 3: v = RNG(U(SEED(3), i), 1ull << 49, 0) | 1ull; break;
        case 4: v = i; break;
        case 5:
            if ((i & 4095) == 4095) {
                v = 18446744073709551557ull; /* 2^64 - 59 */
            } else if ((i & 1023) == 1023) {
                v = g->carm[(i >> 10) - (g->start >> 10)];
            } else {
                uint64_t L = 1 + RNG(U(SEED(5) ^ 0x5555555555555555ull, i), 0, 64);
                uint64_t top = 1ull << (L - 1);
                v = top | (U(SEED(5), i) & (top - 1));
            }
            break;
        default: v = 0;
        }
        g->out[k] = v;
    }
    return NULL;
}

/* out[k] = N_cfg[start + k] for k < count.  Returns 0 on success. */
int gen_config(int cfg, uint64_t start, size_t count, uint64_t* out,
               const uint32_t* valid_k, size_t nvalid, int threads) {
    if (cfg < 1 || cfg > 5) return -1;
    if (count == 0) return 0;
    uint64_t* carm = NULL;
    if (cfg == 5) {
        uint64_t j0 = start >> 10, j1 = (start + count - 1) >> 10;
        size_t need = (size_t)(j1 + 1);
        uint64_t* all = (uint64_t*)malloc(need * sizeof(uint64_t));
        if (!all) return -2;
        if (gen_carmichael_stream(valid_k, nvalid, all, need) == 0) { free(all); return -3; }
        carm = (uint64_t*)malloc((size_t)(j1 - j0 + 1) * sizeof(uint64_t));
        memcpy(carm, all + j0, (size_t)(j1 - j0 + 1) * sizeof(uint64_t));
        free(all);
    }
    if (threads < 1) threads = 1;
    if ((size_t)threads > count) threads = (int)count;
    gen_job* jobs = (gen_job*)calloc((size_t)threads, sizeof(gen_job));
    pthread_t* tids = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
    for (int t = 0; t < threads; t++) {
        jobs[t].cfg = cfg;
        jobs[t].start = start;
        jobs[t].out = out;
        jobs[t].lo = count * (size_t)t / (size_t)threads;
        jobs[t].hi = count * (size_t)(t + 1) / (size_t)threads;
        jobs[t].carm = carm;
    }
    for (int t = 1; t < threads; t++) pthread_create(&tids[t], NULL, gen_worker, &jobs[t]);
    gen_worker(&jobs[0]);
    for (int t = 1; t < threads; t++) pthread_join(tids[t], NULL);
    free(jobs);
    free(tids);
    free(carm);
    return 0;
}

/* Generic seeded uniform draws RNG(U(seed, start+k), lo, hi) (hi = 0 means
 * 2^64), optionally forced odd; for edge-case and sweep tests. */
void gen_uniform(uint64_t seed, uint64_t start, size_t count, uint64_t lo,
                 uint64_t hi, int force_odd, uint64_t* out) {
    for (size_t k = 0; k < count; k++) {
        uint64_t v = RNG(U(seed, start + k), lo, hi);
        out[k] = force_odd ? (v | 1ull) : v;
    }
}

/* Seeded log-uniform bit length in [bmin, bmax]: top bit forced. */
void gen_loguniform(uint64_t seed, uint64_t start, size_t count, int bmin,
                    int bmax, uint64_t* out) {
    for (size_t k = 0; k < count; k++) {
        uint64_t i = start + k;
        uint64_t L = (uint64_t)bmin + RNG(U(seed ^ 0x5555555555555555ull, i), 0,
                                          (uint64_t)(bmax - bmin + 1));
        uint64_t top = 1ull << (L - 1);
        out[k] = top | (U(seed, i) & (top - 1));
    }
}
