// witness.cuh -- strong-probable-prime (Miller-Rabin witness) tests on the
// device, per element, for the two phases of the witness kernels.
//
// The test (Eq 1-3, reading G2): write n - 1 = 2^s d with d
// odd; n passes base a iff a^d == 1 (mod n) or a^(2^r d) == -1 (mod n) for
// some 0 <= r < s.  Bases are reduced mod n and a reduced base of 0 passes
// (reading G3).  All values live in Montgomery form, where 1 and -1 are
// M.one and M.mone.
//
// ModExp is left-to-right exponentiation by squaring.  The
// per-lane bits of d differ across a warp, so the conditional multiply is a
// SELECT, never a branch (no divergence); for base 2 the multiply is the
// ModMultiply case-3 doubling, for other bases a fixed
// window of WIN bits (table of a^0 .. a^(2^WIN - 1)) trades multiplies for a
// register table.  Several bases of one n share d, so their chains run in
// lockstep (NB independent chains per thread = instruction-level parallelism
// for the IMAD pipe).
#pragma once
#include "modmath.cuh"

namespace isp {

// Run step(w) once per exponent bit, most significant first, for the top
// bits of dd (left-aligned): bit 31 of the 32-bit word w is the current bit.
// Two 32-bit passes instead of a 64-bit shift per step (one instruction
// instead of two in every ladder step).
template <typename F>
__device__ __forceinline__ void for_bits_msb(unsigned long long dd, int top, F&& step) {
    uint32_t lo, hi;
    asm("mov.b64 {%0, %1}, %2;" : "=r"(lo), "=r"(hi) : "l"(dd));
    const int k1 = top < 32 ? top : 32;
    uint32_t w = hi;
#pragma unroll 2
    for (int k = 0; k < k1; k++) {
        step(w);
        w += w;
    }
    w = lo;
#pragma unroll 2
    for (int k = 32; k < top; k++) {
        step(w);
        w += w;
    }
}

// ---------------------------------------------------------------- 32-bit ----
// Phase 1 (base 2).  n odd, 3 <= n < 2^32.
__device__ __forceinline__ bool sprp2_32(uint32_t n) {
    const Mont32 M = mont32_setup(n);
    uint32_t d = n - 1;
    const int s = __ffs(d) - 1;
    d >>= s;
    const int top = 31 - __clz(d);
    uint32_t x = madd32(M.one, M.one, n);  // mont(2): top bit of d
    for (int b = top - 1; b >= 0; b--) {
        x = mmul32(x, x, M);
        const uint32_t y = madd32(x, x, n);  // * 2 (ModMultiply case 3)
        x = ((d >> b) & 1u) ? y : x;
    }
    if (x == M.one || x == M.mone) return true;
    for (int r = 1; r < s; r++) {
        x = mmul32(x, x, M);
        if (x == M.mone) return true;
        if (x == M.one) return false;
    }
    return false;
}

// Phase 2: all NB bases of `bases` (each reduced mod n) in lockstep.  Returns
// true iff n passes every base.  n odd, 3 <= n < 2^32.
template <int NB>
__device__ __forceinline__ bool sprp_multi32(uint32_t n, const uint32_t* bases) {
    const Mont32 M = mont32_setup(n);
    const uint32_t R2 = mont32_r2(M);
    uint32_t d = n - 1;
    const int s = __ffs(d) - 1;
    d >>= s;
    const int top = 31 - __clz(d);
    uint32_t A[NB], x[NB];
    bool done[NB], pass[NB];
#pragma unroll
    for (int i = 0; i < NB; i++) {
        uint32_t a = bases[i];
        if (a >= n) a %= n;
        done[i] = pass[i] = (a == 0);  // reading G3: a == 0 (mod n) passes
        A[i] = mmul32(a, R2, M);
        x[i] = A[i];
    }
    for (int b = top - 1; b >= 0; b--) {
        const bool bit = (d >> b) & 1u;
#pragma unroll
        for (int i = 0; i < NB; i++) {
            const uint32_t sq = mmul32(x[i], x[i], M);
            const uint32_t y = mmul32(sq, A[i], M);
            x[i] = bit ? y : sq;
        }
    }
#pragma unroll
    for (int i = 0; i < NB; i++) {
        if (!done[i] && (x[i] == M.one || x[i] == M.mone)) done[i] = pass[i] = true;
    }
    for (int r = 1; r < s; r++) {
        bool all = true;
#pragma unroll
        for (int i = 0; i < NB; i++) {
            if (!done[i]) {
                x[i] = mmul32(x[i], x[i], M);
                if (x[i] == M.mone) done[i] = pass[i] = true;
                else if (x[i] == M.one) done[i] = true;
            }
            all &= done[i];
        }
        if (all) break;
    }
    bool ok = true;
#pragma unroll
    for (int i = 0; i < NB; i++) ok &= pass[i];
    return ok;
}

// ---------------------------------------------------------------- 64-bit ----
#ifndef ISP_MR1_UNROLL
#define ISP_MR1_UNROLL 2
#endif
constexpr int kMr1Unroll = ISP_MR1_UNROLL;  // Montgomery-class base-2 ladders (n >= 2^61); 1 / 2 / 4 measured: C3 phase 1 1.965 / 1.955 / 1.983 ms
// Base-2 ladder in K-bit windows on lazy Montgomery residues (round 2):
// 2^d R mod n (< 2n), d odd.  Each window is K - 1 plain squares and one
// square whose REDC input is shifted left by the window's digit:
// REDC(x^2 2^dig) = x^2 2^dig R^-1, so the multiplication by 2^dig costs the
// shift the one-bit ladder already pays.  The REDC bound T = x^2 2^dig <
// 4 n^2 2^dig <= n R holds for n <= 2^(62 - dig): digits up to 2^K - 1 need
// n < 2^55 for K = 3 and n < 2^59 for K = 2.  The top window starts from
// mont(1) (its square is itself).  Per bit: 8 IMAD.WIDE + 2 IMAD as before,
// the shift and the exponent bookkeeping once per window instead of per bit.
template <int K>
__device__ __forceinline__ uint64_t m2_pow_win(uint64_t d, uint64_t n, uint64_t nn, uint64_t one) {
    const int nb = 64 - __clzll((long long)d);
    const int nw = (nb + K - 1) / K;
    uint64_t x = msqr64_shl_lz_ptx(one, n, nn, (uint32_t)(d >> (K * (nw - 1))));
#pragma unroll 1
    for (int w = nw - 2; w >= 0; w--) {
        const uint32_t dig = (uint32_t)(d >> (K * w)) & ((1u << K) - 1u);
#pragma unroll
        for (int j = 0; j < K - 1; j++) x = msqr64_lz_ptx(x, n, nn);
        x = msqr64_shl_lz_ptx(x, n, nn, dig);
    }
    return mcanon64(x, n);
}

// Phase 1 (base 2).  n odd, n >= 3 (used for n >= 2^32).
__device__ __forceinline__ bool sprp2_64(uint64_t n) {
    const Mont64 M = mont64_setup(n);
    uint64_t d = n - 1;
    const int s = __ffsll((long long)d) - 1;
    d >>= s;
    const int top = 63 - __clzll((long long)d);
    uint64_t x = mdbl64(M.one, n);  // mont(2): the leading bit of d
    const unsigned int act0 = __activemask();
    const int bmax = (int)__reduce_max_sync(act0, (unsigned)(64 - __clzll((long long)n)));
    if (bmax <= 59) {
        // windowed ladder (warp-uniform width from the warp's largest n)
        const uint64_t nn = 0ull - M.ninv;
        x = bmax <= 55 ? m2_pow_win<3>(d, n, nn, M.one) : m2_pow_win<2>(d, n, nn, M.one);
    } else if (top > 0) {
        // remaining bits of d, most significant first, from the top of dd
        uint64_t dd = d << (64 - top);
        // warp-uniform choice (queues are ordered by bit length, so warps
        // rarely straddle 2^61 or 2^63): below 2^61 the fused square-and-double
        // with lazy representatives in [0, 2n); below 2^63 the same with the
        // reduction corrected every step; above, square then double
        const unsigned int act = __activemask();
        // (two 32-bit passes over the exponent below 2^61; above, a 64-bit
        // exponent register measured faster)
        if (!__any_sync(act, (unsigned)(n >> 61))) {
            const uint64_t nn = 0ull - M.ninv;
            for_bits_msb(dd, top, [&](uint32_t w) { x = msqr64_shl_lz_ptx(x, n, nn, w >> 31); });
            x = mcanon64(x, n);
        } else if (!__any_sync(act, (unsigned)(n >> 63))) {
#pragma unroll kMr1Unroll
            for (int k = 0; k < top; k++) {
                x = msqr64_shl_ptx(x, n, M.ninv, (uint32_t)(dd >> 63));
                dd += dd;
            }
        } else {
#pragma unroll kMr1Unroll
            for (int k = 0; k < top; k++) {
                x = mdbl64_if_ptx(msqr64_ptx(x, n, M.ninv), n, (uint32_t)(dd >> 63));
                dd += dd;
            }
        }
    }
    if (x == M.one || x == M.mone) return true;
    for (int r = 1; r < s; r++) {
        x = msqr64(x, M);
        if (x == M.mone) return true;
        if (x == M.one) return false;
    }
    return false;
}

// Select table[digit] (table[0] = one) without dynamic register indexing.
template <int T>
__device__ __forceinline__ uint64_t sel_table(const uint64_t (&tab)[T], uint32_t digit, uint64_t one) {
    uint64_t m = one;
#pragma unroll
    for (int k = 1; k <= T; k++) m = (digit == (uint32_t)k) ? tab[k - 1] : m;
    return m;
}

// Phase 2: NB bases in lockstep with a fixed WIN-bit window, for a modulus
// whose Montgomery context (M, R2, d, s) is already set up.  Returns true iff
// n passes every base.  Bases are reduced mod n.
// SM: the window table lives in shared memory, transposed so that lane t's
// entry (base i, digit k) is st[(i (T + 1) + k) * TS] with st = table + t:
// one LDS per base and window (conflict-free across the warp) replaces the
// 2T selects of sel_table.  TS = threads per block.
// LZ (n < 2^62): lazy additive reductions, representatives in [0, 2n),
// reduced once before the comparisons.
template <int NB, int WIN, bool SM = false, int TS = 256, bool LZ = false>
__device__ __forceinline__ bool sprp_lockstep64(const Mont64& M, uint64_t R2, uint64_t d, int s,
                                                const unsigned long long* bases, unsigned long long* st = nullptr) {
    constexpr int T = (1 << WIN) - 1;
    const uint64_t n = M.n;
    const int nbits = 64 - __clzll((long long)d);
    const int nw = (nbits + WIN - 1) / WIN;
    uint64_t tab[NB][T], x[NB];
    bool done[NB], pass[NB];
    const uint64_t nn = 0ull - M.ninv;
#pragma unroll
    for (int i = 0; i < NB; i++) {
        uint64_t a = bases[i];
        if (a >= n) a %= n;
        done[i] = pass[i] = (a == 0);
        // table entries: lazy (< 2n) in the LZ range, canonical otherwise
        tab[i][0] = LZ ? mmul64_lz_ptx(a, R2, n, nn) : mmul64_ptx(a, R2, n, M.ninv);
#pragma unroll
        for (int k = 1; k < T; k++)
            tab[i][k] = LZ ? mmul64_lz_ptx(tab[i][k - 1], tab[i][0], n, nn) : mmul64_ptx(tab[i][k - 1], tab[i][0], n, M.ninv);
        if (SM) {
            st[(i * (T + 1)) * TS] = M.one;
#pragma unroll
            for (int k = 0; k < T; k++) st[(i * (T + 1) + k + 1) * TS] = tab[i][k];
        }
    }
    {
        const uint32_t lead = (uint32_t)(d >> (WIN * (nw - 1)));  // nonzero
#pragma unroll
        for (int i = 0; i < NB; i++) x[i] = SM ? st[(i * (T + 1) + lead) * TS] : sel_table<T>(tab[i], lead, M.one);
    }
    for (int w = nw - 2; w >= 0; w--) {
        const uint32_t digit = (uint32_t)(d >> (WIN * w)) & (uint32_t)T;
        uint64_t mt[NB];
#pragma unroll
        for (int i = 0; i < NB; i++) mt[i] = SM ? st[(i * (T + 1) + digit) * TS] : sel_table<T>(tab[i], digit, M.one);
        if (LZ) {
#pragma unroll
            for (int j = 0; j < WIN; j++) {
#pragma unroll
                for (int i = 0; i < NB; i++) x[i] = msqr64_lz_ptx(x[i], n, nn);
            }
#pragma unroll
            for (int i = 0; i < NB; i++) x[i] = mmul64_lz_ptx(x[i], mt[i], n, nn);
        } else {
#pragma unroll
            for (int j = 0; j < WIN; j++) {
#pragma unroll
                for (int i = 0; i < NB; i++) x[i] = msqr64_ptx(x[i], n, M.ninv);
            }
#pragma unroll
            for (int i = 0; i < NB; i++) x[i] = mmul64_ptx(x[i], mt[i], n, M.ninv);
        }
    }
#pragma unroll
    for (int i = 0; i < NB; i++) {
        if (LZ) x[i] = mcanon64(x[i], n);
        if (!done[i] && (x[i] == M.one || x[i] == M.mone)) done[i] = pass[i] = true;
    }
    for (int r = 1; r < s; r++) {
        bool all = true;
#pragma unroll
        for (int i = 0; i < NB; i++) {
            if (!done[i]) {
                x[i] = LZ ? mcanon64(msqr64_lz_ptx(x[i], n, nn), n) : msqr64_ptx(x[i], n, M.ninv);
                if (x[i] == M.mone) done[i] = pass[i] = true;
                else if (x[i] == M.one) done[i] = true;
            }
            all &= done[i];
        }
        if (all) break;
    }
    bool ok = true;
#pragma unroll
    for (int i = 0; i < NB; i++) ok &= pass[i];
    return ok;
}

// All NB bases of `bases`, G at a time in lockstep (G | NB), stopping at the
// first group with a witness.  One Montgomery setup per n.
template <int NB, int G, int WIN, bool SM = false, int TS = 256>
__device__ __forceinline__ bool sprp_multi64(uint64_t n, const unsigned long long* bases,
                                             unsigned long long* st = nullptr) {
    const Mont64 M = mont64_setup(n);
    const uint64_t R2 = mont64_r2(M);
    uint64_t d = n - 1;
    const int s = __ffsll((long long)d) - 1;
    d >>= s;
    // warp-uniform: lazy reductions when every active lane's n < 2^62
    if (!__any_sync(__activemask(), (unsigned)(n >> 62))) {
#pragma unroll 1
        for (int g = 0; g < NB; g += G)
            if (!sprp_lockstep64<G, WIN, SM, TS, true>(M, R2, d, s, bases + g, st)) return false;
        return true;
    }
#pragma unroll 1
    for (int g = 0; g < NB; g += G)
        if (!sprp_lockstep64<G, WIN, SM, TS>(M, R2, d, s, bases + g, st)) return false;
    return true;
}

// ------------------------------------------------------- FP64 class ----
// The same two phases on the FP64 pipe for odd n < 2^51 (modmath.cuh, ModF):
// plain residues (no Montgomery form) kept as signed lazy representatives
// |x| < n, so 1 is 1.0 or 1 - n and -1 is -1.0 or n - 1.
//
// Base-2 ladder in K-bit windows (round 2).  2^d = prod over the windows of d
// (MSB first) of x <- x^(2^K) * 2^digit, and the factor 2^digit folds into
// the window's last squaring as an exact power-of-two scaling of one factor
// (an exponent-field add, fscale2): fmul_lazy(2^digit x, x).  fmul_lazy's
// bound (modmath.cuh) holds for |a| < 2^e n, |b| < n when e + bitlen(n) <= 51:
// |h / n| < 2^(e + bitlen n) <= 2^51 keeps the rounding addend valid, and
// (h / n) 2^-53 and |l| / n stay <= 2^(e + bitlen n - 53) <= 1/4, so
// |q - ab/n| < 1 and |r| < n.  With digits up to 2^K - 1, K = 4 serves
// bitlen(n) <= 36, K = 3 <= 44, K = 2 <= 48; above, one bit per step as
// before.  Per exponent bit: one product (6 FP64-pipe instructions) and 1/K of
// the window bookkeeping, instead of a product and a scaling every bit.
__device__ __forceinline__ double fscale2(double x, uint32_t e) {
    return __hiloint2double(__double2hiint(x) + (int)(e << 20), __double2loint(x));
}

template <int K>
__device__ __forceinline__ double f2_pow_win(unsigned long long d, const ModF& M) {
    const int nb = 64 - __clzll((long long)d);  // d odd >= 1
    const int nw = (nb + K - 1) / K;
    const uint32_t top = (uint32_t)(d >> (K * (nw - 1)));  // 1 .. 2^K - 1
    double x = __hiloint2double((int)((1023u + top) << 20), 0);  // 2^top, exact
    {  // 2^top may exceed a small n: one exact reduction, |x| <= n / 2 + 1 < n
        const double q = fma(x, M.ninv, FP_RND) - FP_RND;
        x = fma(-q, M.n, x);
    }
#pragma unroll 1
    for (int w = nw - 2; w >= 0; w--) {
        const uint32_t dig = (uint32_t)(d >> (K * w)) & ((1u << K) - 1u);
#pragma unroll
        for (int j = 0; j < K - 1; j++) x = fmul_lazy(x, x, M);
        x = fmul_lazy(fscale2(x, dig), x, M);
    }
    return x;
}

__device__ __forceinline__ bool sprp2_f64(unsigned long long n) {
    const ModF M = modf_setup(n);
    unsigned long long d = n - 1;
    const int s = __ffsll((long long)d) - 1;
    d >>= s;
    const int top = 63 - __clzll((long long)d);
    // signed lazy residues (fmul_lazy): |x| < n throughout, no per-step correction
    double x = 2.0;  // top bit of d
    // window width from the warp's largest n (warp-uniform: no divergence)
    const int bmax = (int)__reduce_max_sync(__activemask(), (unsigned)(64 - __clzll((long long)n)));
    if (bmax <= 36) {
        x = f2_pow_win<4>(d, M);
    } else if (bmax <= 44) {
        x = f2_pow_win<3>(d, M);
    } else if (bmax <= 48) {
        x = f2_pow_win<2>(d, M);
    } else if (top > 0) {
        unsigned long long dd = d << (64 - top);  // remaining bits, MSB first
        if (bmax <= 50) {
            // n < 2^50: the doubling folded into the product (|2x| < 2n is allowed)
            for_bits_msb(dd, top, [&](uint32_t w) { x = fsqr_dbl_lazy(x, w, M); });
        } else {
            // 2^50 <= n < 2^51: square (|x| < n), then double and reduce once
            // (|2y| < 2n, k = round(2y / n) in {-2 .. 2})
            for_bits_msb(dd, top, [&](uint32_t w) { x = fdbl_if_lazy(fmul_lazy(x, x, M), w, M); });
        }
    }
    if (f_is_one(x, M) || f_is_mone(x, M)) return true;
    for (int r = 1; r < s; r++) {
        x = fmul_lazy(x, x, M);
        if (f_is_mone(x, M)) return true;
        if (f_is_one(x, M)) return false;
    }
    return false;
}

template <int T>
__device__ __forceinline__ double sel_table_f(const double (&tab)[T], uint32_t digit) {
    double m = 1.0;
#pragma unroll
    for (int k = 1; k <= T; k++) m = (digit == (uint32_t)k) ? tab[k - 1] : m;
    return m;
}

template <int NB, int WIN, bool SM = false, int TS = 256>
__device__ __forceinline__ bool sprp_lockstep_f64(const ModF& M, unsigned long long n, unsigned long long d, int s,
                                                  const unsigned long long* bases, double* st = nullptr) {
    constexpr int T = (1 << WIN) - 1;
    const int nbits = 64 - __clzll((long long)d);
    const int nw = (nbits + WIN - 1) / WIN;
    double tab[NB][T], x[NB];
    bool done[NB], pass[NB];
#pragma unroll
    for (int i = 0; i < NB; i++) {
        unsigned long long a = bases[i];
        if (a >= n) a %= n;
        done[i] = pass[i] = (a == 0);
        tab[i][0] = (double)a;
#pragma unroll
        for (int k = 1; k < T; k++) tab[i][k] = fmul_lazy(tab[i][k - 1], tab[i][0], M);
        if (SM) {
            st[(i * (T + 1)) * TS] = 1.0;
#pragma unroll
            for (int k = 0; k < T; k++) st[(i * (T + 1) + k + 1) * TS] = tab[i][k];
        }
    }
    {
        const uint32_t lead = (uint32_t)(d >> (WIN * (nw - 1)));
#pragma unroll
        for (int i = 0; i < NB; i++) x[i] = SM ? st[(i * (T + 1) + lead) * TS] : sel_table_f<T>(tab[i], lead);
    }
    for (int w = nw - 2; w >= 0; w--) {
        const uint32_t digit = (uint32_t)(d >> (WIN * w)) & (uint32_t)T;
        double mt[NB];
#pragma unroll
        for (int i = 0; i < NB; i++) mt[i] = SM ? st[(i * (T + 1) + digit) * TS] : sel_table_f<T>(tab[i], digit);
#pragma unroll
        for (int j = 0; j < WIN; j++) {
#pragma unroll
            for (int i = 0; i < NB; i++) x[i] = fmul_lazy(x[i], x[i], M);
        }
#pragma unroll
        for (int i = 0; i < NB; i++) x[i] = fmul_lazy(x[i], mt[i], M);
    }
#pragma unroll
    for (int i = 0; i < NB; i++) {
        if (!done[i] && (f_is_one(x[i], M) || f_is_mone(x[i], M))) done[i] = pass[i] = true;
    }
    for (int r = 1; r < s; r++) {
        bool all = true;
#pragma unroll
        for (int i = 0; i < NB; i++) {
            if (!done[i]) {
                x[i] = fmul_lazy(x[i], x[i], M);
                if (f_is_mone(x[i], M)) done[i] = pass[i] = true;
                else if (f_is_one(x[i], M)) done[i] = true;
            }
            all &= done[i];
        }
        if (all) break;
    }
    bool ok = true;
#pragma unroll
    for (int i = 0; i < NB; i++) ok &= pass[i];
    return ok;
}

template <int NB, int G, int WIN, bool SM = false, int TS = 256>
__device__ __forceinline__ bool sprp_multi_f64(unsigned long long n, const unsigned long long* bases,
                                               double* st = nullptr) {
    const ModF M = modf_setup(n);
    unsigned long long d = n - 1;
    const int s = __ffsll((long long)d) - 1;
    d >>= s;
#pragma unroll 1
    for (int g = 0; g < NB; g += G)
        if (!sprp_lockstep_f64<G, WIN, SM, TS>(M, n, d, s, bases + g, st)) return false;
    return true;
}

// Remaining bases of the 32-bit class ({7, 61}, reading of Eq 4 by magnitude)
// in 2-bit windows whose digit multiply folds into the window's last square
// (round 2): a^dig < 2^18 for a <= 61, dig <= 3, and x a^dig (|x| < n < 2^32)
// is an exact DMUL below 2^50, so fmul_lazy(a^dig x, x) = x^2 a^dig with the
// bound of sprp2_f64's windows (e + bitlen(n) <= 18 + 33 <= 51).  Per two
// exponent bits: two products and one DMUL, instead of two products, a table
// product and a select chain.  tbl (shared memory): NB rows of {1, a, a^2, a^3}.
// Needs n > 61 (every base below n); the caller sends smaller n elsewhere.
constexpr unsigned long long kSmallBaseMinN = 62;
template <int NB>
__device__ __forceinline__ bool sprp_small32_f64(unsigned long long n, const double* tbl) {
    const ModF M = modf_setup(n);
    uint32_t d = (uint32_t)n - 1u;  // n < 2^32
    const int s = __ffs(d) - 1;
    d >>= s;
    const int nb = 32 - __clz(d);
    const int nw = (nb + 1) >> 1;
    const uint32_t top = d >> (2 * (nw - 1));  // 1 .. 3
    double x[NB];
#pragma unroll
    for (int i = 0; i < NB; i++) {
        x[i] = tbl[4 * i + top];  // a^top < 2^18: one exact reduction below n
        const double q = fma(x[i], M.ninv, FP_RND) - FP_RND;
        x[i] = fma(-q, M.n, x[i]);
    }
#pragma unroll 1
    for (int w = nw - 2; w >= 0; w--) {
        const uint32_t dig = (d >> (2 * w)) & 3u;
#pragma unroll
        for (int i = 0; i < NB; i++) {
            const double c = tbl[4 * i + dig];
            x[i] = fmul_lazy(x[i], x[i], M);
            x[i] = fmul_lazy(x[i] * c, x[i], M);
        }
    }
    bool done[NB], pass[NB];
#pragma unroll
    for (int i = 0; i < NB; i++) done[i] = pass[i] = f_is_one(x[i], M) || f_is_mone(x[i], M);
    for (int r = 1; r < s; r++) {
        bool all = true;
#pragma unroll
        for (int i = 0; i < NB; i++) {
            if (!done[i]) {
                x[i] = fmul_lazy(x[i], x[i], M);
                if (f_is_mone(x[i], M)) done[i] = pass[i] = true;
                else if (f_is_one(x[i], M)) done[i] = true;
            }
            all &= done[i];
        }
        if (all) break;
    }
    bool ok = true;
#pragma unroll
    for (int i = 0; i < NB; i++) ok &= pass[i];
    return ok;
}

// Fill tbl[4 i + k] = bases[i]^k (k < 4) -- threads 0 .. 4 NB - 1 of a block.
template <int NB>
__device__ __forceinline__ void small_base_table(double* tbl, const unsigned long long* bases) {
    const int t = threadIdx.x;
    if (t < 4 * NB) {
        const double a = (double)bases[t >> 2];
        double v = 1.0;
        for (int k = 0; k < (t & 3); k++) v *= a;
        tbl[t] = v;
    }
}

// ------------------------------------------------- strong Lucas (BPSW) ----
// The paper's own next step ("a Baillie-PSW test ... could
// replace the Miller-Rabin bases"): a strong base-2 test (phase 1, above)
// followed by a strong Lucas test with Selfridge's parameters is exact for
// every n < 2^64 (no Baillie-PSW pseudoprime exists below 2^64).  Option
// "witness" = 1 runs it instead of the six remaining Eq 4 bases for the
// 64-bit Montgomery class; the default stays the paper's Eq 4 set.

// n is a perfect square (the Selfridge search below never ends for squares).
__device__ __forceinline__ bool is_square64(uint64_t n) {
    uint64_t r = (uint64_t)sqrt((double)n);
    if (r > 0xFFFFFFFFull) r = 0xFFFFFFFFull;
    while (r * r > n) r--;                                    // r < 2^32: r*r is exact
    while (r < 0xFFFFFFFFull && (r + 1) * (r + 1) <= n) r++;
    return r * r == n;
}

// Jacobi symbol (a / m), m odd > 0, a < 2^32 (binary algorithm).
__host__ __device__ constexpr int jacobi32(uint32_t a, uint32_t m) {
    int t = 1;
    a %= m;
    while (a != 0) {
        while (!(a & 1u)) {
            a >>= 1;
            const uint32_t r = m & 7u;
            if (r == 3u || r == 5u) t = -t;
        }
        const uint32_t tmp = a; a = m; m = tmp;
        if ((a & 3u) == 3u && (m & 3u) == 3u) t = -t;
        a %= m;
    }
    return m == 1u ? t : 0;
}

// Residue classes r (mod a) with (r / a) = -1 resp. 0, as bit masks (a < 32).
__host__ __device__ constexpr uint32_t jacobi_mask(uint32_t a, int v) {
    uint32_t m = 0;
    for (uint32_t r = 0; r < a; r++) if (jacobi32(r, a) == v) m |= 1u << r;
    return m;
}

// Jacobi symbol (D / n) for a small odd D (|D| < 2^31) and odd n:
// (D/n) = (-1/n)^[D<0] (|D|/n), and by reciprocity (|D|/n) = (n mod |D| / |D|)
// (-1)^(((|D|-1)/2)((n-1)/2)).
__device__ __forceinline__ int jacobi_small_n64(int D, uint64_t n) {
    const uint32_t a = (uint32_t)(D < 0 ? -D : D);
    int t = jacobi32((uint32_t)(n % a), a);
    if (((a & 3u) == 3u) && ((n & 3ull) == 3ull)) t = -t;
    if (D < 0 && (n & 3ull) == 3ull) t = -t;
    return t;
}

// The same for the K-th Selfridge candidate D_K = (-1)^K (5 + 2K), K < 14,
// with a compile-time modulus (n mod a by multiply-high; the symbol from two
// constant masks): branch-free, so every lane runs the same instructions.
template <int K>
__device__ __forceinline__ int jacobi_selfridge(uint64_t n) {
    constexpr uint32_t a = 5u + 2u * K;
    constexpr uint32_t mneg = jacobi_mask(a, -1), mzero = jacobi_mask(a, 0);
    const uint32_t r = (uint32_t)(n % a);
    int t = ((mzero >> r) & 1u) ? 0 : (((mneg >> r) & 1u) ? -1 : 1);
    const bool n3 = (n & 3ull) == 3ull;
    if ((a & 3u) == 3u && n3) t = -t;  // reciprocity
    if ((K & 1) && n3) t = -t;          // D < 0: (-1/n)
    return t;
}

template <int K>
__device__ __forceinline__ void selfridge_scan(uint64_t n, int& D, bool& comp) {
    if constexpr (K < 12) {
        const int j = jacobi_selfridge<K>(n);
        if (D == 0) {
            if (j == -1) D = (K & 1) ? -(5 + 2 * K) : (5 + 2 * K);
            else if (j == 0) comp = true;  // gcd(|D|, n) > 1 and |D| < n
        }
        selfridge_scan<K + 1>(n, D, comp);
    }
}

// Strong Lucas probable-prime test, Selfridge method A (P = 1, Q = (1 - D)/4,
// D the first of 5, -7, 9, -11, ... with (D/n) = -1), for odd n >= 2^32 in
// Montgomery form.  n + 1 = d 2^s; passes iff U_d == 0 or V_{d 2^r} == 0 for
// some 0 <= r < s.  V_k, V_{k+1} by a ladder over the bits of d (V_2k = V_k^2 -
// 2Q^k, V_2k+1 = V_k V_k+1 - P Q^k), Q^k alongside; U_d == 0 is tested as
// 2 V_{d+1} == P V_d (D U_k = 2 V_{k+1} - P V_k, gcd(D, n) = 1).  4 modular
// multiplications per bit against ~9 per bit for six Miller-Rabin bases.
// No early return before the ladder: lanes that diverged in a parameter search
// would otherwise run the ladder in separate passes.
__device__ __forceinline__ bool slprp64(uint64_t n, const Mont64& M, uint64_t R2) {
    bool comp = n == ~0ull || is_square64(n);  // 2^64 - 1 = 3 * 5 * 17 * ...
    int D = 0;
    selfridge_scan<0>(n, D, comp);             // the first 12 candidates, branch-free
    if (D == 0 && !comp) {                     // rare (< 2^-12 of non-squares): continue the sequence
        D = 29;
        for (;;) {
            const int j = jacobi_small_n64(D, n);
            if (j == -1) break;
            if (j == 0) { comp = true; break; }
            D = D > 0 ? -(D + 2) : -D + 2;
            if (D > 100000 || D < -100000) { comp = true; break; }  // not reached for non-squares
        }
    }
    if (comp) D = 5;                           // the ladder still runs (uniform); its result is ignored
    const long long Q = (1 - (long long)D) / 4;
    const uint64_t Qmod = Q < 0 ? n - (uint64_t)(-Q) : (uint64_t)Q;
    const uint64_t Qm = mmul64(Qmod, R2, M);                 // mont(Q)
    uint64_t d = n + 1;                                       // n < 2^64 - 1 here (or comp)
    const int s = d ? __ffsll((long long)d) - 1 : 1;
    d = d ? d >> s : 1;
    // ladder state for k = 1: V_1 = P = 1, V_2 = P^2 - 2Q, Q^1 = Q
    const uint64_t one = M.one;
    uint64_t Vk = one;
    uint64_t Vk1 = msub64(one, madd64(Qm, Qm, n), n);
    uint64_t Qk = Qm;
    const int top = 63 - __clzll((long long)d);
    if (top > 0) {
        uint64_t dd = d << (64 - top);                        // bits below the leading one, MSB first
        for (int k = 0; k < top; k++) {
            const bool b = (long long)dd < 0;
            dd += dd;
            const uint64_t Qk1 = mmul64_ptx(Qk, Qm, n, M.ninv);                 // Q^{k+1}
            const uint64_t cross = msub64(mmul64_ptx(Vk, Vk1, n, M.ninv), Qk, n);  // V_{2k+1} = V_k V_{k+1} - Q^k
            const uint64_t vs = b ? Vk1 : Vk;
            const uint64_t qs = b ? Qk1 : Qk;
            const uint64_t sq = msub64(msqr64_ptx(vs, n, M.ninv), madd64(qs, qs, n), n);  // V_{2j} = V_j^2 - 2Q^j
            Vk = b ? cross : sq;
            Vk1 = b ? sq : cross;
            Qk = mmul64_ptx(Qk, qs, n, M.ninv);               // Q^{2k} or Q^{2k+1}
        }
    }
    // U_d == 0  <=>  2 V_{d+1} == V_d  (P = 1)
    bool pass = madd64(Vk1, Vk1, n) == Vk || Vk == 0;
    for (int r = 1; r < s && !pass; r++) {
        Vk = msub64(msqr64_ptx(Vk, n, M.ninv), madd64(Qk, Qk, n), n);   // V_{2j} = V_j^2 - 2Q^j
        pass = Vk == 0;
        Qk = msqr64_ptx(Qk, n, M.ninv);
    }
    return pass && !comp;
}

__device__ __forceinline__ bool slprp64(uint64_t n) {
    const Mont64 M = mont64_setup(n);
    return slprp64(n, M, mont64_r2(M));
}

}  // namespace isp
