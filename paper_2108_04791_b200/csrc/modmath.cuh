// modmath.cuh -- device modular arithmetic for the Miller-Rabin witness
// kernels (layer L0).  sm_100a, integer pipes only (IMAD / IMAD.WIDE /
// IMAD.HI on the FMA-heavy pipe, IADD3 / ISETP / SEL on the ALU pipe).
//
// The paper needs a*b mod m for 64-bit operands without 128-bit integers and
// builds it from ModAdd (Property 1: c = a - (m - b)),
// ModMultiply and ModExp.  On sm_100a the
// hardware gives the high half of a 64x64 product (mul.hi.u64), so the
// saturation-avoiding MATLAB cases are replaced by Montgomery multiplication
// with R = 2^64 (or 2^32 for moduli below 2^32).  What survives from the paper:
//   * ModAdd's Property 1 is the conditional subtraction at the tail of every
//     reduction and the whole of mod_dbl (ModMultiply case 3, a = 2,
//     "c = b - (m - b)"), which is how the base-2 ladder
//     multiplies by its base with no multiply at all;
//   * ModExp is left-to-right exponentiation by squaring over the bits of d.
//
// Reduction used ("subtraction REDC"): for T = a*b < n*R, m = lo(T) * n^-1 mod
// R makes lo(m*n) == lo(T), so T - m*n = (hi(T) - hi(m*n)) * R exactly and
// REDC(T) = hi(T) - hi(m*n) (+ n on borrow) lies in [0, n).  It never needs a
// 65th bit, so it is valid for every odd n < 2^64, including n > 2^63.
#pragma once
#include <stdint.h>

namespace isp {

// ---------------------------------------------------------------- 32-bit ----
struct Mont32 {
    uint32_t n;     // odd modulus, 3 <= n < 2^32
    uint32_t ninv;  // n^-1 mod 2^32
    uint32_t one;   // R mod n  (Montgomery form of 1)
    uint32_t mone;  // n - one  (Montgomery form of n-1, i.e. -1)
};

__device__ __forceinline__ uint32_t inv32(uint32_t n) {
    uint32_t x = (n * 3u) ^ 2u;  // correct to 5 bits for odd n
    x *= 2u - n * x;             // 10
    x *= 2u - n * x;             // 20
    x *= 2u - n * x;             // 40 >= 32
    return x;
}

__device__ __forceinline__ uint32_t redc32(uint64_t T, uint32_t n, uint32_t ninv) {
    uint32_t lo = (uint32_t)T, hi = (uint32_t)(T >> 32);
    uint32_t m = lo * ninv;
    uint32_t mh = __umulhi(m, n);
    uint32_t t = hi - mh;
    return hi < mh ? t + n : t;
}

__device__ __forceinline__ uint32_t mmul32(uint32_t a, uint32_t b, const Mont32& M) {
    return redc32((uint64_t)a * b, M.n, M.ninv);
}

// ModAdd for a, b < n < 2^32, no overflow: 64-bit-free via
// Property 1 (a - (n - b)) when a >= n - b.
__device__ __forceinline__ uint32_t madd32(uint32_t a, uint32_t b, uint32_t n) {
    uint32_t nb = n - b;
    return a >= nb ? a - nb : a + b;
}

__device__ __forceinline__ Mont32 mont32_setup(uint32_t n) {
    Mont32 M;
    M.n = n;
    M.ninv = inv32(n);
    M.one = (0u - n) % n;  // 2^32 mod n
    M.mone = n - M.one;
    return M;
}

// Montgomery form of a (a < n): a * R mod n = REDC(a * R^2 mod n).
// R^2 mod n = Montgomery form of 2^32: start from mont(2^8) = 2^8 R mod n by 8
// modular doublings of R mod n, then square twice (2^16, 2^32).
__device__ __forceinline__ uint32_t mont32_r2(const Mont32& M) {
    uint32_t x = M.one;
#pragma unroll
    for (int i = 0; i < 8; i++) x = madd32(x, x, M.n);
    x = mmul32(x, x, M);
    x = mmul32(x, x, M);
    return x;
}

// ---------------------------------------------------------------- 64-bit ----
struct Mont64 {
    uint64_t n;     // odd modulus, 3 <= n < 2^64
    uint64_t ninv;  // n^-1 mod 2^64
    uint64_t one;   // R mod n
    uint64_t mone;  // n - one
};

__device__ __forceinline__ uint64_t inv64(uint64_t n) {
    uint32_t x32 = inv32((uint32_t)n);     // n^-1 mod 2^32
    uint64_t x = x32;
    x *= 2ull - n * x;                     // 64 bits
    return x;
}

__device__ __forceinline__ uint64_t redc64(uint64_t lo, uint64_t hi, uint64_t n, uint64_t ninv) {
    uint64_t m = lo * ninv;
    uint64_t mh = __umul64hi(m, n);
    uint64_t t = hi - mh;
    return hi < mh ? t + n : t;
}

__device__ __forceinline__ uint64_t mmul64(uint64_t a, uint64_t b, const Mont64& M) {
    return redc64(a * b, __umul64hi(a, b), M.n, M.ninv);
}

__device__ __forceinline__ uint64_t msqr64(uint64_t a, const Mont64& M) {
    return redc64(a * a, __umul64hi(a, a), M.n, M.ninv);
}

// ModAdd, Property 1: a + b mod n = a - (n - b) when a >= n - b.
__device__ __forceinline__ uint64_t madd64(uint64_t a, uint64_t b, uint64_t n) {
    uint64_t nb = n - b;
    return a >= nb ? a - nb : a + b;
}

// ModMultiply case 3: 2b mod n = b - (n - b).
__device__ __forceinline__ uint64_t mdbl64(uint64_t b, uint64_t n) { return madd64(b, b, n); }

__device__ __forceinline__ int bitlen64(uint64_t v) { return 64 - __clzll((long long)v); }

// R mod n without a 128-bit division: with L = bitlen(n), 2^(L-1) < n (n odd,
// L >= 2), so 2^L mod n = 2^L - n; double it (64 - L) more times.
__device__ __forceinline__ uint64_t r_mod_n64(uint64_t n) {
    int L = bitlen64(n);
    uint64_t x = (L == 64) ? (0ull - n) : ((1ull << L) - n);
    for (int i = L; i < 64; i++) x = mdbl64(x, n);
    return x;
}

__device__ __forceinline__ Mont64 mont64_setup(uint64_t n) {
    Mont64 M;
    M.n = n;
    M.ninv = inv64(n);
    M.one = r_mod_n64(n);
    M.mone = n - M.one;
    return M;
}

// R^2 mod n = Montgomery form of 2^64: mont(2^8) by 8 doublings of R mod n,
// then three Montgomery squarings (2^16, 2^32, 2^64).
__device__ __forceinline__ uint64_t mont64_r2(const Mont64& M) {
    uint64_t x = M.one;
#pragma unroll
    for (int i = 0; i < 8; i++) x = mdbl64(x, M.n);
    x = msqr64(x, M);
    x = msqr64(x, M);
    x = msqr64(x, M);
    return x;
}

}  // namespace isp
