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

// Subtraction REDC from the 128-bit product (lo, hi).  Written with
// mul.lo.u64 / mul.hi.u64: ptxas expands them into IMAD.WIDE.U32 chains that
// measured faster on B200 than a hand-written 32-bit-limb C++ version
// (profiles/r1_mr_step.json: 6.6e11 vs 6.1e11 squarings/s).
__device__ __forceinline__ uint64_t redc64(uint64_t lo, uint64_t hi, uint64_t n, uint64_t ninv) {
    const uint64_t m = lo * ninv;
    const uint64_t mh = __umul64hi(m, n);
    const uint64_t t = hi - mh;
    return hi < mh ? t + n : t;
}

// General Montgomery product in the same PTX style: four mul.wide for a*b.
__device__ __forceinline__ uint64_t mmul64_ptx(uint64_t a, uint64_t b, uint64_t n, uint64_t ninv) {
    uint64_t r;
    asm("{\n\t"
        ".reg .u32 a0, a1, b0, b1, n0, n1, i0, i1, p0, p1, c0, c1, e0, e1, h0, h1, t1, t2, t3, m0, m1;\n\t"
        ".reg .u32 q0, q1, f0, f1, g0, g1, d0, d1, u2, u3, r0, r1, bw, k0, k1;\n\t"
        ".reg .u64 W;\n\t"
        "mov.b64 {a0, a1}, %1;\n\t"
        "mov.b64 {b0, b1}, %2;\n\t"
        "mov.b64 {n0, n1}, %3;\n\t"
        "mov.b64 {i0, i1}, %4;\n\t"
        "mul.wide.u32 W, a0, b0;\n\t"
        "mov.b64 {p0, p1}, W;\n\t"
        "mul.wide.u32 W, a0, b1;\n\t"
        "mov.b64 {c0, c1}, W;\n\t"
        "mul.wide.u32 W, a1, b0;\n\t"
        "mov.b64 {e0, e1}, W;\n\t"
        "mul.wide.u32 W, a1, b1;\n\t"
        "mov.b64 {h0, h1}, W;\n\t"
        "add.cc.u32 t1, p1, c0;\n\t"
        "addc.cc.u32 t2, h0, c1;\n\t"
        "addc.u32 t3, h1, 0;\n\t"
        "add.cc.u32 t1, t1, e0;\n\t"
        "addc.cc.u32 t2, t2, e1;\n\t"
        "addc.u32 t3, t3, 0;\n\t"
        "mul.wide.u32 W, p0, i0;\n\t"
        "mov.b64 {m0, m1}, W;\n\t"
        "mad.lo.u32 m1, p0, i1, m1;\n\t"
        "mad.lo.u32 m1, t1, i0, m1;\n\t"
        "mul.wide.u32 W, m0, n0;\n\t"
        "mov.b64 {q0, q1}, W;\n\t"
        "mul.wide.u32 W, m0, n1;\n\t"
        "mov.b64 {f0, f1}, W;\n\t"
        "mul.wide.u32 W, m1, n0;\n\t"
        "mov.b64 {g0, g1}, W;\n\t"
        "mul.wide.u32 W, m1, n1;\n\t"
        "mov.b64 {d0, d1}, W;\n\t"
        "add.cc.u32 q1, q1, f0;\n\t"
        "addc.cc.u32 u2, d0, f1;\n\t"
        "addc.u32 u3, d1, 0;\n\t"
        "add.cc.u32 q1, q1, g0;\n\t"
        "addc.cc.u32 u2, u2, g1;\n\t"
        "addc.u32 u3, u3, 0;\n\t"
        "sub.cc.u32 r0, t2, u2;\n\t"
        "subc.cc.u32 r1, t3, u3;\n\t"
        "subc.u32 bw, 0, 0;\n\t"
        "and.b32 k0, n0, bw;\n\t"
        "and.b32 k1, n1, bw;\n\t"
        "add.cc.u32 r0, r0, k0;\n\t"
        "addc.u32 r1, r1, k1;\n\t"
        "mov.b64 %0, {r0, r1};\n\t"
        "}"
        : "=l"(r)
        : "l"(a), "l"(b), "l"(n), "l"(ninv));
    return r;
}

__device__ __forceinline__ uint64_t mmul64(uint64_t a, uint64_t b, const Mont64& M) {
    return redc64(a * b, __umul64hi(a, b), M.n, M.ninv);
}

__device__ __forceinline__ uint64_t msqr64(uint64_t a, const Mont64& M) {
    return redc64(a * a, __umul64hi(a, a), M.n, M.ninv);
}

// Montgomery squaring written as one PTX block with explicit carry chains
// (add.cc / addc): three mul.wide for x^2 (the cross term added twice instead
// of doubled with shifts), one mul.wide + two mad.lo for m, four mul.wide for
// hi(m*n).  Alone it is as fast as msqr64; followed by the base-2 ladder's
// conditional doubling it is 5% faster (profiles/r1_mr_step.json), so the
// base-2 phase uses it.
__device__ __forceinline__ uint64_t msqr64_ptx(uint64_t x, uint64_t n, uint64_t ninv) {
    uint64_t r;
    asm("{\n\t"
        ".reg .u32 x0, x1, n0, n1, i0, i1, p0, p1, c0, c1, h0, h1, t1, t2, t3, m0, m1;\n\t"
        ".reg .u32 q0, q1, a0, a1, b0, b1, d0, d1, u2, u3, r0, r1, bw, k0, k1;\n\t"
        ".reg .u64 W;\n\t"
        "mov.b64 {x0, x1}, %1;\n\t"
        "mov.b64 {n0, n1}, %2;\n\t"
        "mov.b64 {i0, i1}, %3;\n\t"
        // T = x^2 = (t3 t2 t1 p0)
        "mul.wide.u32 W, x0, x0;\n\t"
        "mov.b64 {p0, p1}, W;\n\t"
        "mul.wide.u32 W, x0, x1;\n\t"
        "mov.b64 {c0, c1}, W;\n\t"
        "mul.wide.u32 W, x1, x1;\n\t"
        "mov.b64 {h0, h1}, W;\n\t"
        "add.cc.u32 t1, p1, c0;\n\t"
        "addc.cc.u32 t2, h0, c1;\n\t"
        "addc.u32 t3, h1, 0;\n\t"
        "add.cc.u32 t1, t1, c0;\n\t"
        "addc.cc.u32 t2, t2, c1;\n\t"
        "addc.u32 t3, t3, 0;\n\t"
        // m = (t1 p0) * ninv mod 2^64
        "mul.wide.u32 W, p0, i0;\n\t"
        "mov.b64 {m0, m1}, W;\n\t"
        "mad.lo.u32 m1, p0, i1, m1;\n\t"
        "mad.lo.u32 m1, t1, i0, m1;\n\t"
        // hi(m*n) = (u3 u2): columns of m0n0, m0n1, m1n0, m1n1
        "mul.wide.u32 W, m0, n0;\n\t"
        "mov.b64 {q0, q1}, W;\n\t"
        "mul.wide.u32 W, m0, n1;\n\t"
        "mov.b64 {a0, a1}, W;\n\t"
        "mul.wide.u32 W, m1, n0;\n\t"
        "mov.b64 {b0, b1}, W;\n\t"
        "mul.wide.u32 W, m1, n1;\n\t"
        "mov.b64 {d0, d1}, W;\n\t"
        "add.cc.u32 q1, q1, a0;\n\t"
        "addc.cc.u32 u2, d0, a1;\n\t"
        "addc.u32 u3, d1, 0;\n\t"
        "add.cc.u32 q1, q1, b0;\n\t"
        "addc.cc.u32 u2, u2, b1;\n\t"
        "addc.u32 u3, u3, 0;\n\t"
        // r = (t3 t2) - (u3 u2), + n on borrow
        "sub.cc.u32 r0, t2, u2;\n\t"
        "subc.cc.u32 r1, t3, u3;\n\t"
        "subc.u32 bw, 0, 0;\n\t"
        "and.b32 k0, n0, bw;\n\t"
        "and.b32 k1, n1, bw;\n\t"
        "add.cc.u32 r0, r0, k0;\n\t"
        "addc.u32 r1, r1, k1;\n\t"
        "mov.b64 %0, {r0, r1};\n\t"
        "}"
        : "=l"(r)
        : "l"(x), "l"(n), "l"(ninv));
    return r;
}

// One step of the base-2 ladder, x <- x^2 * 2^b (b in {0, 1}), as a single
// reduction: REDC(x^2 << b).  ModMultiply case 3 (the
// multiplication by a = 2) becomes a one-bit funnel shift of the 128-bit
// square instead of a separate modular doubling.  Valid for n < 2^63: then
// x^2 * 2 < 2 n^2 < n R, so the subtraction REDC still lands in (-n, n) and
// needs the single "+ n on borrow" correction.  sm_100a: 8 IMAD.WIDE + 2 IMAD
// on the FMA-heavy pipe; the shift is 4 SHF on the ALU pipe, replacing the
// ~10 ALU instructions of compare / subtract / select of a modular doubling.
__device__ __forceinline__ uint64_t msqr64_shl_ptx(uint64_t x, uint64_t n, uint64_t ninv, uint32_t b) {
    uint64_t r;
    asm("{\n\t"
        ".reg .u32 x0, x1, n0, n1, i0, i1, p0, p1, c0, c1, h0, h1, t1, t2, t3, m0, m1;\n\t"
        ".reg .u32 q0, q1, a0, a1, b0, b1, d0, d1, u2, u3, r0, r1, bw, k0, k1;\n\t"
        ".reg .u64 W;\n\t"
        "mov.b64 {x0, x1}, %1;\n\t"
        "mov.b64 {n0, n1}, %2;\n\t"
        "mov.b64 {i0, i1}, %3;\n\t"
        "mul.wide.u32 W, x0, x0;\n\t"
        "mov.b64 {p0, p1}, W;\n\t"
        "mul.wide.u32 W, x0, x1;\n\t"
        "mov.b64 {c0, c1}, W;\n\t"
        "mul.wide.u32 W, x1, x1;\n\t"
        "mov.b64 {h0, h1}, W;\n\t"
        "add.cc.u32 t1, p1, c0;\n\t"
        "addc.cc.u32 t2, h0, c1;\n\t"
        "addc.u32 t3, h1, 0;\n\t"
        "add.cc.u32 t1, t1, c0;\n\t"
        "addc.cc.u32 t2, t2, c1;\n\t"
        "addc.u32 t3, t3, 0;\n\t"
        // T <<= b  (T < 2^127 because x < n < 2^63)
        "shf.l.clamp.b32 t3, t2, t3, %4;\n\t"
        "shf.l.clamp.b32 t2, t1, t2, %4;\n\t"
        "shf.l.clamp.b32 t1, p0, t1, %4;\n\t"
        "shl.b32 p0, p0, %4;\n\t"
        "mul.wide.u32 W, p0, i0;\n\t"
        "mov.b64 {m0, m1}, W;\n\t"
        "mad.lo.u32 m1, p0, i1, m1;\n\t"
        "mad.lo.u32 m1, t1, i0, m1;\n\t"
        "mul.wide.u32 W, m0, n0;\n\t"
        "mov.b64 {q0, q1}, W;\n\t"
        "mul.wide.u32 W, m0, n1;\n\t"
        "mov.b64 {a0, a1}, W;\n\t"
        "mul.wide.u32 W, m1, n0;\n\t"
        "mov.b64 {b0, b1}, W;\n\t"
        "mul.wide.u32 W, m1, n1;\n\t"
        "mov.b64 {d0, d1}, W;\n\t"
        "add.cc.u32 q1, q1, a0;\n\t"
        "addc.cc.u32 u2, d0, a1;\n\t"
        "addc.u32 u3, d1, 0;\n\t"
        "add.cc.u32 q1, q1, b0;\n\t"
        "addc.cc.u32 u2, u2, b1;\n\t"
        "addc.u32 u3, u3, 0;\n\t"
        "sub.cc.u32 r0, t2, u2;\n\t"
        "subc.cc.u32 r1, t3, u3;\n\t"
        "subc.u32 bw, 0, 0;\n\t"
        "and.b32 k0, n0, bw;\n\t"
        "and.b32 k1, n1, bw;\n\t"
        "add.cc.u32 r0, r0, k0;\n\t"
        "addc.u32 r1, r1, k1;\n\t"
        "mov.b64 %0, {r0, r1};\n\t"
        "}"
        : "=l"(r)
        : "l"(x), "l"(n), "l"(ninv), "r"(b));
    return r;
}

// Conditional modular doubling x <- b ? 2x mod n : x for any odd n < 2^64
// (ModAdd Property 1 with a = b = x, as one carry chain): s = x +
// (x & -b) with carry, t = s - n with borrow; t is the answer unless the sum
// did not carry and t borrowed (then s < n).
__device__ __forceinline__ uint64_t mdbl64_if_ptx(uint64_t x, uint64_t n, uint32_t b) {
    uint64_t r;
    asm("{\n\t"
        ".reg .u32 x0, x1, n0, n1, mk, a0, a1, s0, s1, t0, t1, c, k0, k1;\n\t"
        "mov.b64 {x0, x1}, %1;\n\t"
        "mov.b64 {n0, n1}, %2;\n\t"
        "neg.s32 mk, %3;\n\t"
        "and.b32 a0, x0, mk;\n\t"
        "and.b32 a1, x1, mk;\n\t"
        "add.cc.u32 s0, x0, a0;\n\t"
        "addc.cc.u32 s1, x1, a1;\n\t"
        "addc.u32 c, 0, 0;\n\t"
        "sub.cc.u32 t0, s0, n0;\n\t"
        "subc.cc.u32 t1, s1, n1;\n\t"
        "subc.u32 c, c, 0;\n\t"          // carry - borrow: 0 -> t, -1 -> s (+1 cannot occur)
        "and.b32 k0, n0, c;\n\t"
        "and.b32 k1, n1, c;\n\t"
        "add.cc.u32 t0, t0, k0;\n\t"
        "addc.u32 t1, t1, k1;\n\t"
        "mov.b64 %0, {t0, t1};\n\t"
        "}"
        : "=l"(r)
        : "l"(x), "l"(n), "r"(b));
    return r;
}

// ---- lazy additive REDC (n < 2^62) ----------------------------------------
// With nn = -n^-1 mod 2^64 and m = T mod 2^64 * nn mod 2^64, T + m n is a
// multiple of R = 2^64 and (T + m n) / R == T R^-1 (mod n).  For inputs below
// 2n and n < R / 4, T < 4 n^2 and (T + m n) / R < 4 n^2 / R + n < 2n: the
// result is again below 2n with no final correction, so a ladder keeps lazy
// representatives in [0, 2n) and reduces once (mcanon64) before comparing.
// The column sum is three carry chains (T + m0n0 + m1n1, + m0n1, + m1n0):
// 10 ALU operations against 13 for the subtraction form's sum, borrow and
// conditional add.  Same 8 IMAD.WIDE + 2 IMAD on the FMA-heavy pipe.
#define ISP_LZ_REDC_SUM                                  \
    "mul.wide.u32 W, p0, i0;\n\t"                        \
    "mov.b64 {m0, m1}, W;\n\t"                           \
    "mad.lo.u32 m1, p0, i1, m1;\n\t"                     \
    "mad.lo.u32 m1, t1, i0, m1;\n\t"                     \
    "mul.wide.u32 W, m0, n0;\n\t"                        \
    "mov.b64 {q0, q1}, W;\n\t"                           \
    "mul.wide.u32 W, m0, n1;\n\t"                        \
    "mov.b64 {a0, a1}, W;\n\t"                           \
    "mul.wide.u32 W, m1, n0;\n\t"                        \
    "mov.b64 {b0, b1}, W;\n\t"                           \
    "mul.wide.u32 W, m1, n1;\n\t"                        \
    "mov.b64 {d0, d1}, W;\n\t"                           \
    "add.cc.u32 z, p0, q0;\n\t"                          \
    "addc.cc.u32 z, t1, q1;\n\t"                         \
    "addc.cc.u32 r0, t2, d0;\n\t"                        \
    "addc.u32 r1, t3, d1;\n\t"                           \
    "add.cc.u32 z, z, a0;\n\t"                           \
    "addc.cc.u32 r0, r0, a1;\n\t"                        \
    "addc.u32 r1, r1, 0;\n\t"                            \
    "add.cc.u32 z, z, b0;\n\t"                           \
    "addc.cc.u32 r0, r0, b1;\n\t"                        \
    "addc.u32 r1, r1, 0;\n\t"                            \
    "mov.b64 %0, {r0, r1};\n\t"

#define ISP_LZ_REGS                                                                  \
    ".reg .u32 x0, x1, n0, n1, i0, i1, p0, p1, c0, c1, h0, h1, t1, t2, t3, m0, m1;\n\t" \
    ".reg .u32 q0, q1, a0, a1, b0, b1, d0, d1, r0, r1, z;\n\t"                         \
    ".reg .u64 W;\n\t"

// x^2 R^-1 mod n, lazily: x < 2n, n < 2^62 -> result < 2n.  nn = -n^-1 mod 2^64.
__device__ __forceinline__ uint64_t msqr64_lz_ptx(uint64_t x, uint64_t n, uint64_t nn) {
    uint64_t r;
    asm("{\n\t" ISP_LZ_REGS
        "mov.b64 {x0, x1}, %1;\n\t"
        "mov.b64 {n0, n1}, %2;\n\t"
        "mov.b64 {i0, i1}, %3;\n\t"
        "mul.wide.u32 W, x0, x0;\n\t"
        "mov.b64 {p0, p1}, W;\n\t"
        "mul.wide.u32 W, x0, x1;\n\t"
        "mov.b64 {c0, c1}, W;\n\t"
        "mul.wide.u32 W, x1, x1;\n\t"
        "mov.b64 {h0, h1}, W;\n\t"
        "add.cc.u32 t1, p1, c0;\n\t"
        "addc.cc.u32 t2, h0, c1;\n\t"
        "addc.u32 t3, h1, 0;\n\t"
        "add.cc.u32 t1, t1, c0;\n\t"
        "addc.cc.u32 t2, t2, c1;\n\t"
        "addc.u32 t3, t3, 0;\n\t"
        ISP_LZ_REDC_SUM
        "}"
        : "=l"(r)
        : "l"(x), "l"(n), "l"(nn));
    return r;
}

// x^2 2^b R^-1 mod n, lazily (b in {0, 1}): x < 2n, n <= 2^61 -> result < 2n
// (T = 2 x^2 < 8 n^2 <= n R).  The base-2 ladder step of msqr64_shl_ptx
// without its final correction.
__device__ __forceinline__ uint64_t msqr64_shl_lz_ptx(uint64_t x, uint64_t n, uint64_t nn, uint32_t b) {
    uint64_t r;
    asm("{\n\t" ISP_LZ_REGS
        "mov.b64 {x0, x1}, %1;\n\t"
        "mov.b64 {n0, n1}, %2;\n\t"
        "mov.b64 {i0, i1}, %3;\n\t"
        "mul.wide.u32 W, x0, x0;\n\t"
        "mov.b64 {p0, p1}, W;\n\t"
        "mul.wide.u32 W, x0, x1;\n\t"
        "mov.b64 {c0, c1}, W;\n\t"
        "mul.wide.u32 W, x1, x1;\n\t"
        "mov.b64 {h0, h1}, W;\n\t"
        "add.cc.u32 t1, p1, c0;\n\t"
        "addc.cc.u32 t2, h0, c1;\n\t"
        "addc.u32 t3, h1, 0;\n\t"
        "add.cc.u32 t1, t1, c0;\n\t"
        "addc.cc.u32 t2, t2, c1;\n\t"
        "addc.u32 t3, t3, 0;\n\t"
        "shf.l.clamp.b32 t3, t2, t3, %4;\n\t"
        "shf.l.clamp.b32 t2, t1, t2, %4;\n\t"
        "shf.l.clamp.b32 t1, p0, t1, %4;\n\t"
        "shl.b32 p0, p0, %4;\n\t"
        ISP_LZ_REDC_SUM
        "}"
        : "=l"(r)
        : "l"(x), "l"(n), "l"(nn), "r"(b));
    return r;
}

// a b R^-1 mod n, lazily: a, b < 2n, n < 2^62 -> result < 2n.
__device__ __forceinline__ uint64_t mmul64_lz_ptx(uint64_t a, uint64_t b, uint64_t n, uint64_t nn) {
    uint64_t r;
    asm("{\n\t" ISP_LZ_REGS
        ".reg .u32 y0, y1, e0, e1;\n\t"
        "mov.b64 {x0, x1}, %1;\n\t"
        "mov.b64 {y0, y1}, %2;\n\t"
        "mov.b64 {n0, n1}, %3;\n\t"
        "mov.b64 {i0, i1}, %4;\n\t"
        "mul.wide.u32 W, x0, y0;\n\t"
        "mov.b64 {p0, p1}, W;\n\t"
        "mul.wide.u32 W, x0, y1;\n\t"
        "mov.b64 {c0, c1}, W;\n\t"
        "mul.wide.u32 W, x1, y0;\n\t"
        "mov.b64 {e0, e1}, W;\n\t"
        "mul.wide.u32 W, x1, y1;\n\t"
        "mov.b64 {h0, h1}, W;\n\t"
        "add.cc.u32 t1, p1, c0;\n\t"
        "addc.cc.u32 t2, h0, c1;\n\t"
        "addc.u32 t3, h1, 0;\n\t"
        "add.cc.u32 t1, t1, e0;\n\t"
        "addc.cc.u32 t2, t2, e1;\n\t"
        "addc.u32 t3, t3, 0;\n\t"
        ISP_LZ_REDC_SUM
        "}"
        : "=l"(r)
        : "l"(a), "l"(b), "l"(n), "l"(nn));
    return r;
}
#undef ISP_LZ_REDC_SUM
#undef ISP_LZ_REGS

// The canonical representative of a lazy x < 2n.
__device__ __forceinline__ uint64_t mcanon64(uint64_t x, uint64_t n) { return x >= n ? x - n : x; }

// ModAdd, Property 1: a + b mod n = a - (n - b) when a >= n - b.
__device__ __forceinline__ uint64_t madd64(uint64_t a, uint64_t b, uint64_t n) {
    uint64_t nb = n - b;
    return a >= nb ? a - nb : a + b;
}

// a - b mod n for a, b < n.
__device__ __forceinline__ uint64_t msub64(uint64_t a, uint64_t b, uint64_t n) {
    return a >= b ? a - b : a + (n - b);
}

// ModMultiply case 3: 2b mod n = b - (n - b).
__device__ __forceinline__ uint64_t mdbl64(uint64_t b, uint64_t n) { return madd64(b, b, n); }

__device__ __forceinline__ int bitlen64(uint64_t v) { return 64 - __clzll((long long)v); }

// R mod n without a 128-bit division: with L = bitlen(n), 2^(L-1) < n (n odd,
// L >= 2), so 2^L mod n = 2^L - n; double it (64 - L) more times.
// For 2^39 <= n < 2^60 (the Montgomery class starts at 2^51) the quotient is
// estimated in double instead: q = trunc(2^64 / n) < 2^25 is within 1 of
// floor(2^64 / n) (relative error ~2^-52), so with q - 1 the remainder
// 2^64 - (q - 1) n lies in [0, 3n) and two conditional subtractions finish it
// -- about 15 instructions instead of up to 25 doublings.
__device__ __forceinline__ uint64_t r_mod_n64(uint64_t n) {
    int L = bitlen64(n);
    if (L >= 40 && L <= 60) {
        const unsigned long long q = (unsigned long long)(18446744073709551616.0 / (double)n) - 1ull;
        uint64_t r = 0ull - q * n;  // 2^64 - q n, in [0, 3n)
        if (r >= n) r -= n;
        if (r >= n) r -= n;
        return r;
    }
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
    x = msqr64_ptx(x, M.n, M.ninv);
    x = msqr64_ptx(x, M.n, M.ninv);
    x = msqr64_ptx(x, M.n, M.ninv);
    return x;
}

// ------------------------------------------------------- FP64, n < 2^51 ----
// The paper's medium class (2^18 .. 2^49) is the range where
// double precision is exact -- and on B200 the FP64 pipe issues 64 DFMA
// lanes/clk/SM (profiles/r1_imad_peak.json: 63.1) against 25 for the
// IMAD.WIDE.U32 that 64-bit Montgomery needs.  For odd n < 2^51 and a, b < n:
//   h = fl(ab), l = fma(a, b, -h) = ab - h exactly (|l| <= 2^48),
//   q = nearest integer to fl(h * fl(1/n)): |q - ab/n| < 1/2 + 1/4 + 1/4,
//   r = fma(-q, n, h) + l = ab - qn exactly, in (-n, n),
// and one conditional +n gives ab mod n.  Rounding to an integer uses the
// 1.5 * 2^52 addend (valid for |x| < 2^51).  (The paper's class boundary is
// 2^49; the arithmetic's is 2^51, so the 50- and 51-bit values join the FP64
// class.)
constexpr double FP_RND = 6755399441055744.0;  // 1.5 * 2^52
// The FP64 class: odd n < 2^FP_BITS (fmul_lazy's bound below holds to 2^51
// for products of factors below n, to 2^50 with one factor doubled).
constexpr int FP_BITS = 51;
constexpr unsigned long long FP_LIMIT = 1ull << FP_BITS;

struct ModF {
    double n, ninv, nm1;  // n, fl(1/n), n - 1
};

__device__ __forceinline__ ModF modf_setup(unsigned long long n) {
    ModF M;
    M.n = (double)n;
    M.ninv = 1.0 / M.n;
    M.nm1 = M.n - 1.0;
    return M;
}

__device__ __forceinline__ double fmulmod(double a, double b, const ModF& M) {
    const double h = a * b;
    const double l = fma(a, b, -h);
    const double q = __dadd_rn(__dmul_rn(h, M.ninv), FP_RND) - FP_RND;
    const double r = fma(-q, M.n, h) + l;
    return r < 0.0 ? r + M.n : r;
}

// Lazy signed product for the witness loops: a, b exact integers with |a| <
// 2n, |b| < n, n < 2^50 -- or |a|, |b| < n, n < 2^51 (the same three bounds
// below: |h / n| < n < 2^51, |l| <= 2^48, so |l| / n and (h/n) 2^-53 stay
// below 1/4).  Returns the signed representative r == a*b (mod n)
// with |r| < n -- no final correction, because the next square does not care
// about the sign and every later product accepts |.| < n.
//   h + l = a b exactly (|ab| < 2 n^2 < 2^101, so |l| <= ulp(h)/2 <= 2^47);
//   q = round(h * fl(1/n)) in one FMA with the 1.5 * 2^52 addend (valid since
//       |h / n| < 2n <= 2^51):
//       |q - ab/n| <= 1/2 + (h/n) 2^-53 + |l|/n < 1/2 + 1/4 + 1/4 = 1
//       (n < 2^49: < 1/2 + 1/8 + 1/8, |r| < 0.75 n; the bit-length sort
//       keeps 2^49 <= n < 2^50 in warps of their own either way);
//   r = fma(-q, n, h) + l: both steps exact (integers, |h - qn| < n + |l| < 2^51).
// 7 FP64-pipe instructions for a square-and-double step (fsqr_lazy with f = 2)
// against 10 FP64 + 4 select/compare instructions for fmulmod + faddmod.
__device__ __forceinline__ double fmul_lazy(double a, double b, const ModF& M) {
    const double h = a * b;
    const double l = fma(a, b, -h);
    const double q = fma(h, M.ninv, FP_RND) - FP_RND;
    return fma(-q, M.n, h) + l;
}

// x * 2^b for b = bit 31 of w, by adding b to the exponent field of the
// double (exact for any nonzero x of normal magnitude; the ladders' residues of
// powers of 2 are never 0 for odd n) -- three integer instructions instead of
// a 64-bit compare, a select and a DMUL on the FP64 pipe.
__device__ __forceinline__ double fscale2_top(double x, uint32_t w) {
    return __hiloint2double(__double2hiint(x) + (int)((w >> 31) << 20), __double2loint(x));
}

// x^2 * 2^b for the base-2 ladder (ModMultiply case 3 folded in as an exact
// power-of-two scaling of one factor).  |x| < n, b = bit 31 of w.
__device__ __forceinline__ double fsqr_dbl_lazy(double x, uint32_t w, const ModF& M) {
    return fmul_lazy(fscale2_top(x, w), x, M);
}

// 2^b y mod n (b = bit 31 of w) for |y| < n < 2^51, lazily: z = 2^b y exactly (|z| < 2n),
// k = round(z / n) in {-2 .. 2} (the 1.5 * 2^52 addend, |z / n| < 2), r = z - k n
// exact with |r| <= n/2 + 1.  The base-2 ladder's doubling where folding it
// into the product would break fmul_lazy's bound (2^50 <= n < 2^51).
__device__ __forceinline__ double fdbl_if_lazy(double y, uint32_t w, const ModF& M) {
    const double z = fscale2_top(y, w);  // 2^b y, b = bit 31 of w
    const double k = fma(z, M.ninv, FP_RND) - FP_RND;
    return fma(-k, M.n, z);
}

// Signed representative -> congruence tests (|x| < n).
__device__ __forceinline__ bool f_is_one(double x, const ModF& M) { return x == 1.0 || x == 1.0 - M.n; }
__device__ __forceinline__ bool f_is_mone(double x, const ModF& M) { return x == -1.0 || x == M.nm1; }

// ModAdd in doubles: a + b < 2n < 2^50 is exact.
__device__ __forceinline__ double faddmod(double a, double b, const ModF& M) {
    const double s = a + b;
    return s >= M.n ? s - M.n : s;
}

}  // namespace isp
