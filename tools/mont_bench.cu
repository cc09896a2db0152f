// mont_bench.cu -- throughput of 64-bit Montgomery squaring formulations on
// B200 (chains of squarings, CH independent chains per thread, full grid),
// and of FP64-class / Montgomery-class warps sharing an SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/mont_bench tools/mont_bench.cu
// Prints one JSON line: squarings/s per variant, and agreement of the
// variants' results.
//   S0  msqr64_ptx (subtraction REDC, 8 IMAD.WIDE + 2 IMAD)
//   S1  subtraction REDC without the m0*n0 product (7 IMAD.WIDE): its high
//       word follows from the known low 64 bits of m*n (= lo(T))
//   L0  msqr64_lz_ptx (additive lazy REDC, n < 2^62)
//   L1  additive lazy REDC without m0*n0
//   F   FP64 lazy product (fmul_lazy), for the mixed-warp test
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#include "../paper_2108_04791_b200/csrc/modmath.cuh"

using namespace isp;

// subtraction REDC of x^2 with hi(m n) from three products:
// lo64(m n) = lo64(T) = (t1, p0), so hi32(m0 n0) = t1 - lo(m0 n1) - lo(m1 n0)
// (mod 2^32) and the column-1 carry is the borrow of that plus the carry of
// lo(m0 n1) + lo(m1 n0).
__device__ __forceinline__ uint64_t msqr64_s1(uint64_t x, uint64_t n, uint64_t ninv) {
    uint64_t r;
    asm("{\n\t"
        ".reg .u32 x0, x1, n0, n1, i0, i1, p0, p1, c0, c1, h0, h1, t1, t2, t3, m0, m1;\n\t"
        ".reg .u32 l01, h01, l10, h10, l11, h11, s, sc, z, bb, k, u2, u3, r0, r1, bw, k0, k1;\n\t"
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
        "mul.wide.u32 W, p0, i0;\n\t"
        "mov.b64 {m0, m1}, W;\n\t"
        "mad.lo.u32 m1, p0, i1, m1;\n\t"
        "mad.lo.u32 m1, t1, i0, m1;\n\t"
        "mul.wide.u32 W, m0, n1;\n\t"
        "mov.b64 {l01, h01}, W;\n\t"
        "mul.wide.u32 W, m1, n0;\n\t"
        "mov.b64 {l10, h10}, W;\n\t"
        "mul.wide.u32 W, m1, n1;\n\t"
        "mov.b64 {l11, h11}, W;\n\t"
        "add.cc.u32 s, l01, l10;\n\t"
        "addc.u32 sc, 0, 0;\n\t"
        "sub.cc.u32 z, t1, s;\n\t"
        "subc.u32 bb, 0, 0;\n\t"
        "sub.u32 k, sc, bb;\n\t"
        "add.cc.u32 u2, l11, h01;\n\t"
        "addc.u32 u3, h11, 0;\n\t"
        "add.cc.u32 u2, u2, h10;\n\t"
        "addc.u32 u3, u3, 0;\n\t"
        "add.cc.u32 u2, u2, k;\n\t"
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
        : "l"(x), "l"(n), "l"(ninv));
    return r;
}

// additive lazy REDC of x^2 (nn = -n^-1 mod 2^64, n < 2^62, x < 2n -> < 2n)
// without m0 n0: T + m n == 0 (mod 2^64), so column 0 carries (p0 != 0) and
// column 1's total is a multiple of 2^32: k = hi(V) + (lo(V) != 0) with V =
// t1 + (p0 != 0) + lo(m0 n1) + lo(m1 n0).
__device__ __forceinline__ uint64_t msqr64_l1(uint64_t x, uint64_t n, uint64_t nn) {
    uint64_t r;
    asm("{\n\t"
        ".reg .u32 x0, x1, n0, n1, i0, i1, p0, p1, c0, c1, h0, h1, t1, t2, t3, m0, m1;\n\t"
        ".reg .u32 l01, h01, l10, h10, l11, h11, v, vh, cz, kv, k, r0, r1;\n\t"
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
        "mul.wide.u32 W, p0, i0;\n\t"
        "mov.b64 {m0, m1}, W;\n\t"
        "mad.lo.u32 m1, p0, i1, m1;\n\t"
        "mad.lo.u32 m1, t1, i0, m1;\n\t"
        "mul.wide.u32 W, m0, n1;\n\t"
        "mov.b64 {l01, h01}, W;\n\t"
        "mul.wide.u32 W, m1, n0;\n\t"
        "mov.b64 {l10, h10}, W;\n\t"
        "mul.wide.u32 W, m1, n1;\n\t"
        "mov.b64 {l11, h11}, W;\n\t"
        "min.u32 cz, p0, 1;\n\t"
        "add.cc.u32 v, t1, l01;\n\t"
        "addc.u32 vh, 0, 0;\n\t"
        "add.cc.u32 v, v, l10;\n\t"
        "addc.u32 vh, vh, 0;\n\t"
        "add.cc.u32 v, v, cz;\n\t"
        "addc.u32 vh, vh, 0;\n\t"
        "min.u32 kv, v, 1;\n\t"
        "add.u32 k, vh, kv;\n\t"
        "add.cc.u32 r0, t2, h01;\n\t"
        "addc.u32 r1, t3, h11;\n\t"
        "add.cc.u32 r0, r0, h10;\n\t"
        "addc.u32 r1, r1, 0;\n\t"
        "add.cc.u32 r0, r0, l11;\n\t"
        "addc.u32 r1, r1, 0;\n\t"
        "add.cc.u32 r0, r0, k;\n\t"
        "addc.u32 r1, r1, 0;\n\t"
        "mov.b64 %0, {r0, r1};\n\t"
        "}"
        : "=l"(r)
        : "l"(x), "l"(n), "l"(nn));
    return r;
}


// additive lazy REDC with hi(m0 n0) only (IMAD.HI instead of IMAD.WIDE):
// column 0 is p0 + lo(m0 n0) == 0 (mod 2^32), carrying (p0 != 0).
__device__ __forceinline__ uint64_t msqr64_l2(uint64_t x, uint64_t n, uint64_t nn) {
    uint64_t r;
    asm("{\n\t"
        ".reg .u32 x0, x1, n0, n1, i0, i1, p0, p1, c0, c1, h0, h1, t1, t2, t3, m0, m1;\n\t"
        ".reg .u32 q1, a0, a1, b0, b1, d0, d1, r0, r1, z, cz;\n\t"
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
        "mul.wide.u32 W, p0, i0;\n\t"
        "mov.b64 {m0, m1}, W;\n\t"
        "mad.lo.u32 m1, p0, i1, m1;\n\t"
        "mad.lo.u32 m1, t1, i0, m1;\n\t"
        "mul.hi.u32 q1, m0, n0;\n\t"
        "mul.wide.u32 W, m0, n1;\n\t"
        "mov.b64 {a0, a1}, W;\n\t"
        "mul.wide.u32 W, m1, n0;\n\t"
        "mov.b64 {b0, b1}, W;\n\t"
        "mul.wide.u32 W, m1, n1;\n\t"
        "mov.b64 {d0, d1}, W;\n\t"
        "min.u32 cz, p0, 1;\n\t"
        "add.cc.u32 z, t1, q1;\n\t"
        "addc.cc.u32 r0, t2, d0;\n\t"
        "addc.u32 r1, t3, d1;\n\t"
        "add.cc.u32 z, z, a0;\n\t"
        "addc.cc.u32 r0, r0, a1;\n\t"
        "addc.u32 r1, r1, 0;\n\t"
        "add.cc.u32 z, z, b0;\n\t"
        "addc.cc.u32 r0, r0, b1;\n\t"
        "addc.u32 r1, r1, 0;\n\t"
        "add.cc.u32 z, z, cz;\n\t"
        "addc.cc.u32 r0, r0, 0;\n\t"
        "addc.u32 r1, r1, 0;\n\t"
        "mov.b64 %0, {r0, r1};\n\t"
        "}"
        : "=l"(r)
        : "l"(x), "l"(n), "l"(nn));
    return r;
}

// word-by-word (two 32-bit steps) lazy REDC of x^2: np = -n^-1 mod 2^32,
// n < 2^62, x < 2n -> result < 2n.  The products' addends ride in the
// IMAD.WIDE's 64-bit addend: 7 IMAD.WIDE + 2 IMAD per square.
__device__ __forceinline__ uint64_t msqr64_w(uint64_t x, uint64_t n, uint32_t np) {
    uint64_t r;
    asm("{\n\t"
        ".reg .u32 x0, x1, n0, n1, t0, a1, c0, c1, h0, h1, t1, t2, t3, m, z, ah, s0, s1, u1, u2, v2, v3, ch, r0, dh, r1;\n\t"
        ".reg .u64 W, S;\n\t"
        "mov.b64 {x0, x1}, %1;\n\t"
        "mov.b64 {n0, n1}, %2;\n\t"
        "mul.wide.u32 W, x0, x0;\n\t"
        "mov.b64 {t0, a1}, W;\n\t"
        "mul.wide.u32 W, x0, x1;\n\t"
        "mov.b64 {c0, c1}, W;\n\t"
        "mul.wide.u32 W, x1, x1;\n\t"
        "mov.b64 {h0, h1}, W;\n\t"
        "add.cc.u32 t1, a1, c0;\n\t"
        "addc.cc.u32 t2, h0, c1;\n\t"
        "addc.u32 t3, h1, 0;\n\t"
        "add.cc.u32 t1, t1, c0;\n\t"
        "addc.cc.u32 t2, t2, c1;\n\t"
        "addc.u32 t3, t3, 0;\n\t"
        // step 1: m = t0 np; (T + m n) / 2^32
        "mul.lo.u32 m, t0, %3;\n\t"
        "mov.b64 S, {t0, 0};\n\t"
        "mad.wide.u32 W, m, n0, S;\n\t"
        "mov.b64 {z, ah}, W;\n\t"
        "add.cc.u32 s0, t1, ah;\n\t"
        "addc.u32 s1, 0, 0;\n\t"
        "mov.b64 S, {s0, s1};\n\t"
        "mad.wide.u32 W, m, n1, S;\n\t"
        "mov.b64 {u1, u2}, W;\n\t"
        "add.cc.u32 v2, t2, u2;\n\t"
        "addc.u32 v3, t3, 0;\n\t"
        // step 2: m = u1 np
        "mul.lo.u32 m, u1, %3;\n\t"
        "mov.b64 S, {u1, 0};\n\t"
        "mad.wide.u32 W, m, n0, S;\n\t"
        "mov.b64 {z, ch}, W;\n\t"
        "add.cc.u32 s0, v2, ch;\n\t"
        "addc.u32 s1, 0, 0;\n\t"
        "mov.b64 S, {s0, s1};\n\t"
        "mad.wide.u32 W, m, n1, S;\n\t"
        "mov.b64 {r0, dh}, W;\n\t"
        "add.u32 r1, v3, dh;\n\t"
        "mov.b64 %0, {r0, r1};\n\t"
        "}"
        : "=l"(r)
        : "l"(x), "l"(n), "r"(np));
    return r;
}

constexpr int ITERS = 2048;

template <int V, int CH>
__global__ void __launch_bounds__(256) k_sqr(unsigned long long* out, unsigned long long seed) {
    // moduli: V 0/1 in [2^63, 2^64), V >= 2 in [2^61, 2^62)
    unsigned long long n = seed ^ ((unsigned long long)(blockIdx.x * blockDim.x + threadIdx.x) * 0x9E3779B97F4A7C15ull);
    n |= 1ull;
    if (V <= 1) n |= 1ull << 63;
    else n = (n & ((1ull << 62) - 1)) | (1ull << 61);
    const unsigned long long ninv = inv64(n), nn = 0ull - ninv;
    const uint32_t np = (uint32_t)nn;
    unsigned long long x[CH];
#pragma unroll
    for (int c = 0; c < CH; c++) x[c] = ((threadIdx.x + 1) * 0x2545F4914F6CDD1Dull + c * 0x1234567ull) % n;
#pragma unroll 1
    for (int i = 0; i < ITERS; i++) {
#pragma unroll
        for (int c = 0; c < CH; c++) {
            if (V == 0) x[c] = msqr64_ptx(x[c], n, ninv);
            else if (V == 1) x[c] = msqr64_s1(x[c], n, ninv);
            else if (V == 2) x[c] = msqr64_lz_ptx(x[c], n, nn);
            else if (V == 3) x[c] = msqr64_l1(x[c], n, nn);
            else if (V == 4) x[c] = msqr64_l2(x[c], n, nn);
            else x[c] = msqr64_w(x[c], n, np);
        }
    }
    unsigned long long s = 0;
#pragma unroll
    for (int c = 0; c < CH; c++) s ^= (V >= 2 ? mcanon64(x[c], n) : x[c]);
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// mixed: warps with (warp id % MOD) < NF run FP64 lazy chains (n < 2^50),
// the others Montgomery S-variant chains; FP64 warps run FITER iterations
template <int MOD, int NF, int CH>
__global__ void __launch_bounds__(256) k_mixed(unsigned long long* out, unsigned long long seed, int fiters,
                                                int miters) {
    const int w = threadIdx.x >> 5;
    const unsigned long long t = seed ^ ((unsigned long long)(blockIdx.x * blockDim.x + threadIdx.x) * 0x9E3779B97F4A7C15ull);
    unsigned long long s = 0;
    if ((w % MOD) < NF) {
        const unsigned long long n = ((t & ((1ull << 49) - 1)) | (1ull << 49)) | 1ull;
        const ModF M = modf_setup(n);
        double x[CH];
#pragma unroll
        for (int c = 0; c < CH; c++) x[c] = (double)(((threadIdx.x + 7) * 0x2545F4914F6CDD1Dull + c) % n);
#pragma unroll 1
        for (int i = 0; i < fiters; i++) {
#pragma unroll
            for (int c = 0; c < CH; c++) x[c] = fmul_lazy(x[c], x[c], M);
        }
#pragma unroll
        for (int c = 0; c < CH; c++) s ^= (unsigned long long)(long long)x[c];
    } else {
        const unsigned long long n = t | 1ull | (1ull << 63);
        const unsigned long long ninv = inv64(n);
        unsigned long long x[CH];
#pragma unroll
        for (int c = 0; c < CH; c++) x[c] = ((threadIdx.x + 1) * 0x2545F4914F6CDD1Dull + c * 0x1234567ull) % n;
#pragma unroll 1
        for (int i = 0; i < miters; i++) {
#pragma unroll
            for (int c = 0; c < CH; c++) x[c] = msqr64_ptx(x[c], n, ninv);
        }
#pragma unroll
        for (int c = 0; c < CH; c++) s ^= x[c];
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// the base-2 ladder step of mr1 (square, times 2^bit, lazy REDC): CH
// independent ladders per thread, n in [2^60, 2^61), bits from a per-thread
// word (uniform 0/1 mix)
template <int CH, int THREADS>
__global__ void __launch_bounds__(THREADS) k_ladder(unsigned long long* out, unsigned long long seed) {
    unsigned long long n = seed ^ ((unsigned long long)(blockIdx.x * blockDim.x + threadIdx.x) * 0x9E3779B97F4A7C15ull);
    n = (n & ((1ull << 60) - 1)) | (1ull << 60) | 1ull;
    const unsigned long long nn = 0ull - inv64(n);
    uint32_t w = (uint32_t)(n >> 7) * 0x2545F491u;
    unsigned long long x[CH];
#pragma unroll
    for (int c = 0; c < CH; c++) x[c] = ((threadIdx.x + 1) * 0x2545F4914F6CDD1Dull + c * 0x1234567ull) % n;
#pragma unroll 1
    for (int i = 0; i < ITERS; i++) {
#pragma unroll
        for (int c = 0; c < CH; c++) x[c] = msqr64_shl_lz_ptx(x[c], n, nn, w >> 31);
        w = (w << 1) | (w >> 31);
    }
    unsigned long long s = 0;
#pragma unroll
    for (int c = 0; c < CH; c++) s ^= mcanon64(x[c], n);
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int CH, int THREADS>
double ladder_rate(unsigned long long* buf, int sms) {
    int maxb = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&maxb, k_ladder<CH, THREADS>, THREADS, 0);
    const int blocks = sms * (maxb > 0 ? maxb : 1);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    k_ladder<CH, THREADS><<<blocks, THREADS>>>(buf, 3);
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    for (int r = 0; r < 5; r++) k_ladder<CH, THREADS><<<blocks, THREADS>>>(buf, 3);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    return (double)blocks * THREADS * CH * ITERS / (ms / 5 * 1e-3);
}

template <typename F>
float time_ms(F f) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    f();
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    for (int r = 0; r < 5; r++) f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    return ms / 5;
}

template <int V, int CH>
double rate(unsigned long long* buf, int sms) {
    int maxb = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&maxb, k_sqr<V, CH>, 256, 0);
    const int blocks = sms * (maxb > 0 ? maxb : 4);
    const float ms = time_ms([&] { k_sqr<V, CH><<<blocks, 256>>>(buf, 0xD1B54A32D192ED03ull); });
    return (double)blocks * 256 * CH * ITERS / (ms * 1e-3);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    unsigned long long* buf;
    cudaMalloc(&buf, (size_t)sms * 8 * 256 * 8);
    printf("{\"sqr_per_s\": {\"S0_ch3\": %.4e, \"S1_ch3\": %.4e, \"S0_ch4\": %.4e, \"S1_ch4\": %.4e, "
           "\"L0_ch3\": %.4e, \"L1_ch3\": %.4e, \"L0_ch4\": %.4e, \"L1_ch4\": %.4e",
           rate<0, 3>(buf, sms), rate<1, 3>(buf, sms), rate<0, 4>(buf, sms), rate<1, 4>(buf, sms),
           rate<2, 3>(buf, sms), rate<3, 3>(buf, sms), rate<2, 4>(buf, sms), rate<3, 4>(buf, sms));
    printf(", \"L2_ch3\": %.4e, \"L2_ch4\": %.4e, \"W_ch3\": %.4e, \"W_ch4\": %.4e, \"W_ch6\": %.4e}",
           rate<4, 3>(buf, sms), rate<4, 4>(buf, sms), rate<5, 3>(buf, sms), rate<5, 4>(buf, sms), rate<5, 6>(buf, sms));
    printf(", \"ladder_shl_lz_per_s\": {\"ch1_t512\": %.4e, \"ch2_t512\": %.4e, \"ch1_t256\": %.4e, \"ch2_t256\": %.4e, "
           "\"ch3_t256\": %.4e, \"ch4_t256\": %.4e}",
           ladder_rate<1, 512>(buf, sms), ladder_rate<2, 512>(buf, sms), ladder_rate<1, 256>(buf, sms),
           ladder_rate<2, 256>(buf, sms), ladder_rate<3, 256>(buf, sms), ladder_rate<4, 256>(buf, sms));
    // agreement
    unsigned long long h[6];
    k_sqr<0, 3><<<1, 64>>>(buf, 12345);
    cudaMemcpy(&h[0], buf + 37, 8, cudaMemcpyDeviceToHost);
    k_sqr<1, 3><<<1, 64>>>(buf, 12345);
    cudaMemcpy(&h[1], buf + 37, 8, cudaMemcpyDeviceToHost);
    k_sqr<2, 3><<<1, 64>>>(buf, 12345);
    cudaMemcpy(&h[2], buf + 37, 8, cudaMemcpyDeviceToHost);
    k_sqr<3, 3><<<1, 64>>>(buf, 12345);
    cudaMemcpy(&h[3], buf + 37, 8, cudaMemcpyDeviceToHost);
    k_sqr<4, 3><<<1, 64>>>(buf, 12345);
    cudaMemcpy(&h[4], buf + 37, 8, cudaMemcpyDeviceToHost);
    k_sqr<5, 3><<<1, 64>>>(buf, 12345);
    cudaMemcpy(&h[5], buf + 37, 8, cudaMemcpyDeviceToHost);
    printf(", \"agree_S\": %s, \"agree_L\": %s, \"agree_L2\": %s, \"agree_W\": %s", h[0] == h[1] ? "true" : "false",
           h[2] == h[3] ? "true" : "false", h[2] == h[4] ? "true" : "false", h[2] == h[5] ? "true" : "false");
    // mixed warps: FP64-only, Montgomery-only, and half/half on the same SMs
    const int blocks = sms * 4;
    const int fit = 4096, mit = 1024;
    float tf = time_ms([&] { k_mixed<2, 2, 3><<<blocks, 256>>>(buf, 1, fit, mit); });  // all FP64
    float tm = time_ms([&] { k_mixed<2, 0, 3><<<blocks, 256>>>(buf, 1, fit, mit); });  // all Montgomery
    float tx = time_ms([&] { k_mixed<2, 1, 3><<<blocks, 256>>>(buf, 1, fit, mit); });  // half / half
    float tx4 = time_ms([&] { k_mixed<4, 1, 3><<<blocks, 256>>>(buf, 1, fit, mit); });  // 1/4 FP64
    printf(", \"mixed_ms\": {\"fp64_all\": %.4f, \"mont_all\": %.4f, \"half_half\": %.4f, \"quarter_fp64\": %.4f}",
           tf, tm, tx, tx4);
    printf(", \"err\": \"%s\"}\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
