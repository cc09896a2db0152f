// mont_ww_bench.cu -- 64-bit Montgomery squaring / product: the current
// full-width REDC (modmath.cuh msqr64 / msqr64_ptx / mmul64_ptx) against a
// word-wise REDC (two 32-bit reduction steps, m_i = t_i * n^-1 mod 2^32 by
// one IMAD, the cancelled low word of m_i * n0 taken as a carry-free IMAD.HI).
// Checks every variant against exact 128-bit host arithmetic on random and
// edge moduli, then times squaring chains and base-2 ladder steps at full
// occupancy.  Prints JSON lines.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/mont_ww_bench tools/mont_ww_bench.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include "../paper_2108_04791_b200/csrc/modmath.cuh"

using u64 = unsigned long long;
using u128 = unsigned __int128;

// ---- candidate: word-wise subtraction REDC (mirrors the library's version
// once promoted; kept here so the benchmark is self-contained)
__device__ __forceinline__ u64 sqr_ww(u64 x, u64 n, uint32_t ni) {
    u64 r;
    asm("{\n\t"
        ".reg .u32 x0, x1, n0, n1, p0, p1, c0, c1, h0, h1, t1, t2, t3, m0, g0, u0, u1, w1, w2, w3, bb, m1, g1, v0, v1, r0, r1, k0, k1;\n\t"
        ".reg .u64 W, G;\n\t"
        "mov.b64 {x0, x1}, %1;\n\t"
        "mov.b64 {n0, n1}, %2;\n\t"
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
        "mul.lo.u32 m0, p0, %3;\n\t"
        "mul.hi.u32 g0, m0, n0;\n\t"
        "cvt.u64.u32 G, g0;\n\t"
        "mad.wide.u32 W, m0, n1, G;\n\t"
        "mov.b64 {u0, u1}, W;\n\t"
        "sub.cc.u32 w1, t1, u0;\n\t"
        "subc.cc.u32 w2, t2, u1;\n\t"
        "subc.cc.u32 w3, t3, 0;\n\t"
        "subc.u32 bb, 0, 0;\n\t"
        "mul.lo.u32 m1, w1, %3;\n\t"
        "mul.hi.u32 g1, m1, n0;\n\t"
        "cvt.u64.u32 G, g1;\n\t"
        "mad.wide.u32 W, m1, n1, G;\n\t"
        "mov.b64 {v0, v1}, W;\n\t"
        "sub.cc.u32 r0, w2, v0;\n\t"
        "subc.cc.u32 r1, w3, v1;\n\t"
        "subc.u32 bb, bb, 0;\n\t"
        "and.b32 k0, n0, bb;\n\t"
        "and.b32 k1, n1, bb;\n\t"
        "add.cc.u32 r0, r0, k0;\n\t"
        "addc.u32 r1, r1, k1;\n\t"
        "mov.b64 %0, {r0, r1};\n\t"
        "}"
        : "=l"(r)
        : "l"(x), "l"(n), "r"(ni));
    return r;
}

__device__ __forceinline__ u64 mul_ww(u64 a, u64 b, u64 n, uint32_t ni) {
    u64 r;
    asm("{\n\t"
        ".reg .u32 a0, a1, b0, b1, n0, n1, p0, p1, c0, c1, e0, e1, h0, h1, t1, t2, t3, m0, g0, u0, u1, w1, w2, w3, bb, m1, g1, v0, v1, r0, r1, k0, k1;\n\t"
        ".reg .u64 W, G;\n\t"
        "mov.b64 {a0, a1}, %1;\n\t"
        "mov.b64 {b0, b1}, %2;\n\t"
        "mov.b64 {n0, n1}, %3;\n\t"
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
        "mul.lo.u32 m0, p0, %4;\n\t"
        "mul.hi.u32 g0, m0, n0;\n\t"
        "cvt.u64.u32 G, g0;\n\t"
        "mad.wide.u32 W, m0, n1, G;\n\t"
        "mov.b64 {u0, u1}, W;\n\t"
        "sub.cc.u32 w1, t1, u0;\n\t"
        "subc.cc.u32 w2, t2, u1;\n\t"
        "subc.cc.u32 w3, t3, 0;\n\t"
        "subc.u32 bb, 0, 0;\n\t"
        "mul.lo.u32 m1, w1, %4;\n\t"
        "mul.hi.u32 g1, m1, n0;\n\t"
        "cvt.u64.u32 G, g1;\n\t"
        "mad.wide.u32 W, m1, n1, G;\n\t"
        "mov.b64 {v0, v1}, W;\n\t"
        "sub.cc.u32 r0, w2, v0;\n\t"
        "subc.cc.u32 r1, w3, v1;\n\t"
        "subc.u32 bb, bb, 0;\n\t"
        "and.b32 k0, n0, bb;\n\t"
        "and.b32 k1, n1, bb;\n\t"
        "add.cc.u32 r0, r0, k0;\n\t"
        "addc.u32 r1, r1, k1;\n\t"
        "mov.b64 %0, {r0, r1};\n\t"
        "}"
        : "=l"(r)
        : "l"(a), "l"(b), "l"(n), "r"(ni));
    return r;
}

// word-wise REDC written in C (lets ptxas schedule the carries itself)
__device__ __forceinline__ u64 redc_ww_c(u64 lo, u64 hi, u64 n, uint32_t ni) {
    const uint32_t n0 = (uint32_t)n, n1 = (uint32_t)(n >> 32);
    const uint32_t t0 = (uint32_t)lo, t1 = (uint32_t)(lo >> 32);
    const uint32_t m0 = t0 * ni;
    const u64 u = (u64)m0 * n1 + __umulhi(m0, n0);
    // (hi:t1) - u as a 96-bit value with borrow
    const u64 w_lo = (((u64)(uint32_t)hi) << 32 | t1);
    const u64 wl = w_lo - u;
    const uint32_t brw1 = w_lo < u;
    const uint32_t w3 = (uint32_t)(hi >> 32) - brw1;
    const uint32_t bor1 = ((uint32_t)(hi >> 32) < brw1);
    const uint32_t w1 = (uint32_t)wl, w2 = (uint32_t)(wl >> 32);
    const uint32_t m1 = w1 * ni;
    const u64 v = (u64)m1 * n1 + __umulhi(m1, n0);
    const u64 top = ((u64)w3 << 32) | w2;
    const u64 r = top - v;
    const bool neg = bor1 | (top < v);
    return neg ? r + n : r;
}
__device__ __forceinline__ u64 sqr_ww_c(u64 x, u64 n, uint32_t ni) { return redc_ww_c(x * x, __umul64hi(x, x), n, ni); }

template <int V>
__device__ __forceinline__ u64 do_sqr(u64 x, u64 n, u64 ninv) {
    if (V == 0) return isp::redc64(x * x, __umul64hi(x, x), n, ninv);
    if (V == 1) return isp::msqr64_ptx(x, n, ninv);
    if (V == 2) return sqr_ww(x, n, (uint32_t)ninv);
    return sqr_ww_c(x, n, (uint32_t)ninv);
}
template <int V>
__device__ __forceinline__ u64 do_mul(u64 a, u64 b, u64 n, u64 ninv) {
    if (V == 0) return isp::redc64(a * b, __umul64hi(a, b), n, ninv);
    if (V == 1) return isp::mmul64_ptx(a, b, n, ninv);
    if (V == 2) return mul_ww(a, b, n, (uint32_t)ninv);
    return redc_ww_c(a * b, __umul64hi(a, b), n, (uint32_t)ninv);
}

template <int V>
__global__ void k_check(const u64* a, const u64* b, const u64* n, u64* rs, u64* rm, int count) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= count) return;
    const u64 ninv = isp::inv64(n[i]);
    rs[i] = do_sqr<V>(a[i], n[i], ninv);
    rm[i] = do_mul<V>(a[i], b[i], n[i], ninv);
}

constexpr int CH = 4;
constexpr int ITERS = 1024;

template <int V, int MODE>  // MODE 0: squarings, 1: base-2 ladder step, 2: products
__global__ void k_tput(u64* out, u64 seed, u64 dbits) {
    const u64 n = (seed | 1ull | (1ull << 63)) ^ ((u64)threadIdx.x << 20);
    const u64 ninv = isp::inv64(n);
    u64 x[CH], y[CH];
#pragma unroll
    for (int c = 0; c < CH; c++) {
        x[c] = ((threadIdx.x + 1) * 0x9E3779B97F4A7C15ull + c * 0x1234567ull) % n;
        y[c] = (x[c] * 0xD1B54A32D192ED03ull) % n;
    }
    for (int i = 0; i < ITERS; i++) {
        const bool bit = (dbits >> (i & 63)) & 1ull;
#pragma unroll
        for (int c = 0; c < CH; c++) {
            if (MODE == 2) {
                x[c] = do_mul<V>(x[c], y[c], n, ninv);
            } else {
                u64 s = do_sqr<V>(x[c], n, ninv);
                if (MODE == 1) {
                    const u64 z = isp::mdbl64(s, n);
                    s = bit ? z : s;
                }
                x[c] = s;
            }
        }
    }
    u64 s = 0;
#pragma unroll
    for (int c = 0; c < CH; c++) s ^= x[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
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

static u64 rng_state = 0x243F6A8885A308D3ull;
static u64 rnd() {
    u64 z = (rng_state += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
static u64 host_pow(u64 b, u64 e, u64 m) {
    u128 r = 1 % m, x = b % m;
    while (e) { if (e & 1) r = r * x % m; x = x * x % m; e >>= 1; }
    return (u64)r;
}

template <int V>
int check(const std::vector<u64>& A, const std::vector<u64>& B, const std::vector<u64>& N, u64* dA, u64* dB, u64* dN,
          u64* dS, u64* dM) {
    const int cnt = (int)A.size();
    k_check<V><<<(cnt + 255) / 256, 256>>>(dA, dB, dN, dS, dM, cnt);
    std::vector<u64> S(cnt), M(cnt);
    cudaMemcpy(S.data(), dS, cnt * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(M.data(), dM, cnt * 8, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int i = 0; i < cnt; i++) {
        const u64 n = N[i];
        // REDC(T) = T * 2^-64 mod n  <=>  r < n and r * 2^64 == T (mod n)
        const u64 r64 = (u64)(((u128)1 << 64) % n);
        const u64 es = (u64)((u128)A[i] * A[i] % n), em = (u64)((u128)A[i] * B[i] % n);
        const bool ok_s = S[i] < n && (u64)((u128)S[i] * r64 % n) == es;
        const bool ok_m = M[i] < n && (u64)((u128)M[i] * r64 % n) == em;
        if (!ok_s || !ok_m) {
            if (bad < 3) fprintf(stderr, "V%d mismatch n=%llu a=%llu b=%llu\n", V, n, A[i], B[i]);
            bad++;
        }
    }
    (void)host_pow;
    return bad;
}

int main() {
    // correctness: random odd moduli of every bit length 33..64 plus edges
    std::vector<u64> A, B, N;
    const u64 edges[] = {0xFFFFFFFFFFFFFFC5ull, 0xFFFFFFFFFFFFFFFFull, 0xFFFFFFFFFFFFFFC3ull, 0x8000000000000001ull,
                         0x8000000000000003ull, 0x7FFFFFFFFFFFFFFFull, 0x100000001ull, 0xFFFFFFFFull | (1ull << 32)};
    for (int rep = 0; rep < 1 << 20; rep++) {
        u64 n;
        if (rep < 8 * 4096) n = edges[rep & 7];
        else {
            const int L = 33 + (int)(rnd() % 32);
            n = (rnd() >> (64 - L)) | (1ull << (L - 1)) | 1ull;
        }
        u64 a, b;
        switch (rep % 5) {
            case 0: a = n - 1; b = n - 1 - (rnd() % 3); break;
            case 1: a = rnd() % 4; b = n - 1; break;
            default: a = rnd() % n; b = rnd() % n;
        }
        if (b >= n) b = n - 1;
        A.push_back(a); B.push_back(b); N.push_back(n);
    }
    const int cnt = (int)A.size();
    u64 *dA, *dB, *dN, *dS, *dM;
    cudaMalloc(&dA, cnt * 8); cudaMalloc(&dB, cnt * 8); cudaMalloc(&dN, cnt * 8);
    cudaMalloc(&dS, cnt * 8); cudaMalloc(&dM, cnt * 8);
    cudaMemcpy(dA, A.data(), cnt * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), cnt * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(dN, N.data(), cnt * 8, cudaMemcpyHostToDevice);
    const int bad0 = check<0>(A, B, N, dA, dB, dN, dS, dM);
    const int bad1 = check<1>(A, B, N, dA, dB, dN, dS, dM);
    const int bad2 = check<2>(A, B, N, dA, dB, dN, dS, dM);
    const int bad3 = check<3>(A, B, N, dA, dB, dN, dS, dM);
    printf("{\"check_cases\": %d, \"bad\": [%d, %d, %d, %d]}\n", cnt, bad0, bad1, bad2, bad3);

    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const int threads = 256;
    int maxb = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&maxb, k_tput<2, 1>, threads, 0);
    const int blocks = sms * (maxb > 0 ? maxb : 4);
    u64* buf;
    cudaMalloc(&buf, (size_t)blocks * threads * 8);
    const double ops = (double)blocks * threads * CH * ITERS;
    const u64 bits = 0xB5A3C96E1D4F2A87ull, seed = 0xD1B54A32D192ED03ull;
    const char* names[4] = {"c_full", "ptx_full", "ptx_ww", "c_ww"};
    float t[3][4];
    t[0][0] = time_ms([&] { k_tput<0, 0><<<blocks, threads>>>(buf, seed, bits); });
    t[0][1] = time_ms([&] { k_tput<1, 0><<<blocks, threads>>>(buf, seed, bits); });
    t[0][2] = time_ms([&] { k_tput<2, 0><<<blocks, threads>>>(buf, seed, bits); });
    t[0][3] = time_ms([&] { k_tput<3, 0><<<blocks, threads>>>(buf, seed, bits); });
    t[1][0] = time_ms([&] { k_tput<0, 1><<<blocks, threads>>>(buf, seed, bits); });
    t[1][1] = time_ms([&] { k_tput<1, 1><<<blocks, threads>>>(buf, seed, bits); });
    t[1][2] = time_ms([&] { k_tput<2, 1><<<blocks, threads>>>(buf, seed, bits); });
    t[1][3] = time_ms([&] { k_tput<3, 1><<<blocks, threads>>>(buf, seed, bits); });
    t[2][0] = time_ms([&] { k_tput<0, 2><<<blocks, threads>>>(buf, seed, bits); });
    t[2][1] = time_ms([&] { k_tput<1, 2><<<blocks, threads>>>(buf, seed, bits); });
    t[2][2] = time_ms([&] { k_tput<2, 2><<<blocks, threads>>>(buf, seed, bits); });
    t[2][3] = time_ms([&] { k_tput<3, 2><<<blocks, threads>>>(buf, seed, bits); });
    const char* modes[3] = {"sqr", "ladder", "mul"};
    for (int m = 0; m < 3; m++) {
        printf("{\"mode\": \"%s\", \"blocks\": %d, \"clock_mhz\": %d", modes[m], blocks, clk / 1000);
        for (int v = 0; v < 4; v++) printf(", \"%s\": %.4e", names[v], ops / (t[m][v] * 1e-3));
        printf("}\n");
    }
    printf("{\"err\": \"%s\"}\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
