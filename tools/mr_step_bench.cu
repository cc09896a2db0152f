// mr_step_bench.cu -- throughput of one base-2 ladder step (Montgomery square +
// conditional modular doubling) for several formulations of the 64-bit
// Montgomery squaring, 8 independent chains per thread, full grid.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/mr_step_bench tools/mr_step_bench.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include "../paper_2108_04791_b200/csrc/modmath.cuh"

constexpr int CH = 4;
constexpr int ITERS = 1024;

// v0: the original __umul64hi formulation
__device__ __forceinline__ uint64_t sqr_v0(uint64_t a, uint64_t n, uint64_t ninv) {
    uint64_t lo = a * a, hi = __umul64hi(a, a);
    uint64_t m = lo * ninv, mh = __umul64hi(m, n);
    uint64_t t = hi - mh;
    return hi < mh ? t + n : t;
}
// v1: 32-bit-limb C++ (three IMAD.WIDE for a^2 with folded addends)
__device__ __forceinline__ uint64_t sqr_v1(uint64_t a, uint64_t n, uint64_t ninv) {
    const uint32_t a0 = (uint32_t)a, a1 = (uint32_t)(a >> 32);
    const uint64_t p00 = (uint64_t)a0 * a0;
    const uint64_t c = (uint64_t)a0 * a1;
    const uint64_t s1 = (p00 >> 32) + (uint32_t)(c << 1);
    const uint64_t hi = (uint64_t)a1 * a1 + ((c >> 31) + (s1 >> 32));
    const uint64_t lo = (s1 << 32) | (uint32_t)p00;
    const uint32_t t0 = (uint32_t)lo, t1 = (uint32_t)(lo >> 32);
    const uint32_t i0 = (uint32_t)ninv, i1 = (uint32_t)(ninv >> 32);
    const uint64_t mw = (uint64_t)t0 * i0;
    const uint32_t m0 = (uint32_t)mw;
    const uint32_t m1 = (uint32_t)(mw >> 32) + t0 * i1 + t1 * i0;
    const uint32_t n0 = (uint32_t)n, n1 = (uint32_t)(n >> 32);
    const uint64_t q00 = (uint64_t)m0 * n0;
    const uint64_t q01 = (uint64_t)m0 * n1 + (q00 >> 32);
    const uint64_t q10 = (uint64_t)m1 * n0 + (uint32_t)q01;
    const uint64_t mh = (uint64_t)m1 * n1 + ((q01 >> 32) + (q10 >> 32));
    const uint64_t t = hi - mh;
    return hi < mh ? t + n : t;
}
__device__ __forceinline__ uint64_t sqr_v2(uint64_t a, uint64_t n, uint64_t ninv) { return isp::msqr64_ptx(a, n, ninv); }

template <int V, bool DBL>
__global__ void k_step(unsigned long long* out, unsigned long long seed, unsigned long long dbits) {
    const unsigned long long n = (seed | 1ull | (1ull << 63)) ^ ((unsigned long long)threadIdx.x << 20);
    const unsigned long long ninv = isp::inv64(n);
    unsigned long long x[CH];
#pragma unroll
    for (int c = 0; c < CH; c++) x[c] = ((threadIdx.x + 1) * 0x9E3779B97F4A7C15ull + c * 0x1234567ull) % n;
    for (int i = 0; i < ITERS; i++) {
        const bool bit = (dbits >> (i & 63)) & 1ull;
#pragma unroll
        for (int c = 0; c < CH; c++) {
            unsigned long long y = V == 0 ? sqr_v0(x[c], n, ninv) : V == 1 ? sqr_v1(x[c], n, ninv) : sqr_v2(x[c], n, ninv);
            if (DBL) {
                const unsigned long long z = isp::mdbl64(y, n);
                y = bit ? z : y;
            }
            x[c] = y;
        }
    }
    unsigned long long s = 0;
#pragma unroll
    for (int c = 0; c < CH; c++) s ^= x[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// phase-2-like step: 3 lockstep chains, 2-bit window (2 squarings + 1 multiply by a table entry)
template <int V>
__global__ void k_win(unsigned long long* out, unsigned long long seed, unsigned long long dbits) {
    const unsigned long long n = (seed | 1ull | (1ull << 63)) ^ ((unsigned long long)threadIdx.x << 20);
    const unsigned long long ninv = isp::inv64(n);
    isp::Mont64 M; M.n = n; M.ninv = ninv;
    unsigned long long x[3], t[3][3];
#pragma unroll
    for (int c = 0; c < 3; c++) {
        x[c] = ((threadIdx.x + 1) * 0x9E3779B97F4A7C15ull + c * 0x1234567ull) % n;
        for (int k = 0; k < 3; k++) t[c][k] = (x[c] * (k + 3)) % n;
    }
    for (int i = 0; i < ITERS / 4; i++) {
        const unsigned int dg = (dbits >> (2 * (i & 31))) & 3u;
#pragma unroll
        for (int c = 0; c < 3; c++) {
            if (V == 0) { x[c] = isp::msqr64(x[c], M); x[c] = isp::msqr64(x[c], M); }
            else { x[c] = isp::msqr64_ptx(x[c], n, ninv); x[c] = isp::msqr64_ptx(x[c], n, ninv); }
            unsigned long long m = dg == 1 ? t[c][0] : dg == 2 ? t[c][1] : dg == 3 ? t[c][2] : x[c];
            x[c] = V == 0 ? isp::mmul64(x[c], m, M) : isp::mmul64_ptx(x[c], m, n, ninv);
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = x[0] ^ x[1] ^ x[2];
}

template <typename F>
float time_ms(F f) {
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    f(); cudaDeviceSynchronize();
    cudaEventRecord(a);
    for (int r = 0; r < 5; r++) f();
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms = 0; cudaEventElapsedTime(&ms, a, b);
    return ms / 5;
}

int main() {
    int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    unsigned long long* buf; 
    const int threads = 256;
    int maxb = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&maxb, k_step<2, true>, threads, 0);
    const int blocks = sms * (maxb > 0 ? maxb : 4);
    cudaMalloc(&buf, (size_t)blocks * threads * 8);
    const double steps = (double)blocks * threads * CH * ITERS;
    const unsigned long long bits = 0xB5A3C96E1D4F2A87ull;
    float t[6];
    t[0] = time_ms([&] { k_step<0, false><<<blocks, threads>>>(buf, 0xD1B54A32D192ED03ull, bits); });
    t[1] = time_ms([&] { k_step<1, false><<<blocks, threads>>>(buf, 0xD1B54A32D192ED03ull, bits); });
    t[2] = time_ms([&] { k_step<2, false><<<blocks, threads>>>(buf, 0xD1B54A32D192ED03ull, bits); });
    t[3] = time_ms([&] { k_step<0, true><<<blocks, threads>>>(buf, 0xD1B54A32D192ED03ull, bits); });
    t[4] = time_ms([&] { k_step<1, true><<<blocks, threads>>>(buf, 0xD1B54A32D192ED03ull, bits); });
    t[5] = time_ms([&] { k_step<2, true><<<blocks, threads>>>(buf, 0xD1B54A32D192ED03ull, bits); });
    float tw0 = time_ms([&] { k_win<0><<<blocks, threads>>>(buf, 0xD1B54A32D192ED03ull, bits); });
    float tw1 = time_ms([&] { k_win<1><<<blocks, threads>>>(buf, 0xD1B54A32D192ED03ull, bits); });
    unsigned long long hw[2];
    k_win<0><<<1, 32>>>(buf, 99, bits); cudaMemcpy(&hw[0], buf + 3, 8, cudaMemcpyDeviceToHost);
    k_win<1><<<1, 32>>>(buf, 99, bits); cudaMemcpy(&hw[1], buf + 3, 8, cudaMemcpyDeviceToHost);
    const double wsteps = (double)blocks * threads * 3 * 3 * (ITERS / 4);
    printf("{\"win_mulmods_per_s\": {\"v0\": %.4e, \"ptx\": %.4e}, \"win_agree\": %s}\n", wsteps / (tw0 * 1e-3),
           wsteps / (tw1 * 1e-3), hw[0] == hw[1] ? "true" : "false");
    // cross-check: the three squarings agree
    unsigned long long h[3];
    cudaError_t e = cudaDeviceSynchronize();
    for (int v = 0; v < 3; v++) {
        if (v == 0) k_step<0, true><<<1, 32>>>(buf, 77, bits);
        if (v == 1) k_step<1, true><<<1, 32>>>(buf, 77, bits);
        if (v == 2) k_step<2, true><<<1, 32>>>(buf, 77, bits);
        cudaMemcpy(&h[v], buf + 5, 8, cudaMemcpyDeviceToHost);
    }
    printf("{\"blocks\": %d, \"err\": \"%s\", \"agree\": %s, \"steps_per_s\": {\"sqr_v0\": %.4e, \"sqr_v1\": %.4e, \"sqr_ptx\": %.4e, "
           "\"ladder_v0\": %.4e, \"ladder_v1\": %.4e, \"ladder_ptx\": %.4e}}\n",
           blocks, cudaGetErrorString(e), (h[0] == h[1] && h[1] == h[2]) ? "true" : "false",
           steps / (t[0] * 1e-3), steps / (t[1] * 1e-3), steps / (t[2] * 1e-3),
           steps / (t[3] * 1e-3), steps / (t[4] * 1e-3), steps / (t[5] * 1e-3));
    return 0;
}
