// imad_peak.cu -- micro-benchmark of the integer-multiply issue rate on the
// FMA-heavy pipe (IMAD, IMAD.WIDE.U32, IMAD.HI.U32) and of the Montgomery
// mulmods of paper_2108_04791_b200/csrc/modmath.cuh, in lane-ops per clock
// per SM.  Prints one JSON line.  Build + run:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/imad_peak tools/imad_peak.cu && tools/imad_peak
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include "../paper_2108_04791_b200/csrc/modmath.cuh"

constexpr int CH = 8;      // independent chains per thread
constexpr int ITERS = 4096;

__global__ void k_imad_lo(uint32_t* out, uint32_t a, uint32_t b) {
    uint32_t x[CH];
#pragma unroll
    for (int c = 0; c < CH; c++) x[c] = threadIdx.x + c;
    for (int i = 0; i < ITERS; i++) {
#pragma unroll
        for (int c = 0; c < CH; c++) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x[c]) : "r"(a), "r"(b));
    }
    uint32_t s = 0;
#pragma unroll
    for (int c = 0; c < CH; c++) s ^= x[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_imad_wide(unsigned long long* out, uint32_t a) {
    unsigned long long x[CH];
#pragma unroll
    for (int c = 0; c < CH; c++) x[c] = threadIdx.x + c;
    for (int i = 0; i < ITERS; i++) {
#pragma unroll
        for (int c = 0; c < CH; c++) {
            uint32_t lo = (uint32_t)x[c];
            asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(x[c]) : "r"(lo), "r"(a));
        }
    }
    unsigned long long s = 0;
#pragma unroll
    for (int c = 0; c < CH; c++) s ^= x[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_imad_hi(uint32_t* out, uint32_t a, uint32_t b) {
    uint32_t x[CH];
#pragma unroll
    for (int c = 0; c < CH; c++) x[c] = threadIdx.x * 77777u + c;
    for (int i = 0; i < ITERS; i++) {
#pragma unroll
        for (int c = 0; c < CH; c++) asm volatile("mad.hi.u32 %0, %0, %1, %2;" : "+r"(x[c]) : "r"(a), "r"(b));
    }
    uint32_t s = 0;
#pragma unroll
    for (int c = 0; c < CH; c++) s ^= x[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_mont64(unsigned long long* out, unsigned long long n0) {
    const unsigned long long n = n0 | 1ull | (1ull << 63);
    isp::Mont64 M;
    M.n = n; M.ninv = isp::inv64(n); M.one = 0ull - n; M.mone = n - M.one;
    unsigned long long x[CH];
#pragma unroll
    for (int c = 0; c < CH; c++) x[c] = (threadIdx.x * 0x9E3779B97F4A7C15ull + c) % n;
    for (int i = 0; i < ITERS / 8; i++) {
#pragma unroll
        for (int c = 0; c < CH; c++) x[c] = isp::msqr64(x[c], M);
    }
    unsigned long long s = 0;
#pragma unroll
    for (int c = 0; c < CH; c++) s ^= x[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_mont32(uint32_t* out, uint32_t n0) {
    const uint32_t n = n0 | 1u | (1u << 31);
    isp::Mont32 M;
    M.n = n; M.ninv = isp::inv32(n); M.one = 0u - n; M.mone = n - M.one;
    uint32_t x[CH];
#pragma unroll
    for (int c = 0; c < CH; c++) x[c] = (threadIdx.x * 2654435761u + c) % n;
    for (int i = 0; i < ITERS / 2; i++) {
#pragma unroll
        for (int c = 0; c < CH; c++) x[c] = isp::mmul32(x[c], x[c], M);
    }
    uint32_t s = 0;
#pragma unroll
    for (int c = 0; c < CH; c++) s ^= x[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_dfma(double* out, double a, double b) {
    double x[CH];
#pragma unroll
    for (int c = 0; c < CH; c++) x[c] = threadIdx.x * 1e-3 + c;
    for (int i = 0; i < ITERS; i++) {
#pragma unroll
        for (int c = 0; c < CH; c++) x[c] = fma(x[c], a, b);
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < CH; c++) s += x[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// FP64 modular multiplication for n < 2^50: exact product h + l by FMA,
// quotient estimate by the rounded reciprocal, exact remainder by FMA, two fix-ups.
__device__ __forceinline__ double fmulmod(double a, double b, double n, double ninv) {
    const double h = a * b;
    const double l = fma(a, b, -h);
    const double q = (h * ninv + 6755399441055744.0) - 6755399441055744.0;  // round to nearest (|x| < 2^51)
    double r = fma(-q, n, h) + l;
    r = r < 0.0 ? r + n : r;
    r = r >= n ? r - n : r;
    return r;
}

__global__ void k_fmod(double* out, double n0) {
    const double n = n0 + 2.0 * threadIdx.x;
    const double ninv = 1.0 / n;
    double x[CH];
#pragma unroll
    for (int c = 0; c < CH; c++) x[c] = 12345.0 * (threadIdx.x + 1) + 7.0 * c;
    for (int i = 0; i < ITERS / 8; i++) {
#pragma unroll
        for (int c = 0; c < CH; c++) x[c] = fmulmod(x[c], x[c], n, ninv);
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < CH; c++) s += x[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <typename F>
float time_ms(F f) {
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
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

int main() {
    int sms = 0, clk_khz = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
    const int blocks = sms * 8, threads = 256;
    const double nthreads = (double)blocks * threads;
    void* buf = nullptr;
    cudaMalloc(&buf, (size_t)blocks * threads * 8);
    float t_lo = time_ms([&] { k_imad_lo<<<blocks, threads>>>((uint32_t*)buf, 3u, 7u); });
    float t_wide = time_ms([&] { k_imad_wide<<<blocks, threads>>>((unsigned long long*)buf, 3u); });
    float t_hi = time_ms([&] { k_imad_hi<<<blocks, threads>>>((uint32_t*)buf, 0x9E3779B9u, 7u); });
    float t_m64 = time_ms([&] { k_mont64<<<blocks, threads>>>((unsigned long long*)buf, 0xD1B54A32D192ED03ull); });
    float t_m32 = time_ms([&] { k_mont32<<<blocks, threads>>>((uint32_t*)buf, 0xD1B54A33u); });
    float t_dfma = time_ms([&] { k_dfma<<<blocks, threads>>>((double*)buf, 0.999999, 1e-9); });
    float t_fmod = time_ms([&] { k_fmod<<<blocks, threads>>>((double*)buf, 1125899906842597.0 /* 2^50 - 27 */); });
    cudaError_t e = cudaDeviceSynchronize();
    const double ops = nthreads * CH * ITERS;
    auto rate = [&](double n, float ms) { return n / (ms * 1e-3); };
    // lane-ops per clock per SM at the attribute clock (max boost) -- a lower bound if clocks sagged
    const double clk = clk_khz * 1e3;
    printf("{\"sms\": %d, \"clock_attr_mhz\": %.0f, \"err\": \"%s\", "
           "\"imad_lo_per_s\": %.4e, \"imad_wide_per_s\": %.4e, \"imad_hi_per_s\": %.4e, "
           "\"imad_lo_lanes_per_clk_sm\": %.2f, \"imad_wide_lanes_per_clk_sm\": %.2f, \"imad_hi_lanes_per_clk_sm\": %.2f, "
           "\"mont64_sqr_per_s\": %.4e, \"mont32_mul_per_s\": %.4e, \"dfma_per_s\": %.4e, \"dfma_lanes_per_clk_sm\": %.2f, "
           "\"fp64_mulmod50_per_s\": %.4e}\n",
           sms, clk / 1e6, cudaGetErrorString(e),
           rate(ops, t_lo), rate(ops, t_wide), rate(ops, t_hi),
           rate(ops, t_lo) / clk / sms, rate(ops, t_wide) / clk / sms, rate(ops, t_hi) / clk / sms,
           rate(nthreads * CH * (ITERS / 8), t_m64), rate(nthreads * CH * (ITERS / 2), t_m32),
           rate(ops, t_dfma), rate(ops, t_dfma) / clk / sms, rate(nthreads * CH * (ITERS / 8), t_fmod));
    return e == cudaSuccess ? 0 : 1;
}
