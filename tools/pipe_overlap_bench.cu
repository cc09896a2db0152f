// pipe_overlap_bench.cu -- do DFMA (FP64 pipe) and IMAD.WIDE (FMA-heavy pipe)
// streams from different warps of one SM run concurrently on sm_100a?
//
// Three launches with the same per-warp work: all warps run an FP64 FMA loop
// (8 independent chains), all warps run an IMAD.WIDE loop (8 independent
// 64-bit multiply-accumulate chains), and a mixed launch where even warps run
// the FP64 loop and odd warps the integer loop.  If the pipes overlap, the
// mixed launch takes about max(fp64, int) / 2 + ... i.e. close to half of
// (fp64 + int); if they share a datapath, about (fp64 + int) / 2 per warp-half
// means no saving over running them back to back.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/pipe_overlap_bench.cu -o /tmp/pob && /tmp/pob
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;

__device__ __forceinline__ void fp64_work(double* out, double seed) {
    double a[8];
#pragma unroll
    for (int k = 0; k < 8; k++) a[k] = seed + k;
    const double m = 1.0000001, c = 1e-9;
    for (int i = 0; i < ITERS; i++) {
#pragma unroll
        for (int k = 0; k < 8; k++) a[k] = fma(a[k], m, c);
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < 8; k++) s += a[k];
    *out = s;
}

__device__ __forceinline__ void int_work(unsigned long long* out, unsigned long long seed) {
    unsigned long long a[8];
#pragma unroll
    for (int k = 0; k < 8; k++) a[k] = seed + k;
    const unsigned int m = 0x9E3779B1u;
    for (int i = 0; i < ITERS; i++) {
#pragma unroll
        for (int k = 0; k < 8; k++) {
            // one IMAD.WIDE.U32 per step: 64-bit accumulate of a 32x32 product
            a[k] = (unsigned long long)(unsigned int)a[k] * m + (a[k] >> 32);
        }
    }
    unsigned long long s = 0;
#pragma unroll
    for (int k = 0; k < 8; k++) s ^= a[k];
    *out = s;
}

__global__ void k_fp64(double* o) { fp64_work(o + blockIdx.x * blockDim.x + threadIdx.x, threadIdx.x); }
__global__ void k_int(unsigned long long* o) { int_work(o + blockIdx.x * blockDim.x + threadIdx.x, threadIdx.x); }
__global__ void k_mixed(double* o, unsigned long long* p) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if ((threadIdx.x >> 5) & 1) int_work(p + t, threadIdx.x);
    else fp64_work(o + t, threadIdx.x);
}

template <typename F>
float time_it(F f) {
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

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int blocks = sms * 4, threads = 256;
    double* o;
    unsigned long long* p;
    cudaMalloc(&o, sizeof(double) * blocks * threads);
    cudaMalloc(&p, sizeof(unsigned long long) * blocks * threads);
    // same number of warps in every launch; the mixed launch gives each kind half of them
    const float t_fp = time_it([&] { k_fp64<<<blocks, threads>>>(o); });
    const float t_int = time_it([&] { k_int<<<blocks, threads>>>(p); });
    const float t_mix = time_it([&] { k_mixed<<<blocks, threads>>>(o, p); });
    printf("{\"fp64_all_warps_ms\": %.4f, \"int_all_warps_ms\": %.4f, \"mixed_half_each_ms\": %.4f, "
           "\"back_to_back_halves_ms\": %.4f, \"overlap_gain\": %.3f}\n",
           t_fp, t_int, t_mix, 0.5f * (t_fp + t_int), 0.5f * (t_fp + t_int) / t_mix);
    return 0;
}
