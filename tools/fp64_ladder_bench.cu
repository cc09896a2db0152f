// fp64_ladder_bench.cu -- what bounds the FP64-class witness ladders on B200:
// the base-2 square-and-double step of sprp2_f64 (fsqr_dbl_lazy: 6 FP64-pipe
// instructions + 2 integer) run as CH independent chains per thread, at
// several block shapes / occupancies.  Also the dependent-DFMA latency.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/fp64_ladder_bench tools/fp64_ladder_bench.cu
// Prints one JSON line: steps/s per (CH, threads per block, min blocks per SM)
// and the FP64-pipe fraction assuming 64 DFMA lanes/clk/SM (MEASURED_PEAKS sm clock).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#include "../paper_2108_04791_b200/csrc/modmath.cuh"

using namespace isp;

constexpr int STEPS = 512;

template <int CH>
__device__ __forceinline__ void ladder(double (&x)[CH], const ModF (&M)[CH], uint32_t w0) {
    uint32_t w = w0;
#pragma unroll 4
    for (int k = 0; k < STEPS; k++) {
#pragma unroll
        for (int c = 0; c < CH; c++) x[c] = fsqr_dbl_lazy(x[c], w << c, M[c]);
        w = (w << 1) | (w >> 31);
    }
}

template <int CH, int NT, int MINB>
__global__ void __launch_bounds__(NT, MINB) ladder_kernel(const unsigned long long* ns, double* out, uint32_t seed) {
    const unsigned t = blockIdx.x * NT + threadIdx.x;
    ModF M[CH];
    double x[CH];
#pragma unroll
    for (int c = 0; c < CH; c++) {
        M[c] = modf_setup(ns[(t * CH + c) & 4095]);
        x[c] = 2.0;
    }
    ladder<CH>(x, M, seed ^ (t * 0x9E3779B1u));
    double s = 0;
#pragma unroll
    for (int c = 0; c < CH; c++) s += x[c];
    out[t] = s;
}

// base-2 ladder step of sprp2_32 (32-bit Montgomery square, ModAdd doubling,
// select on the exponent bit), CH chains per thread; MIX: odd warps run it,
// even warps the FP64 step (both pipes fed by different warps of one SMSP)
template <int CH, bool MIX>
__global__ void __launch_bounds__(256) mont32_kernel(const unsigned long long* ns, double* out, uint32_t seed) {
    const unsigned t = blockIdx.x * 256 + threadIdx.x;
    if (MIX && ((threadIdx.x >> 5) & 1) == 0) {
        ModF M[CH];
        double x[CH];
#pragma unroll
        for (int c = 0; c < CH; c++) {
            M[c] = modf_setup(ns[(t * CH + c) & 4095]);
            x[c] = 2.0;
        }
        ladder<CH>(x, M, seed ^ (t * 0x9E3779B1u));
        double sum = 0;
#pragma unroll
        for (int c = 0; c < CH; c++) sum += x[c];
        out[t] = sum;
        return;
    }
    Mont32 M[CH];
    uint32_t x[CH];
#pragma unroll
    for (int c = 0; c < CH; c++) {
        M[c] = mont32_setup((uint32_t)ns[(t * CH + c) & 4095]);
        x[c] = madd32(M[c].one, M[c].one, M[c].n);
    }
    uint32_t w = seed ^ (t * 0x9E3779B1u);
#pragma unroll 4
    for (int k = 0; k < STEPS; k++) {
#pragma unroll
        for (int c = 0; c < CH; c++) {
            const uint32_t y = mmul32(x[c], x[c], M[c]);
            const uint32_t z = madd32(y, y, M[c].n);
            x[c] = ((w << c) >> 31) ? z : y;
        }
        w = (w << 1) | (w >> 31);
    }
    uint32_t sum = 0;
#pragma unroll
    for (int c = 0; c < CH; c++) sum += x[c];
    out[t] = (double)sum;
}

template <int CH, bool MIX>
double run_m(const unsigned long long* dn, double* dout, int sms) {
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, mont32_kernel<CH, MIX>, 256, 0);
    const int grid = sms * occ * 8;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    mont32_kernel<CH, MIX><<<grid, 256>>>(dn, dout, 1);
    cudaEventRecord(e0);
    for (int r = 0; r < 3; r++) mont32_kernel<CH, MIX><<<grid, 256>>>(dn, dout, 2 + r);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    return 3.0 * grid * 256 * CH * (double)STEPS / (ms * 1e-3);
}

__global__ void dfma_latency_kernel(double* out, double a, int iters, long long* cyc) {
    double x = a;
    const long long t0 = clock64();
    for (int i = 0; i < iters; i++) x = fma(x, a, 0.5);
    const long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}

template <int CH, int NT, int MINB>
double run(const unsigned long long* dn, double* dout, int sms, int* blocks_per_sm, int smem = 0) {
    int occ = 0;
    if (smem) cudaFuncSetAttribute(ladder_kernel<CH, NT, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, ladder_kernel<CH, NT, MINB>, NT, smem);
    *blocks_per_sm = occ;
    const int grid = sms * occ * 8;  // 8 waves of full occupancy
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    ladder_kernel<CH, NT, MINB><<<grid, NT, smem>>>(dn, dout, 1);
    cudaEventRecord(e0);
    for (int r = 0; r < 3; r++) ladder_kernel<CH, NT, MINB><<<grid, NT, smem>>>(dn, dout, 2 + r);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double steps = 3.0 * grid * NT * CH * (double)STEPS;
    return steps / (ms * 1e-3);
}

int main() {
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    unsigned long long hn[4096];
    unsigned long long s = 88172645463325252ull;
    for (int i = 0; i < 4096; i++) {
        s ^= s << 13; s ^= s >> 7; s ^= s << 17;
        hn[i] = ((s >> 32) | 0x80000000ull) | 1ull;  // odd 32-bit moduli
    }
    unsigned long long* dn;
    double* dout;
    cudaMalloc(&dn, sizeof(hn));
    cudaMemcpy(dn, hn, sizeof(hn), cudaMemcpyHostToDevice);
    cudaMalloc(&dout, (size_t)sms * 2048 * 8 * 8 * sizeof(double));
    long long* dcyc;
    cudaMalloc(&dcyc, sizeof(long long));
    dfma_latency_kernel<<<1, 32>>>(dout, 0.999, 4096, dcyc);
    long long cyc = 0;
    cudaMemcpy(&cyc, dcyc, sizeof(cyc), cudaMemcpyDeviceToHost);
    const double peak_steps = (double)sms * 64.0 * 1965e6 / 6.0;  // 6 FP64 ops per step at 64 lanes/clk/SM
    printf("{\"sms\": %d, \"clock_khz\": %d, \"dfma_dep_latency_cyc\": %.2f, \"peak_steps_per_s_6fp64\": %.4e, \"runs\": [",
           sms, clk, (double)cyc / 4096.0, peak_steps);
    bool first = true;
#define RUN(CH, NT, MINB) RUNS(CH, NT, MINB, 0)
#define RUNS(CH, NT, MINB, SMEM)                                                                             \
    {                                                                                                        \
        int b = 0;                                                                                           \
        const double r = run<CH, NT, MINB>(dn, dout, sms, &b, SMEM);                                         \
        printf("%s{\"ch\": %d, \"threads\": %d, \"minb\": %d, \"blocks_per_sm\": %d, \"warps_per_smsp\": %d, " \
               "\"steps_per_s\": %.4e, \"frac\": %.3f}",                                                     \
               first ? "" : ", ", CH, NT, MINB, b, b * NT / 128, r, r / peak_steps);                         \
        first = false;                                                                                       \
    }
    RUN(1, 256, 1) RUN(1, 256, 4) RUN(1, 256, 8)
    RUN(2, 256, 1) RUN(2, 256, 4) RUN(2, 256, 8)
    RUN(4, 256, 1) RUN(4, 256, 4) RUN(4, 256, 6)
    RUN(1, 512, 2) RUN(2, 512, 2) RUN(1, 1024, 1) RUN(2, 1024, 1)
    // lower occupancy forced through dynamic shared memory: 8 and 4 warps per SMSP
    RUNS(1, 256, 1, 50000) RUNS(2, 256, 1, 50000) RUNS(3, 256, 1, 50000) RUNS(4, 256, 1, 50000)
    RUNS(1, 256, 1, 100000) RUNS(2, 256, 1, 100000) RUNS(4, 256, 1, 100000)
    printf("], \"mont32_steps_per_s\": {\"ch1\": %.4e, \"ch2\": %.4e, \"ch4\": %.4e}, \"mixed_fp64_mont32_steps_per_s\": {\"ch1\": %.4e, \"ch2\": %.4e}",
           run_m<1, false>(dn, dout, sms), run_m<2, false>(dn, dout, sms), run_m<4, false>(dn, dout, sms),
           run_m<1, true>(dn, dout, sms), run_m<2, true>(dn, dout, sms));
    printf(", \"err\": \"%s\"}\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
