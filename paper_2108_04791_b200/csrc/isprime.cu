// isprime.cu -- libisprime.so: C-ABI front end (layer L3) and planner /
// launcher (layer L2) of the B200 elementwise primality classifier.
//
// See include/isprime.h for the contract and DESIGN.md for the design.  Every
// step of the path runs in the kernels of kernels.cuh; the host only
// validates arguments, owns scratch memory and enqueues launches.  There is
// no CPU fallback: without a CUDA device every compute call fails with
// ISP_ENODEV.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/isprime.h"
#include "kernels.cuh"

using namespace isp;

namespace {

struct Options {
    int force_path = 0;      // 0 auto, 1 sieve, 2 mr
    int bases32 = 3;         // 3 -> {2,7,61}; 7 -> full Eq 4 set
    int td32 = kTD32Default; // odd primes 3..97 (round-2 re-sweep with the fused classify: C2 best at 24)
    int td64 = 32;
    int chunk_log2 = 30;     // device chunk: 2^30 elements need <= 64 GB of queues (of 180 GB); halved on ENOMEM
    int win64 = 3;           // phase-2 window bits (tables in shared memory; 3 measured best)
    int warp_p = 2048;
    // plan cost model, fitted on a B200 by tools/costfit.py (profiles/r1_costfit.json)
    long long sieve_fs_per_int = 331;     // femtoseconds per integer of window
    long long sieve_fixed_ns = 4475;
    long long mr32_fs_per_bit = 1594;     // femtoseconds per odd element per bit (trial division + MR)
    long long mr_fixed_ns = 24486;        // witness kernels' latency floor
    unsigned long long sieve_max = 1ull << 32;
    int kernel_timing = 0;
    int count_work = 0;      // witness tests count their algorithmic products (isprime_stats.mulmods*)
    int sieve_cache = 0;
    int pdl = 1;             // programmatic dependent launch of the pipeline kernels
    int mr2_group = 3;       // 64-bit phase-2 bases run G at a time in lockstep (3 or 6)
    long long small_max = 1 << 17;  // n <= small_max (and force_path auto): one fused launch
    long long warp_max = 4096;      // n <= warp_max: one warp per element (one base per lane)
    int small_sieve = 0;     // short arrays: 8-block clusters sieve [0, 2^20) in shared memory for their small values
                             // (measured on par with small_kernel on C1: 13.6-15.3 vs 13.6-14.1 us; kept as an option)
    int sched = 2;           // witness kernels: 0 dynamic guided claims (atomics), 1 static interleaved rounds,
                             // 2 static for the 32-bit class then dynamic for the 64-bit classes
    int fuse_bits = 32;      // classify runs the strong tests itself below 2^fuse_bits: 0 (off), 32, 51
    int graph = 0;           // 1: pipeline calls replay a cached CUDA graph whose conditional nodes skip the stages
                             // the plan / classify find empty (sieve, dense, sort + witness kernels).  Measured
                             // slower than the PDL-chained stream launches (C2 0.159 -> 0.177 ms, C5 3.632 ->
                             // 3.663 ms, C4 6.52 -> 6.63 ms: a conditional node breaks the programmatic edges
                             // and costs more than the ~1.3 us early-exit launch it skips), so off by default
    int witness = 0;         // 0: Eq 4 bases; 1: Baillie-PSW for n >= 2^50; 2: reduced sets by magnitude     // 1: a call may reuse the bitmap sieved by an earlier call
};

Options g_opt;
bool g_opt_env_read = false;
std::mutex g_mu;
std::string g_err;
unsigned long long g_launches = 0;
unsigned long long g_opt_epoch = 0;  // bumped by every option change: a cached graph bakes the options in
bool g_pdl_ok = true;                // false: the next launch follows a conditional node (no programmatic edge)
int g_gon = 0;                       // launches are being captured into a graph with conditional stages
unsigned long long g_gh_tail = 0;    // conditional handle classify sets when it queued survivors

struct Ctx {
    int dev = -1;
    int sms = 0;
    uint2* bp = nullptr;
    int nbp = 0;
    std::vector<uint2> hbp;
    uint8_t* patt = nullptr;
    uint32_t* bitmap = nullptr;
    DevPlan* plan = nullptr;
    unsigned int* segh = nullptr;  // per-classify-block bit-length histograms (the sort's offsets)
    unsigned char* qmem = nullptr;
    size_t qcap = 0;
    Queues q{};
    int grid_cls = 0, grid_mr1 = 0, grid_mr2 = 0, grid_sieve = 0, grid_sort = 0;
    cudaEvent_t last_done = nullptr;
    void* last_stream = nullptr;
    bool has_last = false;
    // host-API staging
    cudaStream_t hs[2] = {nullptr, nullptr};
    cudaEvent_t ev_h2d[2] = {nullptr, nullptr};
    cudaEvent_t ev_d2h[2] = {nullptr, nullptr};
    unsigned long long* din[2] = {nullptr, nullptr};
    uint8_t* dout[2] = {nullptr, nullptr};
    unsigned long long* hin[2] = {nullptr, nullptr};
    uint8_t* hout[2] = {nullptr, nullptr};
    size_t hcap = 0;
    // CUDA graphs of the pipeline (option "graph"), keyed by the call's
    // pointers, size, options and scratch; least recently used evicted past 8
    struct GraphEntry {
        const void* N; const void* out; size_t n; unsigned long long epoch; const void* qmem; size_t qcap;
        cudaGraphExec_t exec; unsigned long long used;
    };
    std::vector<GraphEntry> graphs;
    unsigned long long graph_clock = 0;
    cudaStream_t gs = nullptr, gs2 = nullptr;  // capture streams (the caller's may be the legacy stream)
};

std::vector<Ctx*> g_ctx;

// ---- optional per-kernel timing (events on the launching stream)
enum { K_PLAN, K_SIEVE, K_CLASSIFY, K_SORT, K_MR1, K_MR2, K_POPCOUNT, K_SMALL, K_DENSE, K_NUM };
const char* const k_names[K_NUM] = {"plan", "sieve", "classify", "sort", "mr1", "mr2", "popcount", "small", "dense"};
struct KTPending { cudaEvent_t a, b; int kid; };
std::vector<KTPending> g_kt_pending;
std::vector<cudaEvent_t> g_ev_pool;
double g_kt_ms[K_NUM] = {0};
unsigned long long g_kt_n[K_NUM] = {0};

cudaEvent_t ev_get() {
    if (!g_ev_pool.empty()) { cudaEvent_t e = g_ev_pool.back(); g_ev_pool.pop_back(); return e; }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}

void kt_drain() {
    if (g_kt_pending.empty()) return;
    for (auto& p : g_kt_pending) {
        float ms = 0.f;
        cudaEventSynchronize(p.b);
        if (cudaEventElapsedTime(&ms, p.a, p.b) == cudaSuccess) { g_kt_ms[p.kid] += ms; g_kt_n[p.kid]++; }
        g_ev_pool.push_back(p.a);
        g_ev_pool.push_back(p.b);
    }
    g_kt_pending.clear();
}

struct KScope {
    int kid; cudaStream_t s; cudaEvent_t a = nullptr;
    KScope(int k, cudaStream_t st) : kid(k), s(st) {
        if (g_opt.kernel_timing) { a = ev_get(); cudaEventRecord(a, s); }
    }
    ~KScope() {
        if (a) {
            cudaEvent_t b = ev_get();
            cudaEventRecord(b, s);
            g_kt_pending.push_back({a, b, kid});
            if (g_kt_pending.size() > 4096) kt_drain();
        }
    }
};

void read_env_once() {
    if (g_opt_env_read) return;
    g_opt_env_read = true;
    if (const char* e = getenv("ISPRIME_FORCE_PATH")) {
        if (!strcmp(e, "sieve")) g_opt.force_path = 1;
        else if (!strcmp(e, "mr")) g_opt.force_path = 2;
        else g_opt.force_path = 0;
    }
    if (const char* e = getenv("ISPRIME_BASES32")) g_opt.bases32 = atoi(e) == 7 ? 7 : 3;
    if (const char* e = getenv("ISPRIME_TD32")) g_opt.td32 = atoi(e);
    if (const char* e = getenv("ISPRIME_TD64")) g_opt.td64 = atoi(e);
    if (const char* e = getenv("ISPRIME_WIN64")) g_opt.win64 = atoi(e);
    if (const char* e = getenv("ISPRIME_CHUNK_LOG2")) g_opt.chunk_log2 = atoi(e);
    if (const char* e = getenv("ISPRIME_SIEVE_MAX")) {
        // the sieve works on whole 64-value bitmap words below 2^32
        unsigned long long v = strtoull(e, nullptr, 0) & ~63ull;
        g_opt.sieve_max = v > (1ull << 32) ? (1ull << 32) : v;
    }
    if (const char* e = getenv("ISPRIME_FUSE_BITS")) { const int v = atoi(e); if (v == 0 || v == 32 || v == 51) g_opt.fuse_bits = v; }
}

int cuda_fail(cudaError_t e, const char* what) {
    g_err = std::string(what) + ": " + cudaGetErrorString(e);
    return ISP_ECUDA;
}

#define CK(call)                                         \
    do {                                                 \
        cudaError_t e_ = (call);                         \
        if (e_ != cudaSuccess) return cuda_fail(e_, #call); \
    } while (0)

#define CKL(what)                                        \
    do {                                                 \
        g_launches++;                                    \
        cudaError_t e_ = cudaGetLastError();             \
        if (e_ != cudaSuccess) return cuda_fail(e_, what); \
    } while (0)

// Launch a pipeline kernel with programmatic stream serialisation (option
// "pdl", default 1): its launch overlaps the tail of the kernel before it on
// the stream; the kernel waits (kernels.cuh pdl_wait) before touching memory.
template <typename... KArgs, typename... Args>
cudaError_t launch_k(void (*k)(KArgs...), unsigned grid, unsigned block, size_t smem, cudaStream_t s,
                     Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = (g_opt.pdl && g_pdl_ok) ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    g_pdl_ok = true;
    return cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
}

// mr2_kernel's small-base table lives in dynamic shared memory beside 48 KB of
// static tables: the launch needs the opt-in attribute.
template <typename K>
void mr2_attr(K k) {
    cudaFuncSetAttribute((const void*)k, cudaFuncAttributeMaxDynamicSharedMemorySize, MR2_DYN_SMEM);
}

int occupancy(const void* fn, int threads, size_t smem) {
    int b = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, fn, threads, smem) != cudaSuccess || b < 1) b = 1;
    return b;
}

int init_ctx(Ctx* c) {
    CK(cudaGetDevice(&c->dev));
    CK(cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, c->dev));
    CK(cudaMalloc(&c->bp, 8192 * sizeof(uint2)));
    int* dcount = nullptr;
    CK(cudaMalloc(&dcount, sizeof(int)));
    init_base_primes_kernel<<<1, 1024>>>(c->bp, dcount);
    CKL("init_base_primes_kernel");
    CK(cudaMemcpy(&c->nbp, dcount, sizeof(int), cudaMemcpyDeviceToHost));
    CK(cudaFree(dcount));
    if (c->nbp != 6541) {  // odd primes below 65536
        g_err = "base prime table has " + std::to_string(c->nbp) + " entries, expected 6541";
        return ISP_ECUDA;
    }
    c->hbp.resize(c->nbp);
    CK(cudaMemcpy(c->hbp.data(), c->bp, c->nbp * sizeof(uint2), cudaMemcpyDeviceToHost));
    // trial-division constants -> __constant__
    {
        uint32_t *p32, *i32, *l32;
        unsigned long long *i64, *l64;
        CK(cudaMalloc(&p32, MAX_TD * 4));
        CK(cudaMalloc(&i32, MAX_TD * 4));
        CK(cudaMalloc(&l32, MAX_TD * 4));
        CK(cudaMalloc(&i64, MAX_TD * 8));
        CK(cudaMalloc(&l64, MAX_TD * 8));
        init_td_kernel<<<1, MAX_TD>>>(c->bp, p32, i32, l32, i64, l64);
        CKL("init_td_kernel");
        CK(cudaMemcpyToSymbol(c_td_p, p32, MAX_TD * 4, 0, cudaMemcpyDeviceToDevice));
        CK(cudaMemcpyToSymbol(c_td_inv32, i32, MAX_TD * 4, 0, cudaMemcpyDeviceToDevice));
        CK(cudaMemcpyToSymbol(c_td_lim32, l32, MAX_TD * 4, 0, cudaMemcpyDeviceToDevice));
        CK(cudaMemcpyToSymbol(c_td_inv64, i64, MAX_TD * 8, 0, cudaMemcpyDeviceToDevice));
        CK(cudaMemcpyToSymbol(c_td_lim64, l64, MAX_TD * 8, 0, cudaMemcpyDeviceToDevice));
        CK(cudaDeviceSynchronize());
        cudaFree(p32); cudaFree(i32); cudaFree(l32); cudaFree(i64); cudaFree(l64);
    }
    CK(cudaMalloc(&c->patt, (size_t)PRESIEVE_COPIES * PRESIEVE_LEN));
    init_presieve_kernel<<<256, 256>>>(c->patt);
    CKL("init_presieve_kernel");
    const size_t words = (size_t)(g_opt.sieve_max >> 6) + 1;
    CK(cudaMalloc(&c->bitmap, words * 4));
    CK(cudaMalloc(&c->plan, sizeof(DevPlan)));
    CK(cudaMemset(c->plan, 0, sizeof(DevPlan)));
    CK(cudaMalloc(&c->segh, (size_t)MAX_SEG * 65 * sizeof(unsigned int)));
    c->q.segh = c->segh;
    CK(cudaFuncSetAttribute(sieve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SEG_ODD));
    CK(cudaFuncSetAttribute(dense_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * SEG_ODD));
    CK(cudaFuncSetAttribute(dense2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * SEG_ODD));
    c->grid_sieve = c->sms * occupancy((const void*)sieve_kernel, SIEVE_THREADS, SEG_ODD);
    CK(cudaFuncSetAttribute((const void*)classify_kernel<24, 24>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)sizeof(ClsSmem)));
    c->grid_cls = c->sms * occupancy((const void*)classify_kernel<24, 24>, CLS_THREADS, sizeof(ClsSmem));
    if (c->grid_cls > MAX_SEG) c->grid_cls = MAX_SEG;  // one queue segment per classify block
    c->grid_mr1 = c->sms * occupancy((const void*)mr1_kernel, MR1_THREADS, 0);
    c->grid_sort = c->sms * occupancy((const void*)qscatter_kernel, SORT_THREADS, 0);
    mr2_attr(mr2_kernel<2, false, 3>);
    c->grid_mr2 = c->sms * occupancy((const void*)mr2_kernel<2, false, 3>, MR_THREADS, MR2_DYN_SMEM);
    CK(cudaEventCreateWithFlags(&c->last_done, cudaEventDisableTiming));
    for (int k = 0; k < 2; k++) {
        CK(cudaStreamCreateWithFlags(&c->hs[k], cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&c->ev_h2d[k], cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&c->ev_d2h[k], cudaEventDisableTiming));
    }
    CK(cudaDeviceSynchronize());
    return ISP_OK;
}

int get_ctx(Ctx** out) {
    read_env_once();
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        g_err = "no CUDA device";
        return ISP_ENODEV;
    }
    int dev = 0;
    CK(cudaGetDevice(&dev));
    if ((int)g_ctx.size() <= dev) g_ctx.resize(dev + 1, nullptr);
    if (!g_ctx[dev]) {
        Ctx* c = new Ctx();
        int rc = init_ctx(c);
        if (rc != ISP_OK) { delete c; return rc; }
        g_ctx[dev] = c;
    }
    *out = g_ctx[dev];
    return ISP_OK;
}

// Scratch queues for a chunk: two uint32 arrays of `cap` entries (8 bytes per
// element of the chunk, kernels.cuh Queues), allocated lazily and kept.
int ensure_queues(Ctx* c, size_t cap) {
    if (cap <= c->qcap) return ISP_OK;
    if (c->qmem) { CK(cudaFree(c->qmem)); c->qmem = nullptr; c->qcap = 0; }
    cap = (cap + 4095) & ~(size_t)4095;
    const size_t bytes = cap * 8;
    if (cudaMalloc(&c->qmem, bytes) != cudaSuccess) {
        cudaGetLastError();
        g_err = "queue allocation of " + std::to_string(bytes) + " bytes failed";
        return ISP_ENOMEM;
    }
    c->q.q = reinterpret_cast<uint32_t*>(c->qmem);
    c->q.s = reinterpret_cast<uint32_t*>(c->qmem) + cap;
    c->q.cap = (unsigned int)cap;
    c->q.segh = c->segh;
    c->qcap = cap;
    return ISP_OK;
}

#if ISP_CHECKS
// Checked builds (-DISP_CHECKS=1, tools/build_checked.py): wait for the call
// and turn a failed device-side bounds check into ISP_ECUDA.
int check_device(cudaStream_t s) {
    CK(cudaStreamSynchronize(s));
    unsigned int id = 0;
    CK(cudaMemcpyFromSymbol(&id, g_isp_check, sizeof(id)));
    if (id) {
        const unsigned int zero = 0;
        CK(cudaMemcpyToSymbol(g_isp_check, &zero, sizeof(zero)));
        g_err = "device bounds check " + std::to_string(id) + " failed";
        return ISP_ECUDA;
    }
    return ISP_OK;
}
#endif

// Persistent MR grids never need more blocks than the chunk could queue.
int mr_grid(int full, uint32_t len) {
    // dynamic chunks of MR_CHUNK entries: more warps than len / MR_CHUNK would
    // only contend on the work cursors
    const uint32_t need = (len + MR_THREADS * 8 - 1) / (MR_THREADS * 8);
    return (int)(need < (uint32_t)full ? need : (uint32_t)full);
}

bool overlaps(const void* a, size_t an, const void* b, size_t bn) {
    const uintptr_t a0 = (uintptr_t)a, b0 = (uintptr_t)b;
    return a0 < b0 + bn && b0 < a0 + an;
}

// Trial-division prime counts available as compile-time constants (the
// constant-bank operands then sit in the IMAD instructions themselves).
int td_round(int v) { return v >= 32 ? 32 : v >= 24 ? 24 : v >= 16 ? 16 : v >= 8 ? 8 : 0; }

template <typename K>
void launch_cls(K k, int g, cudaStream_t s, const unsigned long long* N, uint8_t* out, uint32_t len, Ctx* c,
                const TDParams& td, int vin, int vout, uint32_t ss) {
    cudaFuncSetAttribute((const void*)k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(ClsSmem));
    FzParams fz;
    fz.bits = g_opt.fuse_bits;
    fz.p2 = (g_opt.witness == 2 && g_opt.bases32 != 7) ? 2 : g_opt.bases32 == 7 ? 1 : 0;
    fz.wit = g_opt.witness;
    fz.gon = g_gon;
    fz.gh_tail = g_gh_tail;
    launch_k(k, g, CLS_THREADS, sizeof(ClsSmem), s, N, out, len, c->plan, c->bitmap, c->q, td, vin, vout, ss, fz);
}

template <int A>
void launch_classify_b(int n64, int g, cudaStream_t s, const unsigned long long* N, uint8_t* out, uint32_t len,
                       Ctx* c, const TDParams& td, int vin, int vout, uint32_t ss) {
    switch (n64) {
        case 32: launch_cls(classify_kernel<A, 32>, g, s, N, out, len, c, td, vin, vout, ss); break;
        case 24: launch_cls(classify_kernel<A, 24>, g, s, N, out, len, c, td, vin, vout, ss); break;
        case 16: launch_cls(classify_kernel<A, 16>, g, s, N, out, len, c, td, vin, vout, ss); break;
        case 8: launch_cls(classify_kernel<A, 8>, g, s, N, out, len, c, td, vin, vout, ss); break;
        default: launch_cls(classify_kernel<A, 0>, g, s, N, out, len, c, td, vin, vout, ss); break;
    }
}

void launch_classify(int n32, int n64, int g, cudaStream_t s, const unsigned long long* N, uint8_t* out,
                     uint32_t len, Ctx* c, const TDParams& td, int vin, int vout, uint32_t ss) {
    if (g_opt.count_work && n32 == kTD32Default && n64 == 32) {  // the work-counting instantiation (default TD only)
        launch_cls(classify_kernel<kTD32Default, 32, true>, g, s, N, out, len, c, td, vin, vout, ss);
        return;
    }
    switch (n32) {
        case 32: launch_classify_b<32>(n64, g, s, N, out, len, c, td, vin, vout, ss); break;
        case 24: launch_classify_b<24>(n64, g, s, N, out, len, c, td, vin, vout, ss); break;
        case 16: launch_classify_b<16>(n64, g, s, N, out, len, c, td, vin, vout, ss); break;
        case 8: launch_classify_b<8>(n64, g, s, N, out, len, c, td, vin, vout, ss); break;
        default: launch_classify_b<0>(n64, g, s, N, out, len, c, td, vin, vout, ss); break;
    }
}

template <int WIN, int G>
void launch_mr2_w(Ctx* c, cudaStream_t s, const unsigned long long* N, uint8_t* out, uint32_t len, int grid, bool full,
                  int cw) {
    if (full) {
        mr2_attr(mr2_kernel<WIN, true, G>);
        launch_k(mr2_kernel<WIN, true, G>, grid, MR_THREADS, MR2_DYN_SMEM, s, c->plan, c->q, N, out, len, cw, g_opt.sched);
    } else {
        mr2_attr(mr2_kernel<WIN, false, G>);
        launch_k(mr2_kernel<WIN, false, G>, grid, MR_THREADS, MR2_DYN_SMEM, s, c->plan, c->q, N, out, len, cw, g_opt.sched);
    }
}

int launch_mr2(Ctx* c, cudaStream_t s, const unsigned long long* N, uint8_t* out, uint32_t len, int grid) {
    const bool full = g_opt.bases32 == 7;
    const int cw = g_opt.count_work;
    const int g = g_opt.mr2_group == 6 ? 6 : 3;
    if (g_opt.witness == 1) {  // Baillie-PSW for the 64-bit Montgomery class
        mr2_attr(mr2_kernel<3, true, 3, 1>);
        mr2_attr(mr2_kernel<3, false, 3, 1>);
        if (full) launch_k(mr2_kernel<3, true, 3, 1>, grid, MR_THREADS, MR2_DYN_SMEM, s, c->plan, c->q, N, out, len, cw, g_opt.sched);
        else launch_k(mr2_kernel<3, false, 3, 1>, grid, MR_THREADS, MR2_DYN_SMEM, s, c->plan, c->q, N, out, len, cw, g_opt.sched);
        CKL("mr2_kernel");
        return ISP_OK;
    }
    if (g_opt.witness == 2) {  // reduced witness sets by magnitude
        mr2_attr(mr2_kernel<3, true, 3, 2>);
        mr2_attr(mr2_kernel<3, false, 3, 2>);
        if (full) launch_k(mr2_kernel<3, true, 3, 2>, grid, MR_THREADS, MR2_DYN_SMEM, s, c->plan, c->q, N, out, len, cw, g_opt.sched);
        else launch_k(mr2_kernel<3, false, 3, 2>, grid, MR_THREADS, MR2_DYN_SMEM, s, c->plan, c->q, N, out, len, cw, g_opt.sched);
        CKL("mr2_kernel");
        return ISP_OK;
    }
    switch (g_opt.win64 * 10 + g) {
        case 13: launch_mr2_w<1, 3>(c, s, N, out, len, grid, full, cw); break;
        case 16: launch_mr2_w<1, 6>(c, s, N, out, len, grid, full, cw); break;
        case 23: launch_mr2_w<2, 3>(c, s, N, out, len, grid, full, cw); break;
        case 26: launch_mr2_w<2, 6>(c, s, N, out, len, grid, full, cw); break;
        case 33: launch_mr2_w<3, 3>(c, s, N, out, len, grid, full, cw); break;
        default: launch_mr2_w<3, 6>(c, s, N, out, len, grid, full, cw); break;
    }
    CKL("mr2_kernel");
    return ISP_OK;
}

// Graph capture of the pipeline (option "graph"): the capture stream and the
// graph being built.  nullptr: plain stream launches.
struct GBuild { cudaGraph_t g; cudaStream_t s2; };

// One stage of the pipeline that may find nothing to do.  Plain launches: the
// stage's kernels are enqueued on s (each exits at once when the plan says so).
// Graph capture: the stage becomes the body of an IF conditional node on handle
// h, which the plan or classify kernel sets on the device, so an empty stage
// costs no launch at all.  The kernel after a conditional node has no
// programmatic (PDL) edge to it.
template <typename F>
int cond_stage(GBuild* gb, cudaStream_t s, cudaGraphConditionalHandle h, F&& body) {
    if (!gb) return body(s);
    const cudaGraphNode_t* deps = nullptr;
    size_t nd = 0;
    cudaStreamCaptureStatus st;
    CK(cudaStreamGetCaptureInfo(s, &st, nullptr, nullptr, &deps, &nd));
    cudaGraphNodeParams np = {};
    np.type = cudaGraphNodeTypeConditional;
    np.conditional.handle = h;
    np.conditional.type = cudaGraphCondTypeIf;
    np.conditional.size = 1;
    cudaGraphNode_t node;
    CK(cudaGraphAddNode(&node, gb->g, deps, nd, &np));
    CK(cudaStreamUpdateCaptureDependencies(s, &node, 1, cudaStreamSetCaptureDependencies));
    CK(cudaStreamBeginCaptureToGraph(gb->s2, np.conditional.phGraph_out[0], nullptr, nullptr, 0,
                                     cudaStreamCaptureModeRelaxed));
    g_pdl_ok = false;
    const int rc = body(gb->s2);
    cudaGraph_t bg = nullptr;
    const cudaError_t e = cudaStreamEndCapture(gb->s2, &bg);
    g_pdl_ok = false;
    if (rc != ISP_OK) return rc;
    if (e != cudaSuccess) return cuda_fail(e, "cudaStreamEndCapture (conditional stage)");
    return ISP_OK;
}

// The pipeline stages of every device chunk of dN[0..n), on s (or captured
// into gb's graph).
int enqueue_chunks(Ctx* c, const unsigned long long* dN, uint8_t* dout, size_t n, size_t chunk, PlanParams P,
                   const TDParams& td, cudaStream_t s, GBuild* gb) {
    int rc = ISP_OK;
    for (size_t base = 0; base < n; base += chunk) {
        const uint32_t len = (uint32_t)((n - base) < chunk ? (n - base) : chunk);
        const unsigned long long* N = dN + base;
        uint8_t* out = dout + base;
        P.invalidate = (base == 0 && !g_opt.sieve_cache) ? 1 : 0;
        cudaGraphConditionalHandle gh[4] = {0, 0, 0, 0};  // sieve, dense stride 1, dense stride 2, tail
        if (gb)
            for (int k = 0; k < 4; k++) CK(cudaGraphConditionalHandleCreate(&gh[k], gb->g, 0u, cudaGraphCondAssignDefault));
        P.gon = gb ? 1 : 0;
        for (int k = 0; k < 3; k++) P.gh[k] = (unsigned long long)gh[k];
        g_gon = gb ? 1 : 0;
        g_gh_tail = (unsigned long long)gh[3];
        {
            KScope ks(K_PLAN, s);
            launch_k(plan_kernel, 1, PLAN_THREADS, 0, s, N, (unsigned long long)len, c->plan, P);
            CKL("plan_kernel");
        }
        // first base prime >= warp_p (the warp-cooperative / per-thread split)
        int first_large = FIRST_CROSS_PRIME_IDX;
        while (first_large < c->nbp && c->hbp[first_large].x < (uint32_t)g_opt.warp_p) first_large++;
        rc = cond_stage(gb, s, gh[0], [&](cudaStream_t st) -> int {
            KScope ks(K_SIEVE, st);
            launch_k(sieve_kernel, c->grid_sieve, SIEVE_THREADS, SEG_ODD, st, c->plan, c->bitmap, c->bp, c->nbp, c->patt,
                     first_large);
            CKL("sieve_kernel");
            return ISP_OK;
        });
        if (rc != ISP_OK) return rc;
        {
            // 16-byte loads of element pairs need N 16-B aligned and out 2-B aligned
            const int vec = ((((uintptr_t)N & 15) == 0) && (((uintptr_t)out & 1) == 0)) ? 1 : 0;
            rc = cond_stage(gb, s, gh[1], [&](cudaStream_t st) -> int {
                KScope ks(K_DENSE, st);
                launch_k(dense_kernel, c->sms, DENSE_THREADS, 2 * SEG_ODD, st, c->plan, N, out, len, c->bp, c->nbp,
                         c->patt, first_large, vec);
                CKL("dense_kernel");
                return ISP_OK;
            });
            if (rc != ISP_OK) return rc;
            rc = cond_stage(gb, s, gh[2], [&](cudaStream_t st) -> int {
                KScope ks(K_DENSE, st);
                launch_k(dense2_kernel, c->sms, DENSE_THREADS, 2 * SEG_ODD, st, c->plan, N, out, len, c->bp, c->nbp,
                         c->patt, first_large, vec);
                CKL("dense2_kernel");
                return ISP_OK;
            });
            if (rc != ISP_OK) return rc;
        }
        const uint32_t ntiles = (len + CLS_TILE - 1) / CLS_TILE;
        const int gcls = (int)(ntiles < (uint32_t)c->grid_cls ? ntiles : (uint32_t)c->grid_cls);
        // block b of classify owns queue entries [b * seg_stride, (b + 1) * seg_stride):
        // at most ceil(ntiles / gcls) tiles of CLS_TILE elements each
        const uint32_t seg_stride = ((ntiles + gcls - 1) / gcls) * CLS_TILE;
        const int vin = (((uintptr_t)N & 15) == 0) ? 1 : 0;
        const int vout = (((uintptr_t)out & 7) == 0) ? 1 : 0;
        {
            KScope ks(K_CLASSIFY, s);
            launch_classify(td.n32, td.n64, gcls, s, N, out, len, c, td, vin, vout, seg_stride);
            CKL("classify_kernel");
        }
        // the sort and the witness kernels, when classify queued anything
        rc = cond_stage(gb, s, gh[3], [&](cudaStream_t st) -> int {
            {
                KScope ks(K_SORT, st);
                launch_k(qscatter_kernel, gcls, SORT_THREADS, 0, st, c->plan, c->q, gcls, seg_stride);  // one block per segment
                CKL("qscatter_kernel");
            }
            {
                KScope ks(K_MR1, st);
                launch_k(mr1_kernel, mr_grid(c->grid_mr1, len), MR1_THREADS, 0, st, c->plan, c->q, N, len,
                         g_opt.count_work, g_opt.sched);
                CKL("mr1_kernel");
            }
            KScope ks(K_MR2, st);
            return launch_mr2(c, st, N, out, len, mr_grid(c->grid_mr2, len));
        });
        if (rc != ISP_OK) return rc;
    }
    g_gon = 0;
    return ISP_OK;
}

// Replay (or capture, instantiate and cache) the graph of this call's pipeline.
int graph_launch(Ctx* c, const unsigned long long* dN, uint8_t* dout, size_t n, size_t chunk, const PlanParams& P,
                 const TDParams& td, cudaStream_t s) {
    for (auto& g : c->graphs) {
        if (g.N == dN && g.out == dout && g.n == n && g.epoch == g_opt_epoch && g.qmem == c->qmem && g.qcap == c->qcap) {
            g.used = ++c->graph_clock;
            CK(cudaGraphLaunch(g.exec, s));
            return ISP_OK;
        }
    }
    if (!c->gs) {
        CK(cudaStreamCreateWithFlags(&c->gs, cudaStreamNonBlocking));
        CK(cudaStreamCreateWithFlags(&c->gs2, cudaStreamNonBlocking));
    }
    GBuild gb;
    gb.s2 = c->gs2;
    CK(cudaStreamBeginCapture(c->gs, cudaStreamCaptureModeRelaxed));
    cudaStreamCaptureStatus st;
    cudaError_t e = cudaStreamGetCaptureInfo(c->gs, &st, nullptr, &gb.g, nullptr, nullptr);
    g_pdl_ok = false;
    int rc = e == cudaSuccess ? enqueue_chunks(c, dN, dout, n, chunk, P, td, c->gs, &gb) : cuda_fail(e, "cudaStreamGetCaptureInfo");
    g_gon = 0;
    g_pdl_ok = true;
    cudaGraph_t graph = nullptr;
    e = cudaStreamEndCapture(c->gs, &graph);
    if (rc != ISP_OK) {
        if (graph) cudaGraphDestroy(graph);
        return rc;
    }
    if (e != cudaSuccess) return cuda_fail(e, "cudaStreamEndCapture");
    cudaGraphExec_t exec = nullptr;
    e = cudaGraphInstantiate(&exec, graph, 0);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGraphInstantiate");
    if (c->graphs.size() >= 8) {
        size_t lru = 0;
        for (size_t k = 1; k < c->graphs.size(); k++)
            if (c->graphs[k].used < c->graphs[lru].used) lru = k;
        if (c->has_last) CK(cudaEventSynchronize(c->last_done));
        cudaGraphExecDestroy(c->graphs[lru].exec);
        c->graphs.erase(c->graphs.begin() + (long)lru);
    }
    c->graphs.push_back({dN, dout, n, g_opt_epoch, c->qmem, c->qcap, exec, ++c->graph_clock});
    CK(cudaGraphLaunch(exec, s));
    return ISP_OK;
}

// The whole hot path for dN[0..n) on stream s.  Caller holds g_mu.
int device_impl(Ctx* c, const unsigned long long* dN, uint8_t* dout, size_t n, cudaStream_t s) {
    size_t chunk = (size_t)1 << g_opt.chunk_log2;
    // packed queue entries hold the tile number within a classify block in
    // 13 bits (kernels.cuh QE_MAX_TILES)
    while (chunk > ((size_t)1 << 16) && (chunk / CLS_TILE + c->grid_cls - 1) / c->grid_cls > QE_MAX_TILES) chunk >>= 1;
    // classify's per-block queue segments need up to one tile of slack per block;
    // when the device cannot hold the queues of a full chunk, halve the chunk
    int rc;
    for (;;) {
        rc = ensure_queues(c, (n < chunk ? n : chunk) + (size_t)c->grid_cls * CLS_TILE);
        if (rc != ISP_ENOMEM || chunk <= ((size_t)1 << 24) || n <= ((size_t)1 << 24)) break;
        chunk >>= 1;
    }
    if (rc != ISP_OK) return rc;
    if (c->has_last && c->last_stream != (void*)s) CK(cudaStreamWaitEvent(s, c->last_done, 0));
    PlanParams P;
    P.force = g_opt.force_path;
    P.wmax = g_opt.sieve_max;
    P.sieve_ps_per_int = (float)g_opt.sieve_fs_per_int * 1e-3f;
    P.sieve_fixed_ps = (float)g_opt.sieve_fixed_ns * 1e3f;
    P.mr32_ps_per_bit = (float)g_opt.mr32_fs_per_bit * 1e-3f;
    P.mr_fixed_ps = (float)g_opt.mr_fixed_ns * 1e3f;
    TDParams td;
    td.n32 = td_round(g_opt.td32);
    td.n64 = td_round(g_opt.td64);
    {
        const unsigned long long pn = c->hbp[td.n32].x;  // first prime not trial-divided
        const unsigned long long sq = pn * pn;
        td.sq32 = sq > 0xFFFFFFFFull ? 0xFFFFFFFFu : (uint32_t)sq;
        td.rnd = 6755399441055744.0;  // 1.5 * 2^52
    }
    if ((long long)n <= g_opt.small_max && n <= 0xFFFFFFFFull && g_opt.force_path == 0) {
        // short array: one fused launch (small_kernel), latency instead of pipeline stages
        const uint32_t len = (uint32_t)n;
        {
            KScope ks(K_SMALL, s);
            if ((long long)len <= g_opt.warp_max) {  // one warp per element, one base per lane
                const unsigned blocks = (unsigned)(((size_t)len * 32 + 255) / 256);
                if (g_opt.bases32 == 7) small_warp_kernel<true><<<blocks, 256, 0, s>>>(dN, dout, len, td);
                else small_warp_kernel<false><<<blocks, 256, 0, s>>>(dN, dout, len, td);
            } else if (g_opt.small_sieve) {
                // cluster sieve of [0, 2^20) + gather; the grid is a whole number of clusters
                const unsigned blocks = (unsigned)((((size_t)len + SSV_ELEMS - 1) / SSV_ELEMS + SSV_CLUSTER - 1) /
                                                   SSV_CLUSTER * SSV_CLUSTER);
                int first_large = FIRST_CROSS_PRIME_IDX;
                while (first_large < c->nbp && c->hbp[first_large].x < (uint32_t)g_opt.warp_p) first_large++;
                cudaLaunchConfig_t cfg = {};
                cfg.gridDim = dim3(blocks);
                cfg.blockDim = dim3(SSV_THREADS);
                cfg.dynamicSmemBytes = sizeof(SsvSmem);
                cfg.stream = s;
                cudaLaunchAttribute at[1];
                at[0].id = cudaLaunchAttributeClusterDimension;
                at[0].val.clusterDim.x = SSV_CLUSTER;
                at[0].val.clusterDim.y = 1;
                at[0].val.clusterDim.z = 1;
                cfg.attrs = at;
                cfg.numAttrs = 1;
                if (SSV_CLUSTER > 8) {
                    cudaFuncSetAttribute((const void*)small_sieve_kernel<true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
                    cudaFuncSetAttribute((const void*)small_sieve_kernel<false>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
                }
                if (g_opt.bases32 == 7) {
                    cudaFuncSetAttribute((const void*)small_sieve_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)sizeof(SsvSmem));
                    cudaLaunchKernelEx(&cfg, small_sieve_kernel<true>, dN, dout, len, td, (const uint2*)c->bp, c->nbp,
                                       (const uint8_t*)c->patt, first_large);
                } else {
                    cudaFuncSetAttribute((const void*)small_sieve_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)sizeof(SsvSmem));
                    cudaLaunchKernelEx(&cfg, small_sieve_kernel<false>, dN, dout, len, td, (const uint2*)c->bp, c->nbp,
                                       (const uint8_t*)c->patt, first_large);
                }
            } else if (g_opt.bases32 == 7) {
                small_kernel<true><<<(len + 255) / 256, 256, 0, s>>>(dN, dout, len, td);
            } else {
                small_kernel<false><<<(len + 255) / 256, 256, 0, s>>>(dN, dout, len, td);
            }
            CKL("small_kernel");
        }
        CK(cudaEventRecord(c->last_done, s));
        c->has_last = true;
        c->last_stream = (void*)s;
#if ISP_CHECKS
        return check_device(s);
#else
        return ISP_OK;
#endif
    }
    if (g_opt.graph && !g_opt.kernel_timing && !ISP_CHECKS) {
        rc = graph_launch(c, dN, dout, n, chunk, P, td, s);
        if (rc != ISP_OK) return rc;
    } else {
        rc = enqueue_chunks(c, dN, dout, n, chunk, P, td, s, nullptr);
        if (rc != ISP_OK) return rc;
    }
#if ISP_CHECKS
    rc = check_device(s);
    if (rc != ISP_OK) return rc;
#endif
    CK(cudaEventRecord(c->last_done, s));
    c->has_last = true;
    c->last_stream = (void*)s;
    return ISP_OK;
}

int ensure_staging(Ctx* c, size_t cap, bool need_hin, bool need_hout) {
    if (cap > c->hcap) {
        for (int k = 0; k < 2; k++) {
            if (c->din[k]) cudaFree(c->din[k]);
            if (c->dout[k]) cudaFree(c->dout[k]);
            if (c->hin[k]) cudaFreeHost(c->hin[k]);
            if (c->hout[k]) cudaFreeHost(c->hout[k]);
            c->din[k] = nullptr; c->dout[k] = nullptr; c->hin[k] = nullptr; c->hout[k] = nullptr;
        }
        c->hcap = 0;
        for (int k = 0; k < 2; k++) {
            if (cudaMalloc(&c->din[k], cap * 8) != cudaSuccess || cudaMalloc(&c->dout[k], cap) != cudaSuccess) {
                cudaGetLastError();
                g_err = "staging allocation failed";
                return ISP_ENOMEM;
            }
        }
        c->hcap = cap;
    }
    for (int k = 0; k < 2; k++) {
        if (need_hin && !c->hin[k] && cudaMallocHost(&c->hin[k], c->hcap * 8) != cudaSuccess) {
            cudaGetLastError(); g_err = "pinned allocation failed"; return ISP_ENOMEM;
        }
        if (need_hout && !c->hout[k] && cudaMallocHost(&c->hout[k], c->hcap) != cudaSuccess) {
            cudaGetLastError(); g_err = "pinned allocation failed"; return ISP_ENOMEM;
        }
    }
    return ISP_OK;
}

bool is_pinned(const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) { cudaGetLastError(); return false; }
    return a.type == cudaMemoryTypeHost;
}

}  // namespace

extern "C" {

int isprime_device(const uint64_t* dN, uint8_t* dout, size_t n, void* stream) {
    if (n == 0) return ISP_OK;
    if (!dN || !dout) return ISP_EINVAL;
    if (overlaps(dN, n * 8, dout, n)) return ISP_EINVAL;
    std::lock_guard<std::mutex> lk(g_mu);
    Ctx* c = nullptr;
    int rc = get_ctx(&c);
    if (rc != ISP_OK) return rc;
    return device_impl(c, reinterpret_cast<const unsigned long long*>(dN), dout, n, (cudaStream_t)stream);
}

int isprime_popcount_device(const uint8_t* dout, size_t n, uint64_t* dcount, void* stream) {
    if (!dcount) return ISP_EINVAL;
    if (n > 0 && !dout) return ISP_EINVAL;
    std::lock_guard<std::mutex> lk(g_mu);
    Ctx* c = nullptr;
    int rc = get_ctx(&c);
    if (rc != ISP_OK) return rc;
    cudaStream_t s = (cudaStream_t)stream;
    CK(cudaMemsetAsync(dcount, 0, 8, s));
    if (n == 0) return ISP_OK;
    KScope ks(K_POPCOUNT, s);
    popcount_kernel<<<c->sms * 4, 256, 0, s>>>(dout, n, reinterpret_cast<unsigned long long*>(dcount));
    CKL("popcount_kernel");
    return ISP_OK;
}

int isprime_count_device(const uint64_t* dN, uint8_t* dout, size_t n, uint64_t* dcount, void* stream) {
    int rc = isprime_device(dN, dout, n, stream);
    if (rc != ISP_OK) return rc;
    return isprime_popcount_device(dout, n, dcount, stream);
}

int isprime(const uint64_t* N, uint8_t* out, size_t n) {
    if (n == 0) return ISP_OK;
    if (!N || !out) return ISP_EINVAL;
    if (overlaps(N, n * 8, out, n)) return ISP_EINVAL;
    std::lock_guard<std::mutex> lk(g_mu);
    Ctx* c = nullptr;
    int rc = get_ctx(&c);
    if (rc != ISP_OK) return rc;
    const bool in_pinned = is_pinned(N);
    const bool out_pinned = is_pinned(out);
    const size_t hchunk = n < ((size_t)1 << 24) ? n : ((size_t)1 << 24);
    rc = ensure_staging(c, hchunk, !in_pinned, !out_pinned);
    if (rc != ISP_OK) return rc;
    size_t pend_base[2] = {0, 0}, pend_len[2] = {0, 0};
    int ci = 0;
    for (size_t base = 0; base < n; base += hchunk, ci++) {
        const int k = ci & 1;
        cudaStream_t s = c->hs[k];
        const size_t len = (n - base) < hchunk ? (n - base) : hchunk;
        const void* src = N + base;
        if (!in_pinned) {
            CK(cudaEventSynchronize(c->ev_h2d[k]));  // slot's previous upload finished
            memcpy(c->hin[k], N + base, len * 8);
            src = c->hin[k];
        }
        CK(cudaMemcpyAsync(c->din[k], src, len * 8, cudaMemcpyHostToDevice, s));
        CK(cudaEventRecord(c->ev_h2d[k], s));
        rc = device_impl(c, c->din[k], c->dout[k], len, s);
        if (rc != ISP_OK) return rc;
        if (!out_pinned) {
            CK(cudaEventSynchronize(c->ev_d2h[k]));
            if (pend_len[k]) memcpy(out + pend_base[k], c->hout[k], pend_len[k]);
            pend_len[k] = 0;
            CK(cudaMemcpyAsync(c->hout[k], c->dout[k], len, cudaMemcpyDeviceToHost, s));
            pend_base[k] = base;
            pend_len[k] = len;
        } else {
            CK(cudaMemcpyAsync(out + base, c->dout[k], len, cudaMemcpyDeviceToHost, s));
        }
        CK(cudaEventRecord(c->ev_d2h[k], s));
    }
    for (int k = 0; k < 2; k++) {
        CK(cudaStreamSynchronize(c->hs[k]));
        if (pend_len[k]) memcpy(out + pend_base[k], c->hout[k], pend_len[k]);
    }
    return ISP_OK;
}

const char* isprime_strerror(int status) {
    static thread_local std::string msg;
    switch (status) {
        case ISP_OK: msg = "ok"; break;
        case ISP_EINVAL: msg = "invalid argument (NULL pointer with n > 0, overlapping buffers, or bad option)"; break;
        case ISP_ENOMEM: msg = "out of memory: " + g_err; break;
        case ISP_ECUDA: msg = "CUDA error: " + g_err; break;
        case ISP_ENODEV: msg = "no CUDA device"; break;
        default: msg = "unknown status"; break;
    }
    return msg.c_str();
}

void isprime_shutdown(void) {
    std::lock_guard<std::mutex> lk(g_mu);
    int cur = 0;
    cudaGetDevice(&cur);
    for (size_t d = 0; d < g_ctx.size(); d++) {
        Ctx* c = g_ctx[d];
        if (!c) continue;
        cudaSetDevice((int)d);
        cudaDeviceSynchronize();
        cudaFree(c->bp); cudaFree(c->patt); cudaFree(c->bitmap); cudaFree(c->plan); cudaFree(c->segh);
        if (c->qmem) cudaFree(c->qmem);
        for (int k = 0; k < 2; k++) {
            if (c->din[k]) cudaFree(c->din[k]);
            if (c->dout[k]) cudaFree(c->dout[k]);
            if (c->hin[k]) cudaFreeHost(c->hin[k]);
            if (c->hout[k]) cudaFreeHost(c->hout[k]);
            if (c->hs[k]) cudaStreamDestroy(c->hs[k]);
            if (c->ev_h2d[k]) cudaEventDestroy(c->ev_h2d[k]);
            if (c->ev_d2h[k]) cudaEventDestroy(c->ev_d2h[k]);
        }
        if (c->last_done) cudaEventDestroy(c->last_done);
        for (auto& g : c->graphs) cudaGraphExecDestroy(g.exec);
        if (c->gs) cudaStreamDestroy(c->gs);
        if (c->gs2) cudaStreamDestroy(c->gs2);
        delete c;
        g_ctx[d] = nullptr;
    }
    cudaSetDevice(cur);
}

int isprime_set_option(const char* key, long long v) {
    if (!key) return ISP_EINVAL;
    std::lock_guard<std::mutex> lk(g_mu);
    read_env_once();
    if (!strcmp(key, "force_path")) { if (v < 0 || v > 2) return ISP_EINVAL; g_opt.force_path = (int)v; }
    else if (!strcmp(key, "bases32")) { if (v != 3 && v != 7) return ISP_EINVAL; g_opt.bases32 = (int)v; }
    else if (!strcmp(key, "td_primes32")) { if (v < 0 || v > MAX_TD) return ISP_EINVAL; g_opt.td32 = (int)v; }
    else if (!strcmp(key, "td_primes64")) { if (v < 0 || v > MAX_TD) return ISP_EINVAL; g_opt.td64 = (int)v; }
    else if (!strcmp(key, "chunk_log2")) { if (v < 16 || v > 31) return ISP_EINVAL; g_opt.chunk_log2 = (int)v; }
    else if (!strcmp(key, "win64")) { if (v < 1 || v > 3) return ISP_EINVAL; g_opt.win64 = (int)v; }
    else if (!strcmp(key, "warp_p")) { if (v < 17 || v > 65536) return ISP_EINVAL; g_opt.warp_p = (int)v; }
    else if (!strcmp(key, "sieve_fs_per_int")) { if (v < 0) return ISP_EINVAL; g_opt.sieve_fs_per_int = v; }
    else if (!strcmp(key, "sieve_fixed_ns")) { if (v < 0) return ISP_EINVAL; g_opt.sieve_fixed_ns = v; }
    else if (!strcmp(key, "mr32_fs_per_bit")) { if (v < 0) return ISP_EINVAL; g_opt.mr32_fs_per_bit = v; }
    else if (!strcmp(key, "mr_fixed_ns")) { if (v < 0) return ISP_EINVAL; g_opt.mr_fixed_ns = v; }
    else if (!strcmp(key, "kernel_timing")) { if (v < 0 || v > 1) return ISP_EINVAL; g_opt.kernel_timing = (int)v; }
    else if (!strcmp(key, "count_work")) { if (v < 0 || v > 1) return ISP_EINVAL; g_opt.count_work = (int)v; }
    else if (!strcmp(key, "small_sieve")) { if (v < 0 || v > 1) return ISP_EINVAL; g_opt.small_sieve = (int)v; }
    else if (!strcmp(key, "mr2_group")) { if (v != 3 && v != 6) return ISP_EINVAL; g_opt.mr2_group = (int)v; }
    else if (!strcmp(key, "pdl")) { if (v < 0 || v > 1) return ISP_EINVAL; g_opt.pdl = (int)v; }
    else if (!strcmp(key, "sieve_cache")) { if (v < 0 || v > 1) return ISP_EINVAL; g_opt.sieve_cache = (int)v; }
    else if (!strcmp(key, "small_max")) { if (v < 0 || v > 0xFFFFFFFFll) return ISP_EINVAL; g_opt.small_max = v; }
    else if (!strcmp(key, "warp_max")) { if (v < 0 || v > (1 << 26)) return ISP_EINVAL; g_opt.warp_max = v; }
    else if (!strcmp(key, "witness")) { if (v < 0 || v > 2) return ISP_EINVAL; g_opt.witness = (int)v; }
    else if (!strcmp(key, "sched")) { if (v < 0 || v > 2) return ISP_EINVAL; g_opt.sched = (int)v; }
    else if (!strcmp(key, "fuse_bits")) { if (v != 0 && v != 32 && v != 51) return ISP_EINVAL; g_opt.fuse_bits = (int)v; }
    else if (!strcmp(key, "graph")) { if (v < 0 || v > 1) return ISP_EINVAL; g_opt.graph = (int)v; }
    else return ISP_EINVAL;
    g_opt_epoch++;
    return ISP_OK;
}

long long isprime_get_option(const char* key) {
    if (!key) return -1;
    std::lock_guard<std::mutex> lk(g_mu);
    read_env_once();
    if (!strcmp(key, "force_path")) return g_opt.force_path;
    if (!strcmp(key, "bases32")) return g_opt.bases32;
    if (!strcmp(key, "td_primes32")) return g_opt.td32;
    if (!strcmp(key, "td_primes64")) return g_opt.td64;
    if (!strcmp(key, "chunk_log2")) return g_opt.chunk_log2;
    if (!strcmp(key, "win64")) return g_opt.win64;
    if (!strcmp(key, "warp_p")) return g_opt.warp_p;
    if (!strcmp(key, "sieve_fs_per_int")) return g_opt.sieve_fs_per_int;
    if (!strcmp(key, "sieve_fixed_ns")) return g_opt.sieve_fixed_ns;
    if (!strcmp(key, "mr32_fs_per_bit")) return g_opt.mr32_fs_per_bit;
    if (!strcmp(key, "mr_fixed_ns")) return g_opt.mr_fixed_ns;
    if (!strcmp(key, "kernel_timing")) return g_opt.kernel_timing;
    if (!strcmp(key, "count_work")) return g_opt.count_work;
    if (!strcmp(key, "small_sieve")) return g_opt.small_sieve;
    if (!strcmp(key, "sieve_cache")) return g_opt.sieve_cache;
    if (!strcmp(key, "mr2_group")) return g_opt.mr2_group;
    if (!strcmp(key, "pdl")) return g_opt.pdl;
    if (!strcmp(key, "graph")) return g_opt.graph;
    if (!strcmp(key, "small_max")) return g_opt.small_max;
    if (!strcmp(key, "warp_max")) return g_opt.warp_max;
    if (!strcmp(key, "witness")) return g_opt.witness;
    if (!strcmp(key, "sched")) return g_opt.sched;
    if (!strcmp(key, "fuse_bits")) return g_opt.fuse_bits;
    return -1;
}

int isprime_get_stats(isprime_stats* st) {
    if (!st) return ISP_EINVAL;
    std::lock_guard<std::mutex> lk(g_mu);
    Ctx* c = nullptr;
    int rc = get_ctx(&c);
    if (rc != ISP_OK) return rc;
    CK(cudaDeviceSynchronize());
    DevPlan p;
    CK(cudaMemcpy(&p, c->plan, sizeof(p), cudaMemcpyDeviceToHost));
    st->window_lo = p.wlo;
    st->window_hi = p.whi;
    st->sieve_runs = p.sieve_runs;
    st->sieved_integers = p.sieved_ints;
    st->queued32 = p.total[0] + p.counts[0] + p.fzt[0];
    st->queued64 = p.total[1] + p.counts[1] + p.fzt[1];
    st->passed32 = p.total[2] + p.counts[2] + p.fzt[2];
    st->passed64 = p.total[3] + p.counts[3] + p.pf + p.fzt[3];
    st->chunks = p.chunks;
    st->kernel_launches = g_launches;
    for (int k = 0; k < 4; k++) st->mulmods[k] = p.work[k];
    st->mulmods_fp64[0] = p.work_f[0];
    st->mulmods_fp64[1] = p.work_f[1];
    st->mulmods_fused[0] = p.fzw[0];
    st->mulmods_fused[1] = p.fzw[1];
    return ISP_OK;
}

int isprime_reset_stats(void) {
    std::lock_guard<std::mutex> lk(g_mu);
    Ctx* c = nullptr;
    int rc = get_ctx(&c);
    if (rc != ISP_OK) return rc;
    CK(cudaDeviceSynchronize());
    DevPlan p;
    CK(cudaMemcpy(&p, c->plan, sizeof(p), cudaMemcpyDeviceToHost));
    for (int k = 0; k < 4; k++) { p.total[k] = 0; p.counts[k] = 0; p.fzt[k] = 0; }
    p.pf = 0;  // FP64-class base-2 passes of the last chunk (added to total[3] by the next plan)
    p.sieve_runs = 0;
    p.sieved_ints = 0;
    p.chunks = 0;
    for (int k = 0; k < 4; k++) p.work[k] = 0;
    p.work_f[0] = p.work_f[1] = 0;
    p.fzw[0] = p.fzw[1] = 0;
    p.valid_lo = p.valid_hi = 0;  // forget the bitmap: the next call sieves again
    CK(cudaMemcpy(c->plan, &p, sizeof(p), cudaMemcpyHostToDevice));
    g_launches = 0;
    return ISP_OK;
}

int isprime_get_kernel_times(isprime_kernel_time* out, int max, int* count) {
    std::lock_guard<std::mutex> lk(g_mu);
    kt_drain();
    if (count) *count = K_NUM;
    if (!out) return ISP_OK;
    for (int k = 0; k < K_NUM && k < max; k++) {
        memset(out[k].name, 0, sizeof(out[k].name));
        strncpy(out[k].name, k_names[k], sizeof(out[k].name) - 1);
        out[k].launches = g_kt_n[k];
        out[k].ms_total = g_kt_ms[k];
    }
    return ISP_OK;
}

int isprime_reset_kernel_times(void) {
    std::lock_guard<std::mutex> lk(g_mu);
    kt_drain();
    for (int k = 0; k < K_NUM; k++) { g_kt_ms[k] = 0; g_kt_n[k] = 0; }
    return ISP_OK;
}

int isprime_sprp_device(const uint64_t* dn, const uint64_t* da, uint8_t* dout, size_t count, void* stream) {
    if (count == 0) return ISP_OK;
    if (!dn || !da || !dout) return ISP_EINVAL;
    std::lock_guard<std::mutex> lk(g_mu);
    Ctx* c = nullptr;
    int rc = get_ctx(&c);
    if (rc != ISP_OK) return rc;
    const unsigned blocks = (unsigned)((count + 255) / 256);
    cudaStream_t s = (cudaStream_t)stream;
    const auto* n = reinterpret_cast<const unsigned long long*>(dn);
    const auto* a = reinterpret_cast<const unsigned long long*>(da);
    if (g_opt.win64 == 1) sprp_diag_kernel<1><<<blocks, 256, 0, s>>>(n, a, dout, count);
    else if (g_opt.win64 == 2) sprp_diag_kernel<2><<<blocks, 256, 0, s>>>(n, a, dout, count);
    else sprp_diag_kernel<3><<<blocks, 256, 0, s>>>(n, a, dout, count);
    CKL("sprp_diag_kernel");
    return ISP_OK;
}

int isprime_mulmod_device(const uint64_t* da, const uint64_t* db, const uint64_t* dm, uint64_t* dout, size_t count,
                          void* stream) {
    if (count == 0) return ISP_OK;
    if (!da || !db || !dm || !dout) return ISP_EINVAL;
    std::lock_guard<std::mutex> lk(g_mu);
    Ctx* c = nullptr;
    int rc = get_ctx(&c);
    if (rc != ISP_OK) return rc;
    const unsigned blocks = (unsigned)((count + 255) / 256);
    mulmod_diag_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(
        reinterpret_cast<const unsigned long long*>(da), reinterpret_cast<const unsigned long long*>(db),
        reinterpret_cast<const unsigned long long*>(dm), reinterpret_cast<unsigned long long*>(dout), count);
    CKL("mulmod_diag_kernel");
    return ISP_OK;
}

}  // extern "C"
