// eco_api.cu — the C ABI (include/eco_b200.h) over the sm_100a kernels.
//
// Host side only: argument checks, device buffers, launches, conversions
// between the caller's f64 tables (infeasible == j_inf) and the device's
// internal representation (Real, infeasible == +inf).  No CPU compute path.
#include <cuda_runtime.h>

#include <chrono>
#include <immintrin.h>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <algorithm>
#include <memory>
#include <functional>
#include <mutex>
#include <thread>
#include <stdexcept>
#include <vector>

#include <nccl.h>

#include "eco_kernels.cuh"
#include "eco_mpc.cuh"

using namespace eco;

namespace {

thread_local std::string g_err;

struct CudaError {
    cudaError_t e;
    const char* what;
};

#define ECO_CUDA(x)                                                      \
    do {                                                                 \
        cudaError_t e_ = (x);                                            \
        if (e_ != cudaSuccess) throw CudaError{e_, #x};                  \
    } while (0)

struct ArgError {
    std::string msg;
};

template <typename T>
struct DBuf {
    T* p = nullptr;
    size_t n = 0, cap = 0;
    DBuf() = default;
    explicit DBuf(size_t count) { alloc(count); }
    void alloc(size_t count) {
        free();
        n = cap = count;
        if (count) ECO_CUDA(cudaMalloc(&p, count * sizeof(T)));
    }
    // grow-only: keeps the allocation when it is large enough
    void ensure(size_t count) {
        if (count > cap || !p) {
            free();
            if (count) ECO_CUDA(cudaMalloc(&p, count * sizeof(T)));
            cap = count;
        }
        n = count;
    }
    void free() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
        cap = 0;
    }
    ~DBuf() { free(); }
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    void upload(const T* h, size_t count, cudaStream_t s = 0) {
        if (count) ECO_CUDA(cudaMemcpyAsync(p, h, count * sizeof(T), cudaMemcpyHostToDevice, s));
    }
    void download(T* h, size_t count, cudaStream_t s = 0) const {
        if (count) ECO_CUDA(cudaMemcpyAsync(h, p, count * sizeof(T), cudaMemcpyDeviceToHost, s));
    }
};

// ------------------------------------------------------------ conversions
template <typename Real>
__global__ void to_internal_kernel(const double* __restrict__ src, Real* __restrict__ dst, size_t n, double j_inf) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        const double x = src[i];
        dst[i] = (x >= j_inf) ? (Real)INFINITY : (Real)x;
    }
}

template <typename Real>
__global__ void to_external_kernel(const Real* __restrict__ src, double* __restrict__ dst, size_t n, double j_inf) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        const double x = (double)src[i];
        dst[i] = (x < j_inf) ? x : j_inf;
    }
}

// (v, soc, t) levels are stored twice: copy 0 as-is and copy 1 shifted by one
// element, so the stage kernel reads any two consecutive time samples with one
// aligned 64-bit load.  level_stride() is the distance between levels.
// The pad after each copy (>= 128 elements) absorbs the wide-row path's
// loads past a row's last live state.
__host__ __device__ inline size_t level_copy(size_t ns) { return (ns + 135) & ~size_t(7); }
__host__ __device__ inline size_t level_stride(size_t ns) { return 2 * level_copy(ns); }

template <typename Real>
__global__ void to_internal2_kernel(const double* __restrict__ src, Real* __restrict__ dst, size_t n, double j_inf) {
    Real* d1 = dst + level_copy(n);
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n + 8; i += (size_t)gridDim.x * blockDim.x) {
        const Real x = i < n ? ((src[i] >= j_inf) ? (Real)INFINITY : (Real)src[i]) : (Real)INFINITY;
        if (i < n) dst[i] = x; else dst[i] = (Real)INFINITY;
        if (i > 0) d1[i - 1] = x;
        if (i == n + 7) d1[i] = (Real)INFINITY;
    }
}

// copy 0 of `levels` levels `stride` elements apart -> contiguous f64
template <typename Real>
__global__ void to_external_strided_kernel(const Real* __restrict__ src, double* __restrict__ dst, size_t n,
                                           int levels, size_t stride, double j_inf) {
    const size_t total = n * levels;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
        const size_t l = i / n, e = i - l * n;
        const double x = (double)src[l * stride + e];
        dst[i] = (x < j_inf) ? x : j_inf;
    }
}

// copy 0 of `levels` stacked levels -> contiguous f64 (infeasible -> j_inf)
template <typename Real>
__global__ void to_external_levels_kernel(const Real* __restrict__ src, double* __restrict__ dst, size_t n,
                                          int levels, double j_inf) {
    const size_t total = n * levels;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
        const size_t l = i / n, e = i - l * n;
        const double x = (double)src[l * level_stride(n) + e];
        dst[i] = (x < j_inf) ? x : j_inf;
    }
}

inline unsigned grid_for(size_t n, unsigned block = 256) {
    size_t g = (n + block - 1) / block;
    if (g > 148u * 32u) g = 148u * 32u;
    return (unsigned)(g ? g : 1);
}

// ---------------------------------------------------------------- timing
struct EventTimer {
    cudaEvent_t a{}, b{};
    EventTimer() {
        ECO_CUDA(cudaEventCreate(&a));
        ECO_CUDA(cudaEventCreate(&b));
    }
    ~EventTimer() {
        cudaEventDestroy(a);
        cudaEventDestroy(b);
    }
    void start(cudaStream_t s) { ECO_CUDA(cudaEventRecord(a, s)); }
    void stop(cudaStream_t s) { ECO_CUDA(cudaEventRecord(b, s)); }
    double ms() {
        float m = 0.f;
        ECO_CUDA(cudaEventSynchronize(b));
        ECO_CUDA(cudaEventElapsedTime(&m, a, b));
        return m;
    }
};

// Host memcpy spread over up to 16 threads (large pinned <-> pageable copies:
// one core moves ~10 GB/s, the copy engines ~50).
void parallel_memcpy(void* dst, const void* src, size_t n) {
    char* d = static_cast<char*>(dst);
    const char* s = static_cast<const char*>(src);
    if (n < (size_t(8) << 20)) {
        std::memcpy(d, s, n);
        return;
    }
    const unsigned hw = std::thread::hardware_concurrency();
    const int nthr = (int)std::max(1u, std::min(16u, hw ? hw : 1u));
    std::vector<std::thread> th;
    const size_t per = ((n + nthr - 1) / nthr + 4095) & ~size_t(4095);
    for (int t = 0; t < nthr; ++t) {
        const size_t a = (size_t)t * per;
        if (a >= n) break;
        const size_t m = std::min(per, n - a);
        th.emplace_back([=] { std::memcpy(d + a, s + a, m); });
    }
    for (auto& x : th) x.join();
}

// Page-locked host memory (cudaHostAlloc, or registered): the copy engines
// DMA straight into it, so a device -> host copy needs no staging.
inline bool host_pinned(const void* p) {
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();   // pageable memory may report an error on old drivers
        return false;
    }
    return at.type == cudaMemoryTypeHost;
}

// Large device -> pageable-host copies (the J / P stacks of fine-grid solves,
// batch tables): double-buffered pinned staging; chunk i's host-side copy is
// spread over threads (first-touching the destination in parallel) while
// chunk i + 1's DMA runs.  Completes before returning.  A pinned destination
// (eco_host_alloc, the Python pinned pool) takes one direct DMA instead.
void download_big(void* dst, const void* src, size_t bytes, cudaStream_t st) {
    constexpr size_t kChunk = size_t(64) << 20;
    if (bytes < (size_t(32) << 20) || std::getenv("ECO_PLAIN_D2H") || host_pinned(dst)) {
        if (bytes) ECO_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, st));
        ECO_CUDA(cudaStreamSynchronize(st));
        return;
    }
    static std::mutex mu;
    static char* stage[2] = {nullptr, nullptr};
    static cudaEvent_t ev[2];
    std::lock_guard<std::mutex> lock(mu);
    if (!stage[0]) {
        for (int b = 0; b < 2; ++b) {
            ECO_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&stage[b]), kChunk, cudaHostAllocDefault));
            ECO_CUDA(cudaEventCreateWithFlags(&ev[b], cudaEventDisableTiming));
        }
    }
    auto host_copy = [&](char* d, const char* s, size_t n) { parallel_memcpy(d, s, n); };
    char* out = static_cast<char*>(dst);
    const char* in = static_cast<const char*>(src);
    int prev = -1;
    size_t prev_off = 0, prev_n = 0, off = 0;
    for (int i = 0; off < bytes; ++i) {
        const size_t n = std::min(kChunk, bytes - off);
        const int b = i & 1;
        ECO_CUDA(cudaMemcpyAsync(stage[b], in + off, n, cudaMemcpyDeviceToHost, st));
        ECO_CUDA(cudaEventRecord(ev[b], st));
        if (prev >= 0) {
            ECO_CUDA(cudaEventSynchronize(ev[prev]));
            host_copy(out + prev_off, stage[prev], prev_n);
        }
        prev = b; prev_off = off; prev_n = n;
        off += n;
    }
    ECO_CUDA(cudaEventSynchronize(ev[prev]));
    host_copy(out + prev_off, stage[prev], prev_n);
}

inline int env_int(const char* name, int dflt);

// Level-by-level f32 -> f64 download of a solve's J stack (levels H..0 as
// their stages finish, lvl_ev[k]) + the int32 policies, through a ring of
// pinned f32 staging buffers; host threads widen each level into the
// caller's table (infeasible +inf -> j_inf, the to_external conversion)
// while the next levels' DMA runs.  Returns when every level is written.
// f32 -> f64 with infeasible (+inf) -> j_inf over [a, b): streaming
// (non-temporal) stores, so the f64 table is written without first being
// read into the cache -- host memory bandwidth is what bounds this copy.
__attribute__((target("avx2"))) void widen_range_avx2(const float* src, double* dst, size_t a, size_t b,
                                                      double j_inf) {
    size_t i = a;
    for (; i < b && (reinterpret_cast<uintptr_t>(dst + i) & 31); ++i) {
        const double x = (double)src[i];
        dst[i] = x < j_inf ? x : j_inf;
    }
    const __m256d cap = _mm256_set1_pd(j_inf);
    for (; i + 8 <= b; i += 8) {
        const __m256 v = _mm256_loadu_ps(src + i);
        // x < j_inf ? x : j_inf  ==  min(x, j_inf) for x finite or +inf
        const __m256d lo = _mm256_min_pd(_mm256_cvtps_pd(_mm256_castps256_ps128(v)), cap);
        const __m256d hi = _mm256_min_pd(_mm256_cvtps_pd(_mm256_extractf128_ps(v, 1)), cap);
        _mm256_stream_pd(dst + i, lo);
        _mm256_stream_pd(dst + i + 4, hi);
    }
    for (; i < b; ++i) {
        const double x = (double)src[i];
        dst[i] = x < j_inf ? x : j_inf;
    }
    _mm_sfence();
}

// Levels with widen(k) false go the direct way instead (device-side f64
// conversion into d_tmp + f64 DMA): mixing the two balances the PCIe link
// (which the f64 levels load) against host memory bandwidth (which the
// widening loads: DMA write + read + f64 write per level).
template <typename WidenPred>
void widen_levels(const float* d_J, size_t LV, size_t ns, int H, int k_top, double j_inf, const int32_t* d_P,
                  double* J_stack, int32_t* P_stack, const std::vector<cudaEvent_t>& lvl_ev, cudaStream_t st,
                  double* d_tmp, WidenPred widen_level) {
    constexpr int kSlots = 4;
    static std::mutex mu;
    static float* stage[kSlots] = {nullptr, nullptr, nullptr, nullptr};
    static size_t stage_n = 0;
    static cudaEvent_t ev[kSlots];
    std::lock_guard<std::mutex> lock(mu);
    if (stage_n < ns) {
        for (int b = 0; b < kSlots; ++b) {
            if (stage[b]) cudaFreeHost(stage[b]);
            else ECO_CUDA(cudaEventCreateWithFlags(&ev[b], cudaEventDisableTiming));
            ECO_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&stage[b]), ns * sizeof(float), cudaHostAllocDefault));
        }
        stage_n = ns;
    }
    const unsigned hw = std::thread::hardware_concurrency();
    const int nthr = (int)std::max(1u, std::min(16u, hw ? hw : 1u));
    static const bool avx2 = __builtin_cpu_supports("avx2");
    auto widen = [&](const float* src, double* dst) {
        std::vector<std::thread> th;
        const size_t per = ((ns + nthr - 1) / nthr + 1023) & ~size_t(1023);
        for (int t = 0; t < nthr; ++t) {
            const size_t a = (size_t)t * per;
            if (a >= ns) break;
            const size_t b = std::min(ns, a + per);
            th.emplace_back([=] {
                if (avx2) widen_range_avx2(src, dst, a, b, j_inf);
                else
                    for (size_t i = a; i < b; ++i) {
                        const double x = (double)src[i];
                        dst[i] = x < j_inf ? x : j_inf;
                    }
            });
        }
        for (auto& x : th) x.join();
    };
    // the widened levels in completion order; the others are enqueued direct
    std::vector<int> wl;
    for (int k = k_top; k >= 0; --k) {
        if (!widen_level(k)) continue;
        wl.push_back(k);
    }
    const int L = (int)wl.size();
    int queued = 0, k_next = k_top;      // k_next: next level (any kind) to enqueue, in completion order
    auto enqueue_until = [&](int k_stop) {  // enqueue every level down to (and including) k_stop
        for (; k_next >= k_stop; --k_next) {
            const int k = k_next;
            ECO_CUDA(cudaStreamWaitEvent(st, lvl_ev[k], 0));
            if (widen_level(k)) {
                const int b = queued % kSlots;
                ECO_CUDA(cudaMemcpyAsync(stage[b], d_J + (size_t)k * LV, ns * sizeof(float), cudaMemcpyDeviceToHost,
                                         st));
                ECO_CUDA(cudaEventRecord(ev[b], st));
                ++queued;
            } else {
                to_external_levels_kernel<float><<<grid_for(ns), 256, 0, st>>>(d_J + (size_t)k * LV,
                                                                              d_tmp + (size_t)k * ns, ns, 1, j_inf);
                ECO_CUDA(cudaGetLastError());
                ECO_CUDA(cudaMemcpyAsync(J_stack + (size_t)k * ns, d_tmp + (size_t)k * ns, ns * sizeof(double),
                                         cudaMemcpyDeviceToHost, st));
            }
            if (k < H)
                ECO_CUDA(cudaMemcpyAsync(P_stack + (size_t)k * ns, d_P + (size_t)k * ns, ns * sizeof(int32_t),
                                         cudaMemcpyDeviceToHost, st));
        }
    };
    for (int done = 0; done < L; ++done) {
        // keep up to kSlots widened levels in flight (and every direct level
        // in between)
        const int last = std::min(L - 1, done + kSlots - 1);
        if (queued <= last) enqueue_until(wl[last]);
        const int k = wl[done], b = done % kSlots;
        ECO_CUDA(cudaEventSynchronize(ev[b]));
        widen(stage[b], J_stack + (size_t)k * ns);
    }
    enqueue_until(0);                    // direct levels after the last widened one
}

inline int env_int(const char* name, int dflt) {
    const char* v = std::getenv(name);
    return v ? std::atoi(v) : dflt;
}

// Kernel launch with programmatic dependent launch (when pdl and ECO_PDL):
// the kernel may start once the previous kernel in the stream triggered
// griddepcontrol.launch_dependents; it must griddepcontrol.wait before
// reading that kernel's results.
template <typename... KArgs, typename... Args>
void launch_pdl(void (*k)(KArgs...), int grid, int block, cudaStream_t st, bool pdl, Args&&... args) {
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3(grid);
    lc.blockDim = dim3(block);
    lc.dynamicSmemBytes = 0;
    lc.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = (pdl && env_int("ECO_PDL", 1)) ? 1 : 0;
    lc.attrs = attr;
    lc.numAttrs = 1;
    ECO_CUDA(cudaLaunchKernelEx(&lc, k, std::forward<Args>(args)...));
}

// long time ladders take the wide-row stage path (ECO_WIDE=0 disables it)
inline bool wide_rows(int nt) { return nt >= 128 && nt % 2 == 0 && env_int("ECO_WIDE", 1) != 0; }

// wide rows in row blocks (bellman_wide2_kernel, ECO_WIDE2=0 disables it):
// warps per row block (kW2S states each), 0 when not used
inline int w2_wpr(int nt) {
    if (!wide_rows(nt) || env_int("ECO_WIDE2", 1) == 0) return 0;
    const int wpr = (nt + kW2S - 1) / kW2S;
    return wpr <= kW2MaxWarps ? wpr : 0;
}
inline int w2_tj(int nt) { return w2_wpr(nt) ? kW2R : 0; }

template <typename K>
void set_smem_attr(K kernel, size_t smem) {
    // cached per kernel (keeps attribute calls out of stream capture).  The
    // attribute is process-wide, so the cache is too and only ever RAISES the
    // limit: a thread setting a smaller value would invalidate another
    // thread's launches with a larger one
    static std::mutex mu;
    static std::vector<std::pair<const void*, size_t>> done;
    if (smem <= 48 * 1024) return;
    std::lock_guard<std::mutex> lock(mu);
    for (auto& d : done)
        if (d.first == (const void*)kernel) {
            if (d.second >= smem) return;
            d.second = smem;
            ECO_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            return;
        }
    ECO_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    done.emplace_back((const void*)kernel, smem);
}

// --------------------------------------------------------- geometry store
template <typename Real>
struct Geometry {
    GeomDims dims{};
    DBuf<int32_t> count, u, gmax;
    DBuf<int64_t> row_off;
    DBuf<double> dt, c1d, pbat;
    DBuf<ActRec<Real>> act;
    DBuf<RowRec<Real>> row;
    DBuf<RowRec2<Real>> row2;
    DBuf<TilePlan> tiles;
    DBuf<int32_t> order, rank_of;
    int h_gmax[4] = {0, 0, 0, 0};     // [0] max feasible actions of a plane, [1] some tile unstaged
    bool all_staged = false;          // every tile stages its band: no kernel reads the shifted copy
    int64_t rows_total = 0;
    int tj = 0, nchunk = 0, band_cap = 0;   // stage-kernel tile shape the plans were built for
    int plo = 0, phi = -1;                  // tiles of planes [plo, phi) ordered first (slab solves)
    int tj_pref = 0, slices_pref = 0;       // tile shape overrides (0: defaults); the batch prefers 4 x 8

    // grow-only: rebuilding a smaller set of plans (field chunks, ring
    // slots) keeps the allocation
    void alloc(int P, int nv, int U) {
        const size_t np = (size_t)P * nv * U;
        count.ensure((size_t)P * nv); row_off.ensure((size_t)P * nv); gmax.ensure(4);
        u.ensure(np); dt.ensure(np); c1d.ensure(np); pbat.ensure(np); act.ensure(np);
    }
    PairGeom<Real> view() {
        return PairGeom<Real>{count.p, row_off.p, u.p, dt.p, c1d.p, pbat.p, act.p, row.p, gmax.p};
    }
};

template <typename Real>
int light_first(const Geometry<Real>& G, int nt, int nlaunch);

// Compacted pair records + SoC row records for P plans (dims filled by the
// caller).  The row buffer is sized from the feasible-pair count (kept across
// rebuilds of the same route, so refits allocate nothing).
// with_tiles = false: pair + SoC-row records only (what the terminal-field
// sweep reads), no stage-kernel tile plans.
// staged_flag: read back whether every tile stages its band (G.all_staged,
// used by the closed loop to skip the shifted level copy) -- one more host
// round trip, skipped by the stateless solves.
template <typename Real>
void build_geometry(Geometry<Real>& G, const EcoPlant* d_plant, const DevPlan* d_plans, const double* d_vaxes,
                    const double* d_te, const double* d_tb, const double* d_soc, const EcoStage1Tables& d_tab,
                    cudaStream_t st, int64_t* launches, bool with_tiles = true, bool staged_flag = true) {
    const GeomDims& g = G.dims;
    if (G.act.n != (size_t)g.P * g.nv * g.U) G.alloc(g.P, g.nv, g.U);
    ECO_CUDA(cudaMemsetAsync(G.gmax.p, 0, 4 * sizeof(int32_t), st));
    dim3 grid(g.nv, g.P);
    geom_pairs_kernel<Real><<<grid, 256, 0, st>>>(d_plant, d_plans, d_vaxes, d_te, d_tb, g, G.view(), d_tab);
    ECO_CUDA(cudaGetLastError());
    const int npi = g.P * g.nv;
    geom_rowoff_kernel<<<1, 1024, 0, st>>>(G.count.p, G.row_off.p, npi, g.nx);
    ECO_CUDA(cudaGetLastError());
    int64_t last_off = 0;
    int32_t last_cnt = 0;
    ECO_CUDA(cudaMemcpyAsync(&last_off, G.row_off.p + npi - 1, sizeof last_off, cudaMemcpyDeviceToHost, st));
    ECO_CUDA(cudaMemcpyAsync(&last_cnt, G.count.p + npi - 1, sizeof last_cnt, cudaMemcpyDeviceToHost, st));
    ECO_CUDA(cudaMemcpyAsync(G.h_gmax, G.gmax.p, 4 * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    ECO_CUDA(cudaStreamSynchronize(st));
    G.rows_total = last_off + (int64_t)last_cnt * g.nx;
    if (G.row.cap < (size_t)std::max<int64_t>(1, G.rows_total)) G.row.alloc((size_t)std::max<int64_t>(1, G.rows_total));
    const size_t smem = (size_t)g.ntb * g.nx * (sizeof(double) + 1) + 16;
    set_smem_attr(geom_soc_kernel<Real>, smem);
    geom_soc_kernel<Real><<<grid, ECO_SOC_THREADS, smem, st>>>(d_plant, d_vaxes, d_tb, d_soc, g, G.view(),
                                                   d_tab.ok != nullptr ? 1 : 0);
    ECO_CUDA(cudaGetLastError());
    geom_unpack_u_kernel<<<npi, 256, 0, st>>>(G.u.p, G.count.p, g.U);
    ECO_CUDA(cudaGetLastError());
    if (!with_tiles) {
        if (launches) *launches += 4;
        return;
    }
    // staging plans of the (v, soc, t) stage kernel's tiles
    const int upr = (g.nt + kZP - 1) / kZP;
    const int tj_default = G.tj_pref > 0 ? G.tj_pref
                                          : (w2_tj(g.nt) ? w2_tj(g.nt) : (wide_rows(g.nt) ? 2 : std::max(1, 16 / upr)));
    G.tj = w2_tj(g.nt) ? std::min(g.nx, tj_default) : std::min(g.nx, std::max(1, env_int("ECO_TILE_TJ", tj_default)));
    G.nchunk = (g.nx + G.tj - 1) / G.tj;
    // wide-row tiles never stage a band (and get no RowRec2 buffer): cap -1
    // marks every one of them unstaged
    G.band_cap = wide_rows(g.nt) ? -1 : env_int("ECO_BAND_KB", 40) * 1024 / (int)sizeof(Real);
    const size_t ntiles = (size_t)npi * G.nchunk;
    G.tiles.ensure(ntiles);
    // RowRec2 (shared-memory band bases) only serve the staged narrow path:
    // wide-row tiles never stage a band
    if (!wide_rows(g.nt) && G.row2.cap < G.row.cap) G.row2.alloc(G.row.cap);
    G.order.ensure(ntiles);
    G.rank_of.ensure(ntiles);
    const int phi = G.phi < 0 ? g.nv : G.phi;
    const int chunk_major = env_int("ECO_CHUNK_MAJOR", wide_rows(g.nt) ? 1 : 0);
    const int light = chunk_major ? 0 : light_first<Real>(G, g.nt, (phi - G.plo) * G.nchunk);
    geom_order_kernel<<<g.P, 256, 0, st>>>(G.count.p, g.nv, G.nchunk, G.plo, phi, light, chunk_major, G.order.p,
                                           G.rank_of.p);
    ECO_CUDA(cudaGetLastError());
    // one block per (plan, plane) covering all its SoC chunks (coalesced row
    // records); the per-tile kernel remains for grids whose chunk tables
    // exceed shared memory
    const size_t psmem = ((size_t)3 * G.nchunk * g.nv + G.nchunk) * sizeof(int32_t);
    if (wide_rows(g.nt)) {
        const size_t nt_ = ntiles;
        geom_tile_headers_kernel<<<(unsigned)((nt_ + 255) / 256), 256, 0, st>>>(G.count.p, G.row_off.p, g, G.tj,
                                                                              G.nchunk, G.tiles.p, G.rank_of.p,
                                                                              d_plans, d_vaxes, G.gmax.p);
    } else if (psmem <= 200 * 1024 && env_int("ECO_PLANE_TILES", 1) != 0) {
        set_smem_attr(geom_plane_tiles_kernel<Real>, psmem);
        geom_plane_tiles_kernel<Real><<<dim3(g.nv, g.P), 256, psmem, st>>>(
            G.view(), g, G.tj, G.nchunk, G.band_cap, G.tiles.p, G.row2.p, G.rank_of.p, d_plans, d_vaxes);
    } else {
        dim3 tgrid(g.nv * G.nchunk, g.P);
        geom_tiles_kernel<Real><<<tgrid, 256, (size_t)g.nv * 2 * sizeof(int32_t), st>>>(
            G.view(), g, G.tj, G.nchunk, G.band_cap, G.tiles.p, G.row2.p, G.rank_of.p, d_plans, d_vaxes);
    }
    ECO_CUDA(cudaGetLastError());
    if (staged_flag) {
        ECO_CUDA(cudaMemcpyAsync(&G.h_gmax[1], G.gmax.p + 1, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
        ECO_CUDA(cudaStreamSynchronize(st));
        G.all_staged = G.h_gmax[1] == 0 && !wide_rows(g.nt);
    } else {
        G.all_staged = false;
    }
    if (launches) *launches += 6;
}

// Tile shape of the stage kernel: tj SoC rows x n_t, S threads per action
// slice (multiple of 32 so every warp walks one action at a time).
struct TileCfg {
    int tj, nchunk, S, slices;
    int count_max = 0, band_cap = 0;
    int wide = 0;
    int alias = 0;
    size_t smem;
};


template <typename Real>
TileCfg tile_cfg(const Geometry<Real>& G, int nt, int mode, bool alias = false) {
    const int nx = G.dims.nx;
    TileCfg t{};
    if (mode == 1) {
        t.tj = nx;                             // the whole (v, soc) plane per CTA
        t.nchunk = 1;
        t.S = (nx + 31) / 32 * 32;
        if (t.S > 1024) throw ArgError{"n_soc too large for the field kernel"};
        t.slices = std::max(1, std::min(env_int("ECO_FIELD_SLICES", 1024 / t.S), 1024 / t.S));
        t.smem = align16((size_t)t.slices * t.S * sizeof(Real)) + (size_t)t.slices * t.S * sizeof(int32_t);
    } else {
        t.tj = G.tj;
        t.nchunk = G.nchunk;
        if (w2_wpr(nt)) {
            // row blocks: one warp per (kW2R rows, kW2S states), every warp
            // scans all actions (no slices); the reduction buffers only serve
            // the per-state path of standstill tiles (S = block, 1 slice)
            t.wide = w2_wpr(nt);
            t.S = 32 * t.wide;
            t.slices = 1;
            t.count_max = std::max(1, G.h_gmax[0]);
            // the band region holds the per-action W2Quad summaries
            t.band_cap = (int)((t.count_max * sizeof(W2Quad<Real>) + sizeof(Real) - 1) / sizeof(Real));
            t.smem = TileSmem<Real>(nt, t.tj, 1, t.count_max, t.band_cap).total;
            if (t.smem > 227 * 1024) throw ArgError{"tile buffers exceed shared memory"};
            return t;
        }
        if (wide_rows(nt)) {
            // wide rows: S = warps per row x 32 x tj, no shared-memory staging
            t.wide = (nt + 64 * kMW - 1) / (64 * kMW);
            t.S = 32 * t.wide * t.tj;
            if (t.S > 256) throw ArgError{"tile too large for the wide-row path (lower ECO_TILE_TJ)"};
            t.slices = std::max(1, std::min(env_int("ECO_TILE_SLICES", std::max(1, 256 / t.S)), 256 / t.S));
            t.count_max = std::max(1, G.h_gmax[0]);   // record staging, no J band
            t.band_cap = 0;
            t.smem = TileSmem<Real>(nt, t.tj, t.slices, t.count_max, 0).total;
            if (t.smem > 227 * 1024) throw ArgError{"tile reduction buffers exceed shared memory"};
            return t;
        }
        const int upr = (nt + kZP - 1) / kZP;
        // threads per action slice: one per kZP ladder states of the tile (a
        // warp may hold two slices); the per-state path strides over states
        const int per_row = (nt % 2 == 0) ? upr : nt;
        t.S = std::min(256, t.tj * per_row);
        if (nt % 2 == 0 && t.tj * upr > 256) throw ArgError{"stage tile too tall (lower ECO_TILE_TJ)"};
        const int sl_default = G.slices_pref > 0 ? G.slices_pref : std::max(1, 256 / t.S);
        // <= 256 threads: the single-solve stage kernel is built for 256-thread blocks
        t.slices = std::max(1, std::min(env_int("ECO_TILE_SLICES", sl_default), std::max(1, 256 / t.S)));
        t.count_max = std::max(1, G.h_gmax[0]);
        t.band_cap = G.band_cap;
        t.alias = (alias || env_int("ECO_STAGE_ALIAS", 0) != 0) ? 1 : 0;
        t.smem = TileSmem<Real>(nt, t.tj, t.slices, t.count_max, t.band_cap, t.alias != 0).total;
    }
    if (t.smem > 227 * 1024) throw ArgError{"tile reduction buffers exceed shared memory"};
    return t;
}

template <typename Real>
StageArgs<Real> stage_args(Geometry<Real>& G, int p, const double* d_vsrc, int nt, const TileCfg& tc) {
    StageArgs<Real> a{};
    const GeomDims& g = G.dims;
    const size_t off = (size_t)p * g.nv * g.U;
    a.count = G.count.p + (size_t)p * g.nv;
    a.row_off = G.row_off.p + (size_t)p * g.nv;
    a.u = G.u.p + off;
    a.dt = G.dt.p + off;
    a.c1d = G.c1d.p + off;
    a.act = G.act.p + off;
    a.row = G.row.p;
    a.row2 = G.row2.p;
    a.tiles = G.tiles.p + (size_t)p * g.nv * G.nchunk;
    a.order = G.order.p + (size_t)p * g.nv * G.nchunk;
    a.v_src = d_vsrc;
    a.nv = g.nv;
    a.nx = g.nx;
    a.nt = nt;
    a.U = g.U;
    a.tj = tc.tj;
    a.nchunk = tc.nchunk;
    a.S = tc.S;
    a.slices = tc.slices;
    a.count_max = tc.count_max;
    a.band_cap = tc.band_cap;
    a.wide = tc.wide;
    a.alias = tc.alias;
    a.gamma = g.gamma;
    return a;
}


inline int sm_count_cached() {
    static int n = 0;
    if (!n) {
        int dev = 0;
        ECO_CUDA(cudaGetDevice(&dev));
        ECO_CUDA(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
    }
    return n;
}

// Tiles a stage launch puts in front (geom_order_kernel): when the launch is
// between one and two waves of resident CTAs, the overflow count.
template <typename Real>
int light_first(const Geometry<Real>& G, int nt, int nlaunch) {
    if (env_int("ECO_LIGHT_FIRST", 1) == 0) return 0;
    const TileCfg tc = tile_cfg(G, nt, 0);
    auto k = (tc.wide && w2_wpr(nt)) ? bellman_wide2_kernel<Real, false>
                                     : tc.wide ? bellman_wide_kernel<Real, false> : bellman_stage_kernel<Real, false>;
    set_smem_attr(k, tc.smem);
    int per_sm = 0;
    ECO_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, tc.S * tc.slices, tc.smem));
    const int slots = per_sm * sm_count_cached();
    return (slots > 0 && nlaunch > slots && nlaunch < 2 * slots) ? nlaunch - slots : 0;
}

template <typename Real, int MODE>
void launch_stage(const StageArgs<Real>& a, const TileCfg& tc, bool count, cudaStream_t st, int ntiles = -1,
                  bool rev = false) {
    const unsigned grid = (unsigned)(ntiles >= 0 ? ntiles : a.nv * tc.nchunk);
    const unsigned block = (unsigned)(tc.S * tc.slices);
    if (MODE == 0) {
        using KT = void (*)(StageArgs<Real>);
        KT k;
        const bool w2 = tc.wide && w2_wpr(a.nt);
        if (rev) {   // perturb_ties (highest index wins ties): plain solves only
            if (count || a.npeer > 0) throw ArgError{"perturb_ties: not with live counting or slab exchange"};
            k = w2 ? bellman_wide2_kernel<Real, false, false, true>
                   : tc.wide ? bellman_wide_kernel<Real, false, false, true> : bellman_stage_kernel<Real, false, false, true>;
        } else if (w2) {
            const bool fine = a.nt == kW2FineNT && env_int("ECO_W2_NTC", 1) != 0;
            k = a.npeer > 0 ? (count ? bellman_wide2_kernel<Real, true, true>
                                     : fine ? bellman_wide2_kernel<Real, false, true, false, kW2FineNT>
                                            : bellman_wide2_kernel<Real, false, true>)
                            : (count ? bellman_wide2_kernel<Real, true>
                                     : fine ? bellman_wide2_kernel<Real, false, false, false, kW2FineNT>
                                            : bellman_wide2_kernel<Real, false>);
        } else if (a.npeer > 0)
            k = tc.wide ? (count ? bellman_wide_kernel<Real, true, true> : bellman_wide_kernel<Real, false, true>)
                        : (count ? bellman_stage_kernel<Real, true, true> : bellman_stage_kernel<Real, false, true>);
        else
            k = tc.wide ? (count ? bellman_wide_kernel<Real, true> : bellman_wide_kernel<Real, false>)
                        : (count ? bellman_stage_kernel<Real, true> : bellman_stage_kernel<Real, false>);
        set_smem_attr(k, tc.smem);
        // programmatic dependent launch: the prologue overlaps the previous kernel's tail
        cudaLaunchConfig_t lc{};
        lc.gridDim = dim3(grid);
        lc.blockDim = dim3(block);
        lc.dynamicSmemBytes = tc.smem;
        lc.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = env_int("ECO_PDL", 1) ? 1 : 0;
        lc.attrs = attr;
        lc.numAttrs = 1;
        ECO_CUDA(cudaLaunchKernelEx(&lc, k, a));
    } else {
        set_smem_attr(field_stage_kernel<Real>, tc.smem);
        cudaLaunchConfig_t lc{};
        lc.gridDim = dim3(grid);
        lc.blockDim = dim3(block);
        lc.dynamicSmemBytes = tc.smem;
        lc.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = env_int("ECO_PDL", 1) ? 1 : 0;
        lc.attrs = attr;
        lc.numAttrs = 1;
        ECO_CUDA(cudaLaunchKernelEx(&lc, field_stage_kernel<Real>, a));
    }
    ECO_CUDA(cudaGetLastError());
}

void check_problem(const EcoProblem* pr) {
    if (!pr) throw ArgError{"null problem"};
    if (pr->n_v < 2 || pr->n_soc < 2 || pr->n_t < 2 || pr->n_te < 1 || pr->n_tb < 1)
        throw ArgError{"grid sizes must be n_v,n_soc,n_t >= 2 and n_te,n_tb >= 1"};
    if (pr->n_v >= (1 << 23)) throw ArgError{"n_v too large"};
    if (pr->n_soc > 32767) throw ArgError{"n_soc must be < 32768"};
    if ((int64_t)pr->n_te * pr->n_tb > 8192) throw ArgError{"n_te * n_tb must be <= 8192"};
    if (!pr->te_axis || !pr->tb_axis || !pr->soc_axis) throw ArgError{"null axis"};
}

void check_plant(const EcoPlant* p) {
    if (!p) throw ArgError{"null plant"};
    if (p->n_gears < 1 || p->n_gears > ECO_MAX_GEARS || p->n_eng < 2 || p->n_eng > ECO_MAX_AXIS ||
        p->n_fuel_w < 2 || p->n_fuel_w > ECO_MAX_AXIS || p->n_fuel_t < 2 || p->n_fuel_t > ECO_MAX_AXIS ||
        p->n_bsg < 2 || p->n_bsg > ECO_MAX_AXIS || p->n_eff_w < 2 || p->n_eff_w > ECO_MAX_AXIS ||
        p->n_eff_t < 2 || p->n_eff_t > ECO_MAX_AXIS || p->n_voc < 2 || p->n_voc > ECO_MAX_AXIS)
        throw ArgError{"plant table sizes out of range"};
}

DevPlan dev_plan(const EcoStepPlan& s) {
    DevPlan d;
    d.src_kind = s.src_kind;
    d.dest_kind = s.dest_kind;
    d.cos_g = s.cos_grade;
    d.sin_g = s.sin_grade;
    d.v0d = s.v0_dest;
    d.dvd = s.dv_dest;
    return d;
}

struct TablesDev {
    DBuf<uint8_t> ok;
    DBuf<double> v2, dt, pbat, c1, wv, wz;
    DBuf<int32_t> ivlo, ivhi, zoff;
    EcoStage1Tables view{};
    void upload(const EcoStage1Tables* t, size_t n, cudaStream_t s) {
        if (!t) { std::memset(&view, 0, sizeof view); return; }
        ok.alloc(n); v2.alloc(n); dt.alloc(n); pbat.alloc(n); c1.alloc(n); wv.alloc(n); wz.alloc(n);
        ivlo.alloc(n); ivhi.alloc(n); zoff.alloc(n);
        ok.upload(t->ok, n, s); v2.upload(t->v2, n, s); dt.upload(t->dt, n, s); pbat.upload(t->pbat, n, s);
        c1.upload(t->c1, n, s); wv.upload(t->wv, n, s); wz.upload(t->wz, n, s);
        ivlo.upload(t->ivlo, n, s); ivhi.upload(t->ivhi, n, s); zoff.upload(t->zoff, n, s);
        view = EcoStage1Tables{ok.p, v2.p, dt.p, pbat.p, c1.p, ivlo.p, ivhi.p, wv.p, zoff.p, wz.p};
    }
};

// Checked builds: per-stage single-writer shadow counts (see ECO_CHECKED in
// eco_kernels.cuh).  arm() before a stage, verify() after it.
struct WriterCheck {
#ifdef ECO_CHECKED
    DBuf<unsigned> cnt;
    size_t n = 0;
    explicit WriterCheck(size_t ns) : n(ns) {
        cnt.alloc(ns);
        unsigned* p = cnt.p;
        ECO_CUDA(cudaMemcpyToSymbol(g_chk_wcount, &p, sizeof p));
    }
    ~WriterCheck() {
        unsigned* p = nullptr;
        cudaMemcpyToSymbol(g_chk_wcount, &p, sizeof p);
    }
    void arm(cudaStream_t st) { ECO_CUDA(cudaMemsetAsync(cnt.p, 0, n * sizeof(unsigned), st)); }
    void verify(cudaStream_t st) {
        chk_single_writer_kernel<<<grid_for(n), 256, 0, st>>>(cnt.p, n);
        ECO_CUDA(cudaGetLastError());
    }
#else
    explicit WriterCheck(size_t) {}
    void arm(cudaStream_t) {}
    void verify(cudaStream_t) {}
#endif
};

// --------------------------------------------------------- horizon solve
// Per-solve inputs of a horizon solve: plant, the H step plans (DevPlan +
// source speed axis + ladders + stage flags + source kinds), the axes and the
// terminal level, packed into one pinned host block and sent with a single
// copy into a grow-only device block, so repeated solves allocate nothing.
struct HorizonInputs {
    DBuf<char> blob;
    char* host = nullptr;
    size_t host_cap = 0;
    EcoPlant* plant = nullptr;
    DevPlan* plans = nullptr;
    double *v = nullptr, *tdep = nullptr, *wait = nullptr, *te = nullptr, *tb = nullptr, *soc = nullptr;
    double* terminal = nullptr;
    uint8_t *green = nullptr, *dep = nullptr;
    int* flags = nullptr;      // kStageAny* per stage
    int8_t* kinds = nullptr;   // source node kind per stage
    HorizonInputs() = default;
    HorizonInputs(const HorizonInputs&) = delete;
    HorizonInputs& operator=(const HorizonInputs&) = delete;
    ~HorizonInputs() {
        if (host) cudaFreeHost(host);
    }
    // every caller synchronises its stream before returning, so the host
    // block is free again when the next upload fills it
    void upload(const EcoPlant* p, const EcoProblem* pr, const EcoStepPlan* pl, int H, const double* term,
                cudaStream_t st) {
        const size_t nv = pr->n_v, nx = pr->n_soc, nt = pr->n_t, ns = nv * nx * nt;
        size_t off = 0;
        auto take = [&](size_t bytes) {
            const size_t o = off;
            off += (bytes + 255) & ~size_t(255);
            return o;
        };
        const size_t o_plant = take(sizeof(EcoPlant)), o_plans = take(sizeof(DevPlan) * H),
                     o_v = take(sizeof(double) * H * nv), o_tdep = take(sizeof(double) * H * nt),
                     o_wait = take(sizeof(double) * H * nt), o_te = take(sizeof(double) * pr->n_te),
                     o_tb = take(sizeof(double) * pr->n_tb), o_soc = take(sizeof(double) * nx),
                     o_term = take(term ? sizeof(double) * ns : 0), o_green = take((size_t)H * nt),
                     o_dep = take((size_t)H * nt), o_flags = take(sizeof(int) * H), o_kinds = take(H);
        if (off > host_cap) {
            if (host) cudaFreeHost(host);
            host = nullptr;
            host_cap = 0;
            ECO_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&host), off, cudaHostAllocDefault));
            host_cap = off;
        }
        blob.ensure(off);
        char* h = host;
        std::memcpy(h + o_plant, p, sizeof(EcoPlant));
        DevPlan* hp = reinterpret_cast<DevPlan*>(h + o_plans);
        int* hflags = reinterpret_cast<int*>(h + o_flags);
        for (int k = 0; k < H; ++k) {
            const EcoStepPlan& s = pl[k];
            if (!s.v_src || !s.arr_green || !s.dep_ok || !s.t_dep || !s.wait) throw ArgError{"null plan array"};
            hp[k] = dev_plan(s);
            int f = 0;
            for (size_t z = 0; z < nt; ++z) {
                if (s.arr_green[z] == 0) f |= kStageAnyRed;
                if (s.dep_ok[z] == 0 || s.wait[z] > 0.0) f |= kStageAnyHold;
            }
            hflags[k] = f;
            reinterpret_cast<int8_t*>(h + o_kinds)[k] = (int8_t)s.src_kind;
            std::memcpy(h + o_v + sizeof(double) * k * nv, s.v_src, sizeof(double) * nv);
            std::memcpy(h + o_green + (size_t)k * nt, s.arr_green, nt);
            std::memcpy(h + o_dep + (size_t)k * nt, s.dep_ok, nt);
            std::memcpy(h + o_tdep + sizeof(double) * k * nt, s.t_dep, sizeof(double) * nt);
            std::memcpy(h + o_wait + sizeof(double) * k * nt, s.wait, sizeof(double) * nt);
        }
        std::memcpy(h + o_te, pr->te_axis, sizeof(double) * pr->n_te);
        std::memcpy(h + o_tb, pr->tb_axis, sizeof(double) * pr->n_tb);
        std::memcpy(h + o_soc, pr->soc_axis, sizeof(double) * nx);
        if (term) parallel_memcpy(h + o_term, term, sizeof(double) * ns);
        ECO_CUDA(cudaMemcpyAsync(blob.p, host, off, cudaMemcpyHostToDevice, st));
        char* d = blob.p;
        plant = reinterpret_cast<EcoPlant*>(d + o_plant);
        plans = reinterpret_cast<DevPlan*>(d + o_plans);
        v = reinterpret_cast<double*>(d + o_v);
        tdep = reinterpret_cast<double*>(d + o_tdep);
        wait = reinterpret_cast<double*>(d + o_wait);
        te = reinterpret_cast<double*>(d + o_te);
        tb = reinterpret_cast<double*>(d + o_tb);
        soc = reinterpret_cast<double*>(d + o_soc);
        terminal = term ? reinterpret_cast<double*>(d + o_term) : nullptr;
        green = reinterpret_cast<uint8_t*>(d + o_green);
        dep = reinterpret_cast<uint8_t*>(d + o_dep);
        flags = reinterpret_cast<int*>(d + o_flags);
        kinds = reinterpret_cast<int8_t*>(d + o_kinds);
    }
};

// The stateless solvers share one workspace (inputs block, tables, geometry,
// the overlap stream): calls from several host threads are serialised here
// (ctypes releases the GIL, so Python threads do reach this concurrently).
inline std::mutex& workspace_mutex() {
    static std::mutex mu;
    return mu;
}

inline HorizonInputs& horizon_inputs() {
    static HorizonInputs in;
    return in;
}

template <typename Real>
struct HorizonWorkspace {
    Geometry<Real> G;
    DBuf<Real> J;
    DBuf<int32_t> P;
    DBuf<double> tmp;
    DBuf<unsigned long long> live;
    void release() {
        G.~Geometry<Real>();
        new (&G) Geometry<Real>();
        J.free(); P.free(); tmp.free(); live.free();
    }
};

template <typename Real>
HorizonWorkspace<Real>& horizon_workspace() {
    static HorizonWorkspace<Real> w;
    return w;
}

// dp.py:425-475 / dp.py:557-610: H plans, terminal -> J stack, P stack.
template <typename Real>
// skip_terminal: J_stack receives levels 0..H-1 only (the terminal level is
// the caller's own input: backward_step's J_next).
void solve_horizon_impl(const EcoPlant* plant, const EcoProblem* pr, const EcoStepPlan* plans, int H,
                        const EcoStage1Tables* tabs, const double* terminal, double* J_stack, int32_t* P_stack,
                        bool count, EcoStats* stats, bool rev = false, bool skip_terminal = false) {
    const int top = skip_terminal ? H - 1 : H;    // highest level returned
    const int nv = pr->n_v, nx = pr->n_soc, nt = pr->n_t, U = pr->n_te * pr->n_tb;
    const size_t ns = (size_t)nv * nx * nt;
    std::lock_guard<std::mutex> lock(workspace_mutex());
    cudaStream_t st = 0;
    int64_t launches = 0;
    HorizonInputs& in = horizon_inputs();
    const bool dbg_io = env_int("ECO_DEBUG_IO", 0) != 0;
    const auto h0 = std::chrono::steady_clock::now();
    in.upload(plant, pr, plans, H, terminal, st);
    const auto h1 = std::chrono::steady_clock::now();
    TablesDev tdev;   // plant path: no tables

    // device buffers persist across calls (grow-only workspace): repeated
    // solves of one grid allocate nothing; eco_release_workspace() frees them
    HorizonWorkspace<Real>& W = horizon_workspace<Real>();
    Geometry<Real>& G = W.G;
    G.dims = GeomDims{H, nv, nx, nt, U, pr->n_te, pr->n_tb, pr->delta_d, pr->a_min, pr->a_max, pr->gamma, pr->dtg};
    const size_t LV = level_stride(ns), LC = level_copy(ns);
    W.J.ensure((H + 1) * LV);
    W.P.ensure((size_t)H * ns);
    W.tmp.ensure(ns * (H + 1));
    W.live.ensure(1);
    DBuf<Real>& d_J = W.J;
    DBuf<int32_t>& d_P = W.P;
    DBuf<double>& d_tmp = W.tmp;
    DBuf<unsigned long long>& d_live = W.live;
    ECO_CUDA(cudaMemsetAsync(d_live.p, 0, sizeof(unsigned long long), st));

    EventTimer all, sweep;
    all.start(st);
    // toy mode: each step has its own table; geometry built per plan below
    if (!tabs) build_geometry(G, in.plant, in.plans, in.v, in.te, in.tb, in.soc, tdev.view, st, &launches, true, false);
    to_internal2_kernel<Real><<<grid_for(ns + 8), 256, 0, st>>>(in.terminal, d_J.p + (size_t)H * LV, ns, pr->j_inf);
    ECO_CUDA(cudaGetLastError());
    ++launches;
    double sweep_ms = 0.0;
    std::vector<Geometry<Real>> toyG(tabs ? H : 0);
    if (tabs) {
        for (int k = 0; k < H; ++k) {
            TablesDev tk;
            tk.upload(&tabs[k], (size_t)nv * U, st);
            toyG[k].dims = GeomDims{1, nv, nx, nt, U, pr->n_te, pr->n_tb, pr->delta_d, pr->a_min, pr->a_max,
                                    pr->gamma, pr->dtg};
            build_geometry(toyG[k], in.plant, in.plans + k, in.v + (size_t)k * nv, in.te, in.tb, in.soc,
                           tk.view, st, &launches);
            ECO_CUDA(cudaStreamSynchronize(st));   // tk freed at scope end
        }
    }
    std::vector<TileCfg> tcs(H);
    for (int k = 0; k < H; ++k) tcs[k] = tile_cfg(tabs ? toyG[k] : G, nt, 0);
    // large outputs (fine grids): overlap each level's D2H with the later
    // stages.  Small stacks go in one copy at the end: per-level pageable
    // copies cost more than they hide (C2: 1.67 vs 1.16 ms per solve call)
    const bool overlap = !tabs && env_int("ECO_DEBUG_STAGE", 0) == 0 &&
                         ns * (size_t)(H + 1) * sizeof(double) > (size_t(256) << 20);
    static cudaStream_t ovs = nullptr;
    static std::vector<cudaEvent_t> lvl_ev;
    if (overlap) {
        if (!ovs) {
            // highest priority: each level's conversion kernel must not queue
            // behind the remaining stages' pending CTAs, or the downloads
            // would trail the whole sweep instead of overlapping it
            int lo_pri = 0, hi_pri = 0;
            ECO_CUDA(cudaDeviceGetStreamPriorityRange(&lo_pri, &hi_pri));
            ECO_CUDA(cudaStreamCreateWithPriority(&ovs, cudaStreamNonBlocking, hi_pri));
        }
        while ((int)lvl_ev.size() < H + 1) {
            cudaEvent_t e;
            ECO_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            lvl_ev.push_back(e);
        }
        ECO_CUDA(cudaEventRecord(lvl_ev[H], st));       // the terminal level is in place
    }
    WriterCheck wchk(ns);
    sweep.start(st);
    for (int k = H - 1; k >= 0; --k) {
        const TileCfg& tc = tcs[k];
        wchk.arm(st);
        StageArgs<Real> a = tabs ? stage_args(toyG[k], 0, in.v + (size_t)k * nv, nt, tc)
                                 : stage_args(G, k, in.v + (size_t)k * nv, nt, tc);
        a.green = in.green + (size_t)k * nt;
        a.dep_ok = in.dep + (size_t)k * nt;
        a.t_dep = in.tdep + (size_t)k * nt;
        a.wait = in.wait + (size_t)k * nt;
        a.flags = in.flags + k;
        a.J_next = d_J.p + (size_t)(k + 1) * LV;
        a.J_next1 = a.J_next + LC;
        a.lc = LC;
        a.J_out = d_J.p + (size_t)k * LV;
        a.J_out1 = a.J_out + LC;
        a.P_out = d_P.p + (size_t)k * ns;
        a.live = count ? d_live.p : nullptr;
        a.src_kind = plans[k].src_kind;
        a.t0 = pr->t0;
        a.dtg = pr->dtg;
        a.j_inf = (Real)pr->j_inf;
        DBuf<unsigned long long> dbgbuf;
        const bool dbg_on = env_int("ECO_DEBUG_STAGE", 0) != 0;
        if (dbg_on) {
            dbgbuf.alloc((size_t)6 * nv * tc.nchunk);
            ECO_CUDA(cudaMemsetAsync(dbgbuf.p, 0, dbgbuf.n * 8, st));
            a.dbg = dbgbuf.p;
        }
        launch_stage<Real, 0>(a, tc, count, st, -1, rev);
        wchk.verify(st);
        if (overlap) ECO_CUDA(cudaEventRecord(lvl_ev[k], st));
        if (dbg_on) {
            std::vector<unsigned long long> h(dbgbuf.n);
            dbgbuf.download(h.data(), h.size(), st);
            ECO_CUDA(cudaStreamSynchronize(st));
            const int nb = nv * tc.nchunk;
            unsigned long long t0 = ~0ull, t1 = 0;
            for (int b = 0; b < nb; ++b) { t0 = std::min(t0, h[6 * b]); t1 = std::max(t1, h[6 * b + 3]); }
            int cta_per_sm = 0;
            if (tc.wide && w2_wpr(nt))
                ECO_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&cta_per_sm, bellman_wide2_kernel<Real, false>,
                                                                       tc.S * tc.slices, tc.smem));
            else if (!tc.wide)
                ECO_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&cta_per_sm, bellman_stage_kernel<Real, false>,
                                                                       tc.S * tc.slices, tc.smem));
            std::fprintf(stderr, "stage k=%d ctas=%d span=%.2fus tile %dx%d slices %d count_max %d band_cap %d smem %zu "
                         "ctas/SM %d\n", k, nb, (t1 - t0) / 1e3, tc.tj, nt, tc.slices, tc.count_max, tc.band_cap,
                         tc.smem, cta_per_sm);
            for (int b = 0; b < nb; ++b)
                std::fprintf(stderr, "  cta %3d sm %3llu path %llu work %5llu start %7.2f staged %7.2f looped %7.2f end %7.2f\n",
                             b, h[6 * b + 4] & 0xFFFF, h[6 * b + 4] >> 16, h[6 * b + 5], (h[6 * b] - t0) / 1e3,
                             h[6 * b + 1] ? (h[6 * b + 1] - t0) / 1e3 : -1.0, (h[6 * b + 2] - t0) / 1e3,
                             (h[6 * b + 3] - t0) / 1e3);
        }
        ++launches;
    }
    sweep.stop(st);
    if (overlap) {
        // level k is final once stage k ran: its conversion and download run
        // on a side stream while the remaining stages sweep
        all.stop(st);
        // pinned destinations: every level's conversion + DMA is enqueued at
        // once (the copy engine streams levels out as the sweep produces
        // them); pageable ones go through download_big's staging per level
        const bool direct = host_pinned(J_stack) && host_pinned(P_stack);
        // fp32 levels cross PCIe as f32 (half the bytes) and are widened to
        // the caller's f64 tables by host threads, level by level while
        // later levels are still in flight: the C3 tables are 9 GB as f64 /
        // int32 and the link (57 GB/s) bounds the solve end to end
        if (sizeof(Real) == 4 && direct && env_int("ECO_HOST_WIDEN", 1) != 0) {
            // every level widened measured best (C3 e2e: all 164 ms, every
            // 2nd 182, none 191): host memory, not the link, bounds the mix
            const int every = std::max(1, env_int("ECO_WIDEN_EVERY", 1));
            widen_levels(reinterpret_cast<const float*>(d_J.p), LV, ns, H, top, pr->j_inf, d_P.p, J_stack, P_stack,
                         lvl_ev, ovs, d_tmp.p, [&](int k) { return (H - k) % every == 0; });
        } else
        for (int k = top; k >= 0; --k) {
            ECO_CUDA(cudaStreamWaitEvent(ovs, lvl_ev[k], 0));
            to_external_levels_kernel<Real><<<grid_for(ns), 256, 0, ovs>>>(d_J.p + (size_t)k * LV,
                                                                           d_tmp.p + (size_t)k * ns, ns, 1,
                                                                           pr->j_inf);
            ECO_CUDA(cudaGetLastError());
            ++launches;
            if (direct) {
                ECO_CUDA(cudaMemcpyAsync(J_stack + (size_t)k * ns, d_tmp.p + (size_t)k * ns, ns * sizeof(double),
                                         cudaMemcpyDeviceToHost, ovs));
                if (k < H)
                    ECO_CUDA(cudaMemcpyAsync(P_stack + (size_t)k * ns, d_P.p + (size_t)k * ns, ns * sizeof(int32_t),
                                             cudaMemcpyDeviceToHost, ovs));
                continue;
            }
            download_big(J_stack + (size_t)k * ns, d_tmp.p + (size_t)k * ns, ns * sizeof(double), ovs);
            if (k < H) download_big(P_stack + (size_t)k * ns, d_P.p + (size_t)k * ns, ns * sizeof(int32_t), ovs);
        }
        ECO_CUDA(cudaStreamSynchronize(ovs));
        if (dbg_io) {
            const auto h2 = std::chrono::steady_clock::now();
            std::fprintf(stderr, "io: upload(host) %.2f ms, all %.2f ms, direct=%d, outputs done at %.2f ms after "
                                 "the upload\n",
                         std::chrono::duration<double, std::milli>(h1 - h0).count(), all.ms(), direct ? 1 : 0,
                         std::chrono::duration<double, std::milli>(h2 - h1).count());
        }
    } else {
        to_external_levels_kernel<Real><<<grid_for(ns * (top + 1)), 256, 0, st>>>(d_J.p, d_tmp.p, ns, top + 1,
                                                                                 pr->j_inf);
        ECO_CUDA(cudaGetLastError());
        ++launches;
        all.stop(st);
        download_big(J_stack, d_tmp.p, ns * (top + 1) * sizeof(double), st);
        download_big(P_stack, d_P.p, ns * H * sizeof(int32_t), st);
    }
    unsigned long long live = 0;
    ECO_CUDA(cudaMemcpyAsync(&live, d_live.p, sizeof live, cudaMemcpyDeviceToHost, st));
    ECO_CUDA(cudaStreamSynchronize(st));
    sweep_ms = sweep.ms();
    if (stats) {
        stats->device_ms = all.ms();
        stats->dominant_ms = sweep_ms;
        stats->dense_updates = (int64_t)ns * U * H;
        stats->live_updates = count ? (int64_t)live : -1;
        stats->stages = H;
        stats->kernel_launches = launches;
    }
}

template <typename F>
int run_guarded(F&& f) {
    try {
        int n = 0;
        if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
            g_err = "no CUDA device visible";
            return ECO_ERR_NODEV;
        }
        f();
        return ECO_OK;
    } catch (const ArgError& a) {
        g_err = a.msg;
        return ECO_ERR_ARG;
    } catch (const CudaError& c) {
        g_err = std::string(c.what) + ": " + cudaGetErrorString(c.e);
        return ECO_ERR_CUDA;
    } catch (const std::exception& e) {
        g_err = e.what();
        return ECO_ERR_CUDA;
    }
}

// ------------------------------------------------------------- route side
struct RouteDev {
    DBuf<double> v_min, v_max, grade, cos_g, sin_g, cycle, offset, win, vaxes;
    DBuf<int8_t> kinds;
    DBuf<int32_t> nwin;
    DevRoute view{};
    std::vector<double> h_vaxes;

    void upload(const EcoRoute* r, int nv, cudaStream_t s) {
        const int n = r->node_count;
        if (n < 2) throw ArgError{"route needs >= 2 nodes"};
        if (!r->v_min || !r->v_max || !r->grade || !r->cos_grade || !r->sin_grade || !r->kinds || !r->sig_cycle ||
            !r->sig_offset || !r->sig_nwin || !r->sig_win)
            throw ArgError{"null route array"};
        // ensure(): a re-upload of a same-sized route keeps every device
        // pointer (captured CUDA graphs stay valid)
        v_min.ensure(n); v_max.ensure(n); grade.ensure(n); cos_g.ensure(n); sin_g.ensure(n);
        cycle.ensure(n); offset.ensure(n); win.ensure((size_t)n * ECO_MAX_WINDOWS * 2);
        kinds.ensure(n); nwin.ensure(n); vaxes.ensure((size_t)n * nv);
        v_min.upload(r->v_min, n, s); v_max.upload(r->v_max, n, s); grade.upload(r->grade, n, s);
        cos_g.upload(r->cos_grade, n, s); sin_g.upload(r->sin_grade, n, s);
        cycle.upload(r->sig_cycle, n, s); offset.upload(r->sig_offset, n, s);
        win.upload(r->sig_win, (size_t)n * ECO_MAX_WINDOWS * 2, s);
        kinds.upload(r->kinds, n, s); nwin.upload(r->sig_nwin, n, s);
        // GridSpec.v_axis dp.py:68-69 = np.linspace(v_min, v_max, n_v)
        h_vaxes.resize((size_t)n * nv);
        for (int m = 0; m < n; ++m) {
            const double a = r->v_min[m], b = r->v_max[m];
            const double step = (b - a) / (double)(nv - 1);
            for (int i = 0; i < nv; ++i) h_vaxes[(size_t)m * nv + i] = (double)i * step + a;
            h_vaxes[(size_t)m * nv + nv - 1] = b;
        }
        vaxes.upload(h_vaxes.data(), h_vaxes.size(), s);
        view = DevRoute{n, r->delta_d, r->accel_min, r->accel_max, r->stop_dwell, v_min.p, v_max.p, grade.p,
                        cos_g.p, sin_g.p, kinds.p, cycle.p, offset.p, nwin.p, win.p};
    }
};

// route-level plans: plan m = step m -> m+1 for m = 0..n-2
std::vector<DevPlan> route_plans(const EcoRoute* r, const std::vector<double>& vaxes, int nv) {
    const int n = r->node_count;
    std::vector<DevPlan> out(n - 1);
    for (int m = 0; m < n - 1; ++m) {
        DevPlan d;
        d.src_kind = r->kinds[m];
        d.dest_kind = r->kinds[m + 1];
        d.cos_g = r->cos_grade[m];
        d.sin_g = r->sin_grade[m];
        const double* vd = &vaxes[(size_t)(m + 1) * nv];
        d.v0d = vd[0];
        d.dvd = (vd[nv - 1] - vd[0]) / (nv - 1);
        out[m] = d;
    }
    return out;
}

// build_terminal_cost mpc.py:96-158 destination row
__global__ void field_init_kernel(const double* soc, const double* v_end, int nv, int nx, double target, double weight,
                                  double j_inf, int stop_end, double* G_ext) {
    for (int i = threadIdx.x + blockIdx.x * blockDim.x; i < nv * nx; i += blockDim.x * gridDim.x) {
        const int iv = i / nx, jx = i - iv * nx;
        const double d = soc[jx] - target;
        double q = weight * (d * d);
        if (!(q < j_inf)) q = j_inf;    // np.minimum(quad, j_inf)
        if (stop_end && v_end[iv] > 0.0) q = j_inf;
        G_ext[i] = q;
    }
}

// build_terminal_cost mpc.py:96-158 on the device: N-1 (v, soc) sweeps.
// Replayable capture of the N-1 field launches (per session).
struct FieldGraph {
    cudaGraphExec_t exec = nullptr;
    std::vector<long long> key;
    ~FieldGraph() {
        if (exec) cudaGraphExecDestroy(exec);
    }
};

// chunk (nullable): geometry on demand -- chunk(m0, m1) builds plans
// [m0, m1) into G (plan m at index m - m0) for grids whose all-route
// geometry does not fit; the sweep then walks the route backwards chunk by
// chunk, chunk_plans plans at a time (no graph: the builds sync the host).
template <typename Real>
void field_build_impl(const int8_t* kinds, int n, double dwell, const EcoMpcConfig* c, Geometry<Real>& G,
                      RouteDev& R, const double* d_soc, DBuf<Real>& d_G, DBuf<double>& d_field_ext,
                      cudaStream_t st, int64_t* launches, double* sweep_ms, FieldGraph* fg = nullptr,
                      const std::function<void(int, int)>& chunk = {}, int chunk_plans = 0) {
    const int nv = c->n_v, nx = c->n_soc;
    const size_t lvl = (size_t)nv * nx;
    field_init_kernel<<<1, 256, 0, st>>>(d_soc, R.vaxes.p + (size_t)(n - 1) * nv, nv, nx, c->soc_target,
                                         c->soc_weight, c->j_inf, kinds[n - 1] == ECO_NODE_STOP ? 1 : 0,
                                         d_field_ext.p + (size_t)(n - 1) * lvl);
    to_internal_kernel<Real><<<grid_for(lvl), 256, 0, st>>>(d_field_ext.p + (size_t)(n - 1) * lvl,
                                                            d_G.p + (size_t)(n - 1) * lvl, lvl, c->j_inf);
    ECO_CUDA(cudaGetLastError());
    *launches += 2;
    // stages s = s_hi - 1 .. s_lo of the sweep; plan s sits at index s - base of G
    auto enqueue = [&](cudaStream_t qs, int s_lo, int s_hi, int base) {
        const TileCfg tc = tile_cfg(G, 1, 1);
        for (int s = s_hi - 1; s >= s_lo; --s) {
            StageArgs<Real> a = stage_args(G, s - base, R.vaxes.p + (size_t)s * nv, 1, tc);
            a.J_next = d_G.p + (size_t)(s + 1) * lvl;
            a.J_out = d_G.p + (size_t)s * lvl;
            a.P_out = nullptr;
            // always-green field: a light is an ordinary launch point (mpc.py:141-142)
            a.src_kind = kinds[s] == ECO_NODE_SIGNAL ? ECO_NODE_PLAIN : kinds[s];
            a.dwell = dwell;
            a.j_inf = (Real)c->j_inf;
            launch_stage<Real, 1>(a, tc, false, qs);
        }
    };
    double ms = 0.0;
    if (chunk) {
        const int C = std::max(1, chunk_plans);
        for (int m1 = n - 1; m1 > 0;) {
            const int m0 = std::max(0, m1 - C);
            chunk(m0, m1);
            EventTimer tm;
            tm.start(st);
            enqueue(st, m0, m1, m0);
            tm.stop(st);
            ms += tm.ms();
            m1 = m0;
        }
    } else if (fg && st && env_int("ECO_GRAPH", 1) != 0) {
        // the N-1 launches as one graph (captured once per geometry / buffers)
        const TileCfg tc = tile_cfg(G, 1, 1);
        const std::vector<long long> key = {(long long)(size_t)G.act.p, (long long)(size_t)G.row.p,
                                            (long long)(size_t)d_G.p, tc.slices, n};
        if (!fg->exec || fg->key != key) {
            if (fg->exec) { cudaGraphExecDestroy(fg->exec); fg->exec = nullptr; }
            cudaGraph_t graph;
            ECO_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
            enqueue(st, 0, n - 1, 0);
            ECO_CUDA(cudaStreamEndCapture(st, &graph));
            ECO_CUDA(cudaGraphInstantiate(&fg->exec, graph, 0));
            cudaGraphDestroy(graph);
            fg->key = key;
        }
        EventTimer tm;
        tm.start(st);
        ECO_CUDA(cudaGraphLaunch(fg->exec, st));
        tm.stop(st);
        ms = tm.ms();
    } else {
        EventTimer tm;
        tm.start(st);
        enqueue(st, 0, n - 1, 0);
        tm.stop(st);
        ms = tm.ms();
    }
    *launches += n - 1;
    to_external_kernel<Real><<<grid_for((size_t)(n - 1) * lvl), 256, 0, st>>>(d_G.p, d_field_ext.p,
                                                                             (size_t)(n - 1) * lvl, c->j_inf);
    ECO_CUDA(cudaGetLastError());
    ++*launches;
    if (sweep_ms) *sweep_ms += ms;
}

void check_cfg(const EcoMpcConfig* c) {
    if (!c) throw ArgError{"null config"};
    if (c->n_v < 2 || c->n_soc < 2 || c->n_t < 2 || c->n_te < 1 || c->n_tb < 1 || c->horizon < 1)
        throw ArgError{"invalid grid / horizon"};
    if (c->n_soc > 32767) throw ArgError{"n_soc must be < 32768"};
    if (!(c->gamma >= 0.0 && c->gamma <= 1.0)) throw ArgError{"gamma must lie in [0, 1]"};
    if (!(c->dt > 0.0)) throw ArgError{"dt must be positive"};
    if (c->start_node < 0) throw ArgError{"start_node must be >= 0"};
    if (!c->te_axis || !c->tb_axis) throw ArgError{"null action axis"};
}

std::vector<double> soc_axis(const EcoPlant* p, int nx) {
    std::vector<double> s(nx);
    const double step = (p->soc_max - p->soc_min) / (double)(nx - 1);
    for (int i = 0; i < nx; ++i) s[i] = (double)i * step + p->soc_min;
    s[nx - 1] = p->soc_max;
    return s;
}

// Route-level context shared by field build and closed loop.
template <typename Real>
struct RouteCtx {
    DBuf<EcoPlant> plant;
    RouteDev R;
    DBuf<DevPlan> plans;
    DBuf<double> te, tb, soc;
    std::vector<double> h_soc;
    Geometry<Real> G;

    // ring: no all-route geometry (fine grids build plans on demand)
    void init(const EcoPlant* p, const EcoRoute* r, const EcoMpcConfig* c, cudaStream_t st, bool ring = false) {
        plant.alloc(1);
        plant.upload(p, 1, st);
        R.upload(r, c->n_v, st);
        std::vector<DevPlan> hp = route_plans(r, R.h_vaxes, c->n_v);
        plans.alloc(hp.size());
        plans.upload(hp.data(), hp.size(), st);
        te.alloc(c->n_te); tb.alloc(c->n_tb);
        te.upload(c->te_axis, c->n_te, st);
        tb.upload(c->tb_axis, c->n_tb, st);
        h_soc = soc_axis(p, c->n_soc);
        soc.alloc(c->n_soc);
        soc.upload(h_soc.data(), c->n_soc, st);
        G.dims = GeomDims{r->node_count - 1, c->n_v, c->n_soc, c->n_t, c->n_te * c->n_tb, c->n_te, c->n_tb,
                          r->delta_d, r->accel_min, r->accel_max, c->gamma, c->dt};
        if (!ring) G.alloc(G.dims.P, G.dims.nv, G.dims.U);
    }
    // new route data of the same shape (speed limits, grades, node kinds,
    // signal programs): arrays re-uploaded in place, plans rebuilt
    void reupload(const EcoRoute* r, const EcoMpcConfig* c, cudaStream_t st) {
        R.upload(r, c->n_v, st);
        std::vector<DevPlan> hp = route_plans(r, R.h_vaxes, c->n_v);
        plans.upload(hp.data(), hp.size(), st);
        G.dims.delta_d = r->delta_d;
        G.dims.a_min = r->accel_min;
        G.dims.a_max = r->accel_max;
        ECO_CUDA(cudaStreamSynchronize(st));
    }
    // route-level geometry: stage-1 + SoC cells of every spatial step
    void geometry(cudaStream_t st, int64_t* launches) {
        EcoStage1Tables none{};
        build_geometry(G, plant.p, plans.p, R.vaxes.p, te.p, tb.p, soc.p, none, st, launches);
    }
};

// ------------------------------------------------------------- sessions
// A session owns everything one route needs on the device: the uploaded
// route / plant, the route-level geometry (one plan per spatial step), the
// terminal field and the loop buffers.  create() only allocates and uploads;
// fit() computes geometry + field (EcoDrivingMPC.fit, mpc.py:379-391);
// run() drives the closed loop (simulate_closed_loop, mpc.py:513-596).
struct SessionBase {
    int precision = 0;
    virtual ~SessionBase() = default;
    virtual void upload_route(const EcoRoute* r) = 0;
    virtual void fit(const double* field_in, double* field_out, EcoStats* stats) = 0;
    virtual void run(int start_node, int max_steps, const double* x0, EcoTrajRow* rows, int32_t* n_rows,
                     int32_t* status, int32_t* status_node, double* final_state, int flags, EcoStats* stats) = 0;
    virtual void step_times(double* out_ms, int n) = 0;
};

constexpr int kRunCountLive = 1;

template <typename Real>
struct Session : SessionBase {
    EcoMpcConfig cfg{};
    std::vector<double> te_h, tb_h;
    std::vector<int8_t> kinds;
    int n = 0;
    double stop_dwell = 0.0;
    RouteCtx<Real> ctx;
    DBuf<double> field;            // external f64 (n, nv, nx)
    DBuf<Real> field_int;          // internal (n, nv, nx)
    bool fitted = false;
    DBuf<LoopState> state;
    DBuf<unsigned long long> step_ns;   // per-step solve clocks of the last run
    int last_rows = 0;
    DBuf<DecideCand> dec_cand;      // split decide: per-action candidate records
    DBuf<DecideHead> dec_head;
    cudaStream_t dec_side = nullptr;
    cudaEvent_t dec_fork = nullptr, dec_join = nullptr;
    DBuf<uint8_t> green, dep;
    DBuf<double> tdep, wait, tax;
    DBuf<int> sflags;              // kStageAny* per stage of the current solve
    DBuf<Real> J;
    DBuf<EcoTrajRow> rows;
    DBuf<unsigned long long> live;
    cudaStream_t st = 0;
    // CUDA graph of a whole closed loop (prepare / H stage sweeps / decide per
    // node), captured on first use and replayed: no per-kernel launch gaps
    cudaGraphExec_t gexec = nullptr;
    std::vector<long long> gkey;
    FieldGraph fgraph;             // the terminal-field sweep, replayed per fit
    // Ring mode (grids whose all-route geometry does not fit in HBM, e.g. the
    // C3 grid: ~0.3 GB of records per plan, 699 plans): the H + 1 plans a
    // receding-horizon step can touch live in a ring of slots; plan s + H is
    // built on a side stream while step s sweeps, into the slot plan s - 1
    // vacated.  The terminal field is swept chunk by chunk.
    bool ring = false;
    std::vector<std::unique_ptr<Geometry<Real>>> slots;
    std::vector<int> slot_plan;
    std::vector<cudaEvent_t> slot_ev;
    Geometry<Real> fieldG;
    int field_chunk = 1;
    cudaStream_t geo_st = nullptr;
    cudaEvent_t stage_ev[2] = {nullptr, nullptr};
    int32_t* h_status = nullptr;   // pinned mirror of the loop status, per step parity

    static bool decide_ring(const EcoMpcConfig* c, int n) {
        const int forced = env_int("ECO_RING", -1);
        if (forced >= 0) return forced != 0;
        const double U = (double)c->n_te * c->n_tb;
        // records of all plans at ~35 % feasible (plan, plane, action, SoC row)
        const double est = (double)(n - 1) * c->n_v * U * (44.0 + 0.35 * c->n_soc * 32.0);
        size_t fr = 0, tot = 0;
        if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) return est > 40e9;
        return est > 0.3 * (double)fr;
    }

    Session(const EcoPlant* p, const EcoRoute* r, const EcoMpcConfig* c) {
        cfg = *c;
        te_h.assign(c->te_axis, c->te_axis + c->n_te);
        tb_h.assign(c->tb_axis, c->tb_axis + c->n_tb);
        cfg.te_axis = te_h.data();
        cfg.tb_axis = tb_h.data();
        n = r->node_count;
        kinds.assign(r->kinds, r->kinds + n);
        stop_dwell = r->stop_dwell;
        ring = decide_ring(c, n);
        ctx.init(p, r, &cfg, st, ring);
        if (ring) {
            const int H1 = c->horizon + 1;
            slots.resize(H1);
            for (auto& g : slots) g = std::make_unique<Geometry<Real>>();
            slot_plan.assign(H1, -1);
            slot_ev.resize(H1);
            for (auto& e : slot_ev) ECO_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            for (auto& e : stage_ev) ECO_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            ECO_CUDA(cudaStreamCreateWithFlags(&geo_st, cudaStreamNonBlocking));
            ECO_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&h_status), 2 * sizeof(int32_t), cudaHostAllocDefault));
            const double per_plan = (double)c->n_v * c->n_te * c->n_tb * (44.0 + 0.35 * c->n_soc * 16.0);
            field_chunk = (int)std::max(1.0, std::min((double)(n - 1), 8e9 / per_plan));
        }
        const int nv = cfg.n_v, nx = cfg.n_soc, nt = cfg.n_t, H = cfg.horizon;
        const size_t ns = (size_t)nv * nx * nt;
        field.alloc((size_t)n * nv * nx);
        field_int.alloc((size_t)n * nv * nx);
        state.alloc(1);
        green.alloc((size_t)(H + 1) * nt); dep.alloc((size_t)(H + 1) * nt);
        tdep.alloc((size_t)(H + 1) * nt); wait.alloc((size_t)(H + 1) * nt); tax.alloc(nt);
        sflags.alloc(H);
        J.alloc((size_t)2 * (H + 1) * level_stride(ns));   // two stacks, alternating by step
        rows.alloc(n - 1);
        live.alloc(1);
        ECO_CUDA(cudaStreamSynchronize(st));
        // a blocking stream of its own (stream capture is impossible on the
        // legacy default stream; blocking keeps it ordered with stream 0)
        ECO_CUDA(cudaStreamCreate(&st));
    }
    ~Session() override {
        for (auto& e : slot_ev) if (e) cudaEventDestroy(e);
        for (auto& e : stage_ev) if (e) cudaEventDestroy(e);
        if (geo_st) cudaStreamDestroy(geo_st);
        if (h_status) cudaFreeHost(h_status);
        if (gexec) cudaGraphExecDestroy(gexec);
        if (dec_fork) cudaEventDestroy(dec_fork);
        if (dec_join) cudaEventDestroy(dec_join);
        if (dec_side) cudaStreamDestroy(dec_side);
        if (st) cudaStreamDestroy(st);
    }

    void step_times(double* out_ms, int n_req) override {
        if (n_req < 0 || n_req > last_rows) throw ArgError{"more step times requested than the last run took"};
        std::vector<unsigned long long> h((size_t)n_req);
        if (n_req) step_ns.download(h.data(), (size_t)n_req, st);
        ECO_CUDA(cudaStreamSynchronize(st));
        for (int i = 0; i < n_req; ++i) out_ms[i] = (double)h[i] * 1e-6;
    }

    void upload_route(const EcoRoute* r) override {
        if (r->node_count != n) throw ArgError{"route node count differs from the session's"};
        if (!r->kinds) throw ArgError{"null route array"};
        // node kinds, dwell, spacing and comfort box are kernel arguments
        // baked into the captured graphs (ctx.R.view is passed by value)
        const bool same_kinds = std::equal(kinds.begin(), kinds.end(), r->kinds) && stop_dwell == r->stop_dwell &&
                                r->delta_d == ctx.R.view.delta_d && r->accel_min == ctx.R.view.accel_min &&
                                r->accel_max == ctx.R.view.accel_max;
        ctx.reupload(r, &cfg, st);
        kinds.assign(r->kinds, r->kinds + n);
        stop_dwell = r->stop_dwell;
        if (!same_kinds) {
            if (gexec) { cudaGraphExecDestroy(gexec); gexec = nullptr; }
            gkey.clear();
            if (fgraph.exec) { cudaGraphExecDestroy(fgraph.exec); fgraph.exec = nullptr; }
            fgraph.key.clear();
        }
        fitted = false;              // geometry and field depend on the route
    }

    // plans [m0, m1) into G (P = m1 - m0), from the uploaded route
    void build_plans(Geometry<Real>& G, int m0, int m1, cudaStream_t qs, int64_t* launches, bool tiles) {
        G.dims = ctx.G.dims;
        G.dims.P = m1 - m0;
        EcoStage1Tables none{};
        build_geometry(G, ctx.plant.p, ctx.plans.p + m0, ctx.R.vaxes.p + (size_t)m0 * cfg.n_v, ctx.te.p, ctx.tb.p,
                       ctx.soc.p, none, qs, launches, tiles);
    }

    void fit(const double* field_in, double* field_out, EcoStats* stats) override {
        int64_t launches = 0;
        EventTimer all;
        all.start(st);
        if (!ring) ctx.geometry(st, &launches);
        else std::fill(slot_plan.begin(), slot_plan.end(), -1);     // the route may have changed
        double sweep_ms = 0.0;
        const size_t lvl = (size_t)cfg.n_v * cfg.n_soc;
        if (cfg.use_terminal_field) {
            if (field_in) field.upload(field_in, (size_t)n * lvl, st);
            else if (ring)
                field_build_impl<Real>(kinds.data(), n, stop_dwell, &cfg, fieldG, ctx.R, ctx.soc.p, field_int, field,
                                       st, &launches, &sweep_ms, nullptr,
                                       [&](int m0, int m1) { build_plans(fieldG, m0, m1, st, &launches, false); },
                                       field_chunk);
            else field_build_impl<Real>(kinds.data(), n, stop_dwell, &cfg, ctx.G, ctx.R, ctx.soc.p, field_int,
                                        field, st, &launches, &sweep_ms, &fgraph);
        }
        all.stop(st);
        if (field_out && cfg.use_terminal_field) field.download(field_out, (size_t)n * lvl, st);
        ECO_CUDA(cudaStreamSynchronize(st));
        fitted = true;
        if (stats) {
            stats->device_ms = all.ms();
            stats->dominant_ms = sweep_ms;
            stats->dense_updates = (cfg.use_terminal_field && !field_in)
                                       ? (int64_t)(n - 1) * cfg.n_v * cfg.n_soc * cfg.n_te * cfg.n_tb : 0;
            stats->live_updates = -1;
            stats->stages = (cfg.use_terminal_field && !field_in) ? n - 1 : 0;
            stats->kernel_launches = launches;
        }
    }

    void run(int start_node, int max_steps, const double* x0, EcoTrajRow* out_rows, int32_t* n_rows,
             int32_t* status, int32_t* status_node, double* final_state, int flags, EcoStats* stats) override {
        if (!fitted) throw ArgError{"session not fitted: call eco_session_fit first"};
        if (start_node < 0 || start_node > n - 2) throw ArgError{"start_node out of range"};
        const int nv = cfg.n_v, nx = cfg.n_soc, nt = cfg.n_t, H = cfg.horizon;
        const int U = cfg.n_te * cfg.n_tb;
        const size_t ns = (size_t)nv * nx * nt;
        const bool count = flags & kRunCountLive;
        int64_t launches = 0;
        LoopState h0{};
        h0.x[0] = x0[0]; h0.x[1] = x0[1]; h0.x[2] = x0[2];
        EventTimer all;
        Ladders lad{green.p, dep.p, tdep.p, wait.p, tax.p, sflags.p};
        LoopCfg lc{nv, nx, nt, cfg.n_te, cfg.n_tb, U, H, cfg.teleport, cfg.use_terminal_field, cfg.dt, cfg.gamma,
                   cfg.soc_target, cfg.soc_weight, cfg.j_inf, ctx.te.p, ctx.tb.p, ctx.soc.p, ctx.R.vaxes.p};
        const int s_end = max_steps < 0 ? n - 1 : std::min(n - 1, start_node + max_steps);
        const TileCfg tc = ring ? TileCfg{} : tile_cfg(ctx.G, nt, 0);
        if (!dec_side) {
            ECO_CUDA(cudaStreamCreateWithFlags(&dec_side, cudaStreamNonBlocking));
            ECO_CUDA(cudaEventCreateWithFlags(&dec_fork, cudaEventDisableTiming));
            ECO_CUDA(cudaEventCreateWithFlags(&dec_join, cudaEventDisableTiming));
        }
        dec_cand.ensure((size_t)U);
        dec_head.ensure(1);
        step_ns.ensure((size_t)n);
        int64_t stages = 0;
        auto enqueue = [&](cudaStream_t qs) {
            stages = 0;
            launches = 0;
            const size_t LV = level_stride(ns), LC = level_copy(ns);
            const int seed_grid = std::max(1, (int)std::min<size_t>(148, (ns + 255) / 256));
            const double* fld = cfg.use_terminal_field ? (const double*)field.p : nullptr;
            // two J stacks, alternating by step: step s + 1's terminal level is
            // seeded on the side branch while step s still sweeps its own
            auto Jstack = [&](int s) { return J.p + (size_t)((s - start_node) & 1) * (H + 1) * LV; };
            auto horizon = [&](int s) { return H < n - 1 - s ? H : n - 1 - s; };
            for (int s = start_node; s < s_end; ++s) {
                const int h = horizon(s);
                Real* Js = Jstack(s);
                if (s == start_node) {
                    mpc_ladders_kernel<<<1, 256, 0, qs>>>(ctx.R.view, lc, state.p, s, h, lad);
                    mpc_seed_kernel<Real><<<seed_grid, 256, 0, qs>>>(lc, s, h, fld, Js + (size_t)h * LV,
                                                                     Js + (size_t)h * LV + LC);
                    ECO_CUDA(cudaGetLastError());
                    launches += 2;
                }
                // beside the sweeps: the J-independent half of the decision and
                // the next step's terminal level
                ECO_CUDA(cudaEventRecord(dec_fork, qs));
                ECO_CUDA(cudaStreamWaitEvent(dec_side, dec_fork, 0));
                mpc_candidates_kernel<<<(U + kCandThreads - 1) / kCandThreads, kCandThreads, 0, dec_side>>>(
                    ctx.plant.p, ctx.R.view, lc, state.p, s, lad, dec_cand.p, dec_head.p);
                ++launches;
                if (s + 1 < s_end) {
                    const int h1 = horizon(s + 1);
                    Real* Jn = Jstack(s + 1);
                    mpc_seed_kernel<Real><<<seed_grid, 256, 0, dec_side>>>(lc, s + 1, h1, fld, Jn + (size_t)h1 * LV,
                                                                          Jn + (size_t)h1 * LV + LC);
                    ++launches;
                }
                ECO_CUDA(cudaGetLastError());
                ECO_CUDA(cudaEventRecord(dec_join, dec_side));
                for (int k = h - 1; k >= 0; --k) {
                    StageArgs<Real> a = stage_args(ctx.G, s + k, ctx.R.vaxes.p + (size_t)(s + k) * nv, nt, tc);
                    a.green = green.p + (size_t)(k + 1) * nt;
                    a.dep_ok = dep.p + (size_t)k * nt;
                    a.t_dep = tdep.p + (size_t)k * nt;
                    a.wait = wait.p + (size_t)k * nt;
                    a.J_next = Js + (size_t)(k + 1) * LV;
                    a.J_next1 = a.J_next + LC;
                    a.lc = LC;
                    a.J_out = Js + (size_t)k * LV;
                    // the shifted copy only serves unstaged tiles (global-memory pair loads)
                    a.J_out1 = ctx.G.all_staged ? nullptr : a.J_out + LC;
                    // the closed loop decides at the exact state from J_1
                    // (mpc.py:189-278): no policy table is needed
                    a.P_out = nullptr;
                    a.status = &state.p->status;
                    a.live = count ? live.p : nullptr;
                    a.src_kind = kinds[s + k];
                    a.flags = sflags.p + k;
                    a.t0_dev = tax.p;   // ladder origin depends on the device-resident clock
                    a.dtg = cfg.dt;
                    a.j_inf = (Real)cfg.j_inf;
                    launch_stage<Real, 0>(a, tc, count, qs);
                    ++launches;
                    ++stages;
                }
                ECO_CUDA(cudaStreamWaitEvent(qs, dec_join, 0));
                const int s_next = s + 1 < s_end ? s + 1 : -1;
                launch_pdl(mpc_pick_kernel<Real>, 1, std::min(kDecideThreads, (U + 31) / 32 * 32), qs, true,
                           (const EcoPlant*)ctx.plant.p, ctx.R.view, lc, state.p, s, h, (const Real*)(Js + LV),
                           (const DecideCand*)dec_cand.p, (const DecideHead*)dec_head.p, lad, rows.p, step_ns.p,
                           s_next, s_next < 0 ? 0 : horizon(s_next));
                ECO_CUDA(cudaGetLastError());
                ++launches;
            }
        };
        // ring mode: the same per-step sequence, launched directly (plan
        // builds sync the host: no graph), the geometry of the step's new
        // plan built beside the previous step's sweeps
        auto ring_enqueue = [&]() {
            stages = 0;
            launches = 0;
            const size_t LV = level_stride(ns), LC = level_copy(ns);
            const int seed_grid = std::max(1, (int)std::min<size_t>(148, (ns + 255) / 256));
            const double* fld = cfg.use_terminal_field ? (const double*)field.p : nullptr;
            auto Jstack = [&](int s) { return J.p + (size_t)((s - start_node) & 1) * (H + 1) * LV; };
            auto horizon = [&](int s) { return H < n - 1 - s ? H : n - 1 - s; };
            const int H1 = H + 1;
            auto ensure_plan = [&](int m, cudaStream_t qs) {
                const int j = m % H1;
                if (slot_plan[j] == m) return;
                slot_plan[j] = -1;
                build_plans(*slots[j], m, m + 1, qs, &launches, true);
                slot_plan[j] = m;
                ECO_CUDA(cudaEventRecord(slot_ev[j], qs));
            };
            ECO_CUDA(cudaStreamSynchronize(geo_st));     // a previous run's last plan build
            for (int m = start_node; m < start_node + horizon(start_node); ++m) ensure_plan(m, st);
            h_status[0] = h_status[1] = 0;
            for (int s = start_node; s < s_end; ++s) {
                // the device loop stopped (infeasible / plant failure): the
                // status of step s - 2 has reached the host by now
                if (s - start_node >= 2 && h_status[s & 1] != 0) break;
                const int h = horizon(s);
                Real* Js = Jstack(s);
                if (s == start_node) {
                    mpc_ladders_kernel<<<1, 256, 0, st>>>(ctx.R.view, lc, state.p, s, h, lad);
                    mpc_seed_kernel<Real><<<seed_grid, 256, 0, st>>>(lc, s, h, fld, Js + (size_t)h * LV,
                                                                     Js + (size_t)h * LV + LC);
                    ECO_CUDA(cudaGetLastError());
                    launches += 2;
                }
                ECO_CUDA(cudaEventRecord(dec_fork, st));
                ECO_CUDA(cudaStreamWaitEvent(dec_side, dec_fork, 0));
                mpc_candidates_kernel<<<(U + kCandThreads - 1) / kCandThreads, kCandThreads, 0, dec_side>>>(
                    ctx.plant.p, ctx.R.view, lc, state.p, s, lad, dec_cand.p, dec_head.p);
                ++launches;
                if (s + 1 < s_end) {
                    const int h1 = horizon(s + 1);
                    Real* Jn = Jstack(s + 1);
                    mpc_seed_kernel<Real><<<seed_grid, 256, 0, dec_side>>>(lc, s + 1, h1, fld, Jn + (size_t)h1 * LV,
                                                                          Jn + (size_t)h1 * LV + LC);
                    ++launches;
                }
                ECO_CUDA(cudaGetLastError());
                ECO_CUDA(cudaEventRecord(dec_join, dec_side));
                for (int m = s; m < s + h; ++m) ECO_CUDA(cudaStreamWaitEvent(st, slot_ev[m % H1], 0));
                for (int k = h - 1; k >= 0; --k) {
                    Geometry<Real>& G = *slots[(s + k) % H1];
                    const TileCfg tk = tile_cfg(G, nt, 0);
                    StageArgs<Real> a = stage_args(G, 0, ctx.R.vaxes.p + (size_t)(s + k) * nv, nt, tk);
                    a.green = green.p + (size_t)(k + 1) * nt;
                    a.dep_ok = dep.p + (size_t)k * nt;
                    a.t_dep = tdep.p + (size_t)k * nt;
                    a.wait = wait.p + (size_t)k * nt;
                    a.J_next = Js + (size_t)(k + 1) * LV;
                    a.J_next1 = a.J_next + LC;
                    a.lc = LC;
                    a.J_out = Js + (size_t)k * LV;
                    a.J_out1 = G.all_staged ? nullptr : a.J_out + LC;
                    a.P_out = nullptr;
                    a.status = &state.p->status;
                    a.live = count ? live.p : nullptr;
                    a.src_kind = kinds[s + k];
                    a.flags = sflags.p + k;
                    a.t0_dev = tax.p;
                    a.dtg = cfg.dt;
                    a.j_inf = (Real)cfg.j_inf;
                    launch_stage<Real, 0>(a, tk, count, st);
                    ++launches;
                    ++stages;
                }
                ECO_CUDA(cudaEventRecord(stage_ev[s & 1], st));
                ECO_CUDA(cudaStreamWaitEvent(st, dec_join, 0));
                const int s_next = s + 1 < s_end ? s + 1 : -1;
                launch_pdl(mpc_pick_kernel<Real>, 1, std::min(kDecideThreads, (U + 31) / 32 * 32), st, true,
                           (const EcoPlant*)ctx.plant.p, ctx.R.view, lc, state.p, s, h, (const Real*)(Js + LV),
                           (const DecideCand*)dec_cand.p, (const DecideHead*)dec_head.p, lad, rows.p, step_ns.p,
                           s_next, s_next < 0 ? 0 : horizon(s_next));
                ECO_CUDA(cudaGetLastError());
                ++launches;
                ECO_CUDA(cudaMemcpyAsync(h_status + (s & 1), &state.p->status, sizeof(int32_t),
                                         cudaMemcpyDeviceToHost, st));
                // the plan step s + 1 adds, built while step s sweeps, into the
                // slot plan s - 1 held (free once step s - 1's sweeps are done)
                if (s + 1 < s_end) {
                    const int m = s + horizon(s + 1);
                    if (slot_plan[m % H1] != m) {
                        ECO_CUDA(cudaStreamWaitEvent(geo_st, stage_ev[(s - 1) & 1], 0));
                        ensure_plan(m, geo_st);
                    }
                }
            }
        };
        const bool use_graph = !ring && !count && env_int("ECO_GRAPH", 1) != 0;
        if (ring) {
            all.start(st);
            state.upload(&h0, 1, st);
            if (count) ECO_CUDA(cudaMemsetAsync(live.p, 0, sizeof(unsigned long long), st));
            ring_enqueue();
        } else if (use_graph) {
            const std::vector<long long> key = {start_node, s_end, (long long)(size_t)ctx.G.row2.p,
                                                (long long)(size_t)ctx.G.tiles.p, (long long)(size_t)ctx.G.order.p,
                                                (long long)(size_t)field.p, tc.tj, tc.slices,
                                                ctx.G.all_staged ? 1 : 0};
            if (!gexec || key != gkey) {
                if (gexec) { cudaGraphExecDestroy(gexec); gexec = nullptr; }
                cudaGraph_t graph;
                ECO_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
                enqueue(st);
                ECO_CUDA(cudaStreamEndCapture(st, &graph));
                ECO_CUDA(cudaGraphInstantiate(&gexec, graph, 0));
                cudaGraphDestroy(graph);
                gkey = key;
            }
            // counters of the captured loop (same structure every replay)
            stages = 0;
            for (int s = start_node; s < s_end; ++s) stages += H < n - 1 - s ? H : n - 1 - s;
            // candidates, seed, pick per step (+ first ladders / seed) + stages
            launches = (int64_t)(s_end - start_node) * 3 + 1 + stages;
            all.start(st);
            state.upload(&h0, 1, st);
            ECO_CUDA(cudaGraphLaunch(gexec, st));
        } else {
            all.start(st);
            state.upload(&h0, 1, st);
            if (count) ECO_CUDA(cudaMemsetAsync(live.p, 0, sizeof(unsigned long long), st));
            enqueue(st);
        }
        all.stop(st);
        if (ring) ECO_CUDA(cudaStreamSynchronize(geo_st));
        LoopState hs{};
        state.download(&hs, 1, st);
        unsigned long long nlive = 0;
        if (count) ECO_CUDA(cudaMemcpyAsync(&nlive, live.p, sizeof nlive, cudaMemcpyDeviceToHost, st));
        ECO_CUDA(cudaStreamSynchronize(st));
        rows.download(out_rows, hs.n_rows, st);
        ECO_CUDA(cudaStreamSynchronize(st));
        *n_rows = hs.n_rows;
        last_rows = hs.n_rows;
        *status = hs.status;
        *status_node = hs.status_node;
        final_state[0] = hs.x[0]; final_state[1] = hs.x[1]; final_state[2] = hs.x[2];
        if (stats) {
            stats->device_ms = all.ms();
            stats->dominant_ms = (double)hs.sweep_ns * 1e-6;   // summed per-step solve clocks
            stats->dense_updates = stages * (int64_t)ns * U;
            stats->live_updates = count ? (int64_t)nlive : -1;
            stats->stages = stages;
            stats->kernel_launches = launches;
        }
    }
};

SessionBase* make_session(const EcoPlant* p, const EcoRoute* r, const EcoMpcConfig* c) {
    SessionBase* s;
    if (c->precision == ECO_FP64) s = new Session<double>(p, r, c);
    else s = new Session<float>(p, r, c);
    s->precision = c->precision;
    return s;
}

// ------------------------------------------------------------- batches
// Many independent horizon solves over one route geometry (C4).  The
// route-level geometry (and the optional terminal field) is built once on the
// first solve and stays resident; each solve uploads the scenarios' start
// nodes, clocks and signal timings, builds their ladders and terminal levels
// on the device, and runs H launches, each sweeping stage k of every scenario
// of the chunk (bellman_batch_kernel).
struct BatchBase {
    int precision = 0;
    virtual ~BatchBase() = default;
    virtual void solve(int n_scen, const EcoSignalTiming* tim, const int32_t* s, const double* t_start, double* J0,
                       int32_t* P0, int flags, EcoStats* stats) = 0;
};

template <typename Real>
struct Batch : BatchBase {
    EcoMpcConfig cfg{};
    std::vector<double> te_h, tb_h;
    std::vector<int8_t> kinds;
    int n = 0, n_sig = 0;
    double stop_dwell = 0.0;
    RouteCtx<Real> ctx;
    DBuf<double> field;
    DBuf<Real> field_int;
    DBuf<int32_t> sig_of_node;
    bool fitted = false;
    size_t cap = 0;                       // scenarios the per-chunk buffers hold
    DBuf<EcoSignalTiming> tim;
    DBuf<int32_t> s_d, h_d, ord_d, P0_d[2];
    DBuf<double> t_d, tdep, wait, tax, J0_d[2];
    cudaStream_t st_out = 0;       // D2H of chunk c overlaps the compute of chunk c + 1
    cudaEvent_t ev_out[2]{};
    DBuf<uint8_t> green, dep;
    DBuf<int> bflags;
    DBuf<Real> J;
    DBuf<unsigned long long> live;
    cudaStream_t st = 0;

    Batch(const EcoPlant* p, const EcoRoute* r, const EcoMpcConfig* c) {
        cfg = *c;
        te_h.assign(c->te_axis, c->te_axis + c->n_te);
        tb_h.assign(c->tb_axis, c->tb_axis + c->n_tb);
        cfg.te_axis = te_h.data();
        cfg.tb_axis = tb_h.data();
        n = r->node_count;
        kinds.assign(r->kinds, r->kinds + n);
        stop_dwell = r->stop_dwell;
        ctx.init(p, r, &cfg, st);
        // throughput-bound (many waves): taller tiles, fewer slices (measured
        // on C4: 4 x 8 beats the single-solve 2 x 16 by 13 %)
        if (!wide_rows(cfg.n_t)) {
            ctx.G.tj_pref = env_int("ECO_BATCH_TJ", 4);
            ctx.G.slices_pref = env_int("ECO_BATCH_SLICES", 8);
        }
        std::vector<int32_t> so(n, -1);
        for (int m = 0; m < n; ++m)
            if (kinds[m] == ECO_NODE_SIGNAL) so[m] = n_sig++;
        sig_of_node.alloc(n);
        sig_of_node.upload(so.data(), n, st);
        if (cfg.use_terminal_field) {
            field.alloc((size_t)n * cfg.n_v * cfg.n_soc);
            field_int.alloc((size_t)n * cfg.n_v * cfg.n_soc);
        }
        live.alloc(1);
        ECO_CUDA(cudaStreamSynchronize(st));
        ECO_CUDA(cudaStreamCreate(&st));
        ECO_CUDA(cudaStreamCreateWithFlags(&st_out, cudaStreamNonBlocking));
        for (auto& e : ev_out) ECO_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    ~Batch() override {
        for (auto& e : ev_out) if (e) cudaEventDestroy(e);
        if (st_out) cudaStreamDestroy(st_out);
        if (st) cudaStreamDestroy(st);
    }

    void reserve(size_t B, int H, size_t ns) {
        if (B <= cap) return;
        const int nt = cfg.n_t;
        tim.alloc(B * std::max(1, n_sig));
        s_d.alloc(B); h_d.alloc(B); t_d.alloc(B); ord_d.alloc(B);
        green.alloc(B * (H + 1) * nt); dep.alloc(B * (H + 1) * nt);
        tdep.alloc(B * (H + 1) * nt); wait.alloc(B * (H + 1) * nt); tax.alloc(B * nt);
        bflags.alloc(B * H);
        J.alloc(B * 2 * level_stride(ns));
        cap = B;
    }

    void solve(int n_scen, const EcoSignalTiming* tim_h, const int32_t* s_h, const double* t_h, double* J0,
               int32_t* P0, int flags, EcoStats* stats) override {
        const int nv = cfg.n_v, nx = cfg.n_soc, nt = cfg.n_t, H = cfg.horizon;
        const int U = cfg.n_te * cfg.n_tb;
        const size_t ns = (size_t)nv * nx * nt;
        const bool count = flags & kRunCountLive;
        for (int i = 0; i < n_scen; ++i) {
            if (s_h[i] < 0 || s_h[i] > n - 2) throw ArgError{"scenario start node out of range"};
            if (!std::isfinite(t_h[i])) throw ArgError{"scenario start time must be finite"};
        }
        if (n_sig && n_scen && !tim_h) throw ArgError{"null signal timings"};
        for (int i = 0; i < n_scen * n_sig; ++i)
            if (tim_h[i].nwin < 0 || tim_h[i].nwin > ECO_MAX_WINDOWS || !(tim_h[i].cycle > 0.0))
                throw ArgError{"invalid signal timing"};
        int64_t launches = 0;
        double fit_ms = 0.0, sweep_ms = 0.0, all_ms = 0.0;
        if (!fitted) {
            EventTimer ft;
            ft.start(st);
            ctx.geometry(st, &launches);
            if (cfg.use_terminal_field) {
                double fs = 0.0;
                field_build_impl<Real>(kinds.data(), n, stop_dwell, &cfg, ctx.G, ctx.R, ctx.soc.p, field_int, field,
                                       st, &launches, &fs);
            }
            ft.stop(st);
            fit_ms = ft.ms();
            fitted = true;
        }
        const bool outs = J0 || P0;
        // with host outputs, smaller chunks let chunk c's D2H overlap chunk c + 1
        const int chunk = std::max(1, std::min(outs ? env_int("ECO_BATCH_OUT_CHUNK", 1024)
                                                    : env_int("ECO_BATCH_CHUNK", 4096), 65535));
        int pending = -1;                 // chunk whose outputs still wait for their D2H
        int pend_c0 = 0, pend_B = 0;
        auto drain = [&]() {
            if (pending < 0) return;
            const int b = pending & 1;
            ECO_CUDA(cudaStreamWaitEvent(st_out, ev_out[b], 0));
            if (J0) download_big(J0 + (size_t)pend_c0 * ns, J0_d[b].p, (size_t)pend_B * ns * sizeof(double), st_out);
            if (P0) download_big(P0 + (size_t)pend_c0 * ns, P0_d[b].p, (size_t)pend_B * ns * sizeof(int32_t), st_out);
            ECO_CUDA(cudaStreamSynchronize(st_out));
            pending = -1;
        };
        const TileCfg tc = tile_cfg(ctx.G, nt, 0, env_int("ECO_BATCH_ALIAS", 1) != 0);
        const size_t LV = level_stride(ns), LC = level_copy(ns);
        LoopCfg lc{nv, nx, nt, cfg.n_te, cfg.n_tb, U, H, cfg.teleport, cfg.use_terminal_field, cfg.dt, cfg.gamma,
                   cfg.soc_target, cfg.soc_weight, cfg.j_inf, ctx.te.p, ctx.tb.p, ctx.soc.p, ctx.R.vaxes.p};
        if (tc.wide) throw ArgError{"batch solves support n_t < 128 (the wide-row path is single-solve only)"};
        auto kern = count ? bellman_batch_kernel<Real, true> : bellman_batch_kernel<Real, false>;
        set_smem_attr(kern, tc.smem);
        int64_t stages = 0;
        unsigned long long nlive = 0;
        if (count) ECO_CUDA(cudaMemsetAsync(live.p, 0, sizeof(unsigned long long), st));
        for (int c0 = 0, ci = 0; c0 < n_scen; c0 += chunk, ++ci) {
            const int B = std::min(chunk, n_scen - c0);
            const int ob = ci & 1;
            reserve((size_t)std::min(chunk, n_scen), H, ns);
            std::vector<int32_t> hh(B);
            int Hmax = 0;
            for (int i = 0; i < B; ++i) {
                const int s = s_h[c0 + i];
                hh[i] = H < n - 1 - s ? H : n - 1 - s;
                Hmax = std::max(Hmax, hh[i]);
                stages += hh[i];
            }
            EventTimer all, sw;
            all.start(st);
            s_d.upload(s_h + c0, B, st);
            t_d.upload(t_h + c0, B, st);
            h_d.upload(hh.data(), B, st);
            // launch order of the scenarios: by start node (stable)
            std::vector<int32_t> ord(B);
            for (int i = 0; i < B; ++i) ord[i] = i;
            std::stable_sort(ord.begin(), ord.end(), [&](int x, int y) { return s_h[c0 + x] < s_h[c0 + y]; });
            const bool sorted = env_int("ECO_BATCH_SORT", 1) != 0;
            if (sorted) ord_d.upload(ord.data(), B, st);
            if (n_sig) tim.upload(tim_h + (size_t)c0 * n_sig, (size_t)B * n_sig, st);
            const unsigned pblocks = (unsigned)std::max<size_t>(1, std::min<size_t>(64, (ns + 255) / 256));
            batch_prepare_kernel<Real><<<dim3(pblocks, B), 256, 0, st>>>(
                ctx.R.view, lc, sig_of_node.p, n_sig, tim.p, s_d.p, h_d.p, t_d.p, Hmax,
                cfg.use_terminal_field ? field.p : nullptr, green.p, dep.p, tdep.p, wait.p, tax.p, J.p, LV, LC,
                bflags.p);
            ECO_CUDA(cudaGetLastError());
            ++launches;
            BatchArgs<Real> ba{};
            ba.base = stage_args(ctx.G, 0, nullptr, nt, tc);
            ba.base.live = count ? live.p : nullptr;
            ba.base.dtg = cfg.dt;
            ba.base.j_inf = (Real)cfg.j_inf;
            ba.pair_stride = (size_t)nv * U;
            ba.tile_stride = nv * tc.nchunk;
            ba.Hmax = Hmax;
            ba.s = s_d.p; ba.h = h_d.p;
            ba.green = green.p; ba.dep_ok = dep.p; ba.t_dep = tdep.p; ba.wait = wait.p; ba.t_axis = tax.p;
            ba.flags = bflags.p;
            ba.J = J.p; ba.LV = LV; ba.LC = LC;
            ba.order = sorted ? ord_d.p : nullptr;
            if (P0 && P0_d[ob].n < (size_t)B * ns) P0_d[ob].alloc((size_t)std::min(chunk, n_scen) * ns);
            ba.P0 = P0 ? P0_d[ob].p : nullptr;
            sw.start(st);
            for (int k = Hmax - 1; k >= 0; --k) {
                ba.k = k;
                cudaLaunchConfig_t cl{};
                cl.gridDim = dim3((unsigned)(nv * tc.nchunk), (unsigned)B);
                cl.blockDim = dim3((unsigned)(tc.S * tc.slices));
                cl.dynamicSmemBytes = tc.smem;
                cl.stream = st;
                cudaLaunchAttribute attr[1];
                attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
                attr[0].val.programmaticStreamSerializationAllowed = env_int("ECO_PDL", 1) ? 1 : 0;
                cl.attrs = attr;
                cl.numAttrs = 1;
                ECO_CUDA(cudaLaunchKernelEx(&cl, kern, ba));
                ++launches;
            }
            sw.stop(st);
            if (J0) {
                if (J0_d[ob].n < (size_t)B * ns) J0_d[ob].alloc((size_t)std::min(chunk, n_scen) * ns);
                to_external_strided_kernel<Real><<<grid_for((size_t)B * ns), 256, 0, st>>>(J.p, J0_d[ob].p, ns, B,
                                                                                          2 * LV, cfg.j_inf);
                ECO_CUDA(cudaGetLastError());
                ++launches;
            }
            all.stop(st);
            if (outs) ECO_CUDA(cudaEventRecord(ev_out[ob], st));
            // previous chunk's D2H (blocks this thread) while this chunk computes
            drain();
            if (outs) { pending = ci; pend_c0 = c0; pend_B = B; }
            sweep_ms += sw.ms();
            all_ms += all.ms();
        }
        drain();
        if (count) {
            ECO_CUDA(cudaMemcpyAsync(&nlive, live.p, sizeof nlive, cudaMemcpyDeviceToHost, st));
            ECO_CUDA(cudaStreamSynchronize(st));
        }
        if (stats) {
            stats->device_ms = all_ms + fit_ms;
            stats->dominant_ms = sweep_ms;
            stats->dense_updates = stages * (int64_t)ns * U;
            stats->live_updates = count ? (int64_t)nlive : -1;
            stats->stages = stages;
            stats->kernel_launches = launches;
        }
    }
};

BatchBase* make_batch(const EcoPlant* p, const EcoRoute* r, const EcoMpcConfig* c) {
    BatchBase* b;
    if (c->precision == ECO_FP64) b = new Batch<double>(p, r, c);
    else b = new Batch<float>(p, r, c);
    b->precision = c->precision;
    return b;
}

// ---------------------------------------------------------------- slabs
// Slab-partitioned horizon solve (C5): rank g of G computes the
// speed planes [lo_g, hi_g) of every level (make_partition, parallel.py:87-101)
// reading the full J_{k+1}; after each stage the slabs are exchanged so every
// rank again holds the full level.
//   ECO_XCHG_P2P  the stage kernel's epilogue stores its slab straight into
//                 every peer's replica over NVLink (CUDA IPC), followed by a
//                 flag barrier across the GPUs (slab_barrier_kernel);
//   ECO_XCHG_NCCL one grouped ncclBroadcast per slab after the stage kernel.
// Policies stay sharded: each rank returns its own planes.
constexpr int kSlabInfoBytes = 256;     // [J handle 64][flag handle 64][nccl id 128]

struct SlabBase {
    int precision = 0;
    virtual ~SlabBase() = default;
    virtual void info(unsigned char* out) = 0;
    virtual void connect(const unsigned char* all) = 0;
    virtual void solve(const EcoPlant* plant, const EcoProblem* pr, const EcoStepPlan* plans, int H,
                       const double* terminal, double* J_stack, int32_t* P_slab, int count, EcoStats* stats) = 0;
    virtual void set_host_barrier(void (*fn)(void*), void* user) = 0;
};

template <typename Real>
struct Slab : SlabBase {
    int nranks, rank, exchange, Hmax;
    int nv, nx, nt;
    size_t ns, LV, LC;
    std::vector<int> lo, hi;
    DBuf<Real> J;                      // (Hmax + 1) levels, IPC-exported
    DBuf<unsigned> flag;               // barrier counter, IPC-exported
    DBuf<int> err;
    DBuf<int32_t> P;
    HorizonInputs in;
    DBuf<double> tmp;
    DBuf<unsigned long long> live;
    Geometry<Real> G;
    std::vector<Real*> peer_J;         // opened replicas (excluding self)
    std::vector<unsigned*> peer_flag;
    DBuf<Real*> d_peer_J;
    DBuf<unsigned*> d_peer_flag;
    unsigned long long barriers = 0;
    ncclComm_t comm = nullptr;
    ncclUniqueId nid{};
    bool connected = false;
    cudaStream_t st = 0;
    // host-side stage barrier (tests of the P2P data path with several ranks
    // on ONE GPU, where a GPU-side spin barrier across processes may not be
    // used): stream sync + the caller's barrier instead of slab_barrier_kernel
    void (*host_barrier)(void*) = nullptr;
    void* host_barrier_user = nullptr;

    void gpu_or_host_barrier() {
        ++barriers;
        if (host_barrier) {
            ECO_CUDA(cudaStreamSynchronize(st));
            host_barrier(host_barrier_user);
            return;
        }
        slab_barrier_kernel<<<1, 32, 0, st>>>(d_peer_flag.p, (int)peer_flag.size(), flag.p,
                                              (unsigned)(barriers * nranks), err.p);
        ECO_CUDA(cudaGetLastError());
    }

    Slab(int nranks_, int rank_, int exchange_, const int32_t* bounds, int nv_, int nx_, int nt_, int Hmax_)
        : nranks(nranks_), rank(rank_), exchange(exchange_), Hmax(Hmax_), nv(nv_), nx(nx_), nt(nt_) {
        if (nranks < 1 || rank < 0 || rank >= nranks) throw ArgError{"invalid rank / world size"};
        if (exchange != ECO_XCHG_P2P && exchange != ECO_XCHG_NCCL) throw ArgError{"unknown exchange mode"};
        // the host's make_partition (parallel.py:87-101): contiguous,
        // non-empty, covering [0, n_v)
        if (bounds[0] != 0 || bounds[nranks] != nv) throw ArgError{"partition does not cover the speed planes"};
        lo.resize(nranks); hi.resize(nranks);
        for (int g = 0; g < nranks; ++g) {
            lo[g] = bounds[g];
            hi[g] = bounds[g + 1];
            if (hi[g] <= lo[g]) throw ArgError{"partition ranges must be non-empty and ordered"};
        }
        ns = (size_t)nv * nx * nt;
        LV = level_stride(ns);
        LC = level_copy(ns);
        J.alloc((size_t)(Hmax + 1) * LV);
        flag.alloc(1);
        ECO_CUDA(cudaMemset(flag.p, 0, sizeof(unsigned)));
        err.alloc(1);
        ECO_CUDA(cudaMemset(err.p, 0, sizeof(int)));
        live.alloc(1);
        if (exchange == ECO_XCHG_NCCL && rank == 0) {
            if (ncclGetUniqueId(&nid) != ncclSuccess) throw std::runtime_error("ncclGetUniqueId failed");
        }
        ECO_CUDA(cudaStreamCreate(&st));
    }
    ~Slab() override {
        if (comm) ncclCommDestroy(comm);
        for (Real* p : peer_J) cudaIpcCloseMemHandle(p);
        for (unsigned* p : peer_flag) cudaIpcCloseMemHandle(p);
        if (st) cudaStreamDestroy(st);
    }

    void set_host_barrier(void (*fn)(void*), void* user) override {
        host_barrier = fn;
        host_barrier_user = user;
    }

    void info(unsigned char* out) override {
        std::memset(out, 0, kSlabInfoBytes);
        cudaIpcMemHandle_t hj{}, hf{};
        if (exchange == ECO_XCHG_P2P && nranks > 1) {
            ECO_CUDA(cudaIpcGetMemHandle(&hj, J.p));
            ECO_CUDA(cudaIpcGetMemHandle(&hf, flag.p));
        }
        std::memcpy(out, &hj, sizeof hj);
        std::memcpy(out + 64, &hf, sizeof hf);
        std::memcpy(out + 128, &nid, sizeof nid);
    }

    void connect(const unsigned char* all) override {
        if (connected) throw ArgError{"slab session already connected"};
        if (exchange == ECO_XCHG_P2P) {
            for (int g = 0; g < nranks; ++g) {
                if (g == rank) continue;
                cudaIpcMemHandle_t hj, hf;
                std::memcpy(&hj, all + (size_t)g * kSlabInfoBytes, sizeof hj);
                std::memcpy(&hf, all + (size_t)g * kSlabInfoBytes + 64, sizeof hf);
                void* pj = nullptr;
                void* pf = nullptr;
                ECO_CUDA(cudaIpcOpenMemHandle(&pj, hj, cudaIpcMemLazyEnablePeerAccess));
                ECO_CUDA(cudaIpcOpenMemHandle(&pf, hf, cudaIpcMemLazyEnablePeerAccess));
                peer_J.push_back(static_cast<Real*>(pj));
                peer_flag.push_back(static_cast<unsigned*>(pf));
            }
            if (!peer_J.empty()) {
                d_peer_J.alloc(peer_J.size());
                d_peer_J.upload(peer_J.data(), peer_J.size(), st);
                d_peer_flag.alloc(peer_flag.size());
                d_peer_flag.upload(peer_flag.data(), peer_flag.size(), st);
            }
        } else {
            std::memcpy(&nid, all + 128, sizeof nid);      // rank 0's id
            if (ncclCommInitRank(&comm, nranks, nid, rank) != ncclSuccess) throw std::runtime_error("ncclCommInitRank failed");
        }
        ECO_CUDA(cudaStreamSynchronize(st));
        connected = true;
    }

    // After stage k: every rank holds copy 0 of the full level (peers' slabs
    // arrived by NVLink stores + barrier, or by broadcast); copy 1 (the
    // shifted twin) is rebuilt locally instead of crossing the links.
    void exchange_level(int k) {
        Real* Lk = J.p + (size_t)k * LV;
        const size_t plane = (size_t)nx * nt;
        if (exchange == ECO_XCHG_P2P) {
            gpu_or_host_barrier();
        } else {
            const ncclDataType_t ty = sizeof(Real) == 4 ? ncclFloat32 : ncclFloat64;
            if (ncclGroupStart() != ncclSuccess) throw std::runtime_error("ncclGroupStart failed");
            for (int g = 0; g < nranks; ++g) {
                const size_t o0 = (size_t)lo[g] * plane, n0 = (size_t)(hi[g] - lo[g]) * plane;
                if (!n0) continue;
                if (ncclBroadcast(Lk + o0, Lk + o0, n0, ty, g, comm, st) != ncclSuccess)
                    throw std::runtime_error("ncclBroadcast failed");
            }
            if (ncclGroupEnd() != ncclSuccess) throw std::runtime_error("ncclGroupEnd failed");
        }
        shift_copy_kernel<Real><<<grid_for(ns + 8), 256, 0, st>>>(Lk, ns, LC);
        ECO_CUDA(cudaGetLastError());
    }

    void solve(const EcoPlant* plant, const EcoProblem* pr, const EcoStepPlan* plans, int H, const double* terminal,
               double* J_stack, int32_t* P_slab, int count, EcoStats* stats) override {
        if (!connected) throw ArgError{"slab session not connected"};
        if (pr->n_v != nv || pr->n_soc != nx || pr->n_t != nt) throw ArgError{"grid differs from the slab session"};
        if (H < 1 || H > Hmax) throw ArgError{"horizon exceeds the slab session's capacity"};
        const int U = pr->n_te * pr->n_tb;
        const int plo = lo[rank], phi = hi[rank];
        const size_t plane = (size_t)nx * nt, slab_ns = (size_t)(phi - plo) * plane;
        int64_t launches = 0;
        in.upload(plant, pr, plans, H, terminal, st);
        P.ensure((size_t)H * slab_ns);
        if (J_stack) tmp.ensure(ns * (size_t)(H + 1));
        ECO_CUDA(cudaMemsetAsync(live.p, 0, sizeof(unsigned long long), st));
        EventTimer all, sweep;
        all.start(st);
        G.dims = GeomDims{H, nv, nx, nt, U, pr->n_te, pr->n_tb, pr->delta_d, pr->a_min, pr->a_max, pr->gamma, pr->dtg};
        G.plo = plo;
        G.phi = phi;
        TablesDev tdev;
        build_geometry(G, in.plant, in.plans, in.v, in.te, in.tb, in.soc, tdev.view, st, &launches, true, false);
        to_internal2_kernel<Real><<<grid_for(ns + 8), 256, 0, st>>>(in.terminal, J.p + (size_t)H * LV, ns, pr->j_inf);
        ECO_CUDA(cudaGetLastError());
        ++launches;
        const TileCfg tc = tile_cfg(G, nt, 0);
        // P2P: no rank may store into a peer's levels while that peer still
        // reads its previous solve's tables (output conversion, D2H)
        if (exchange == ECO_XCHG_P2P && nranks > 1) {
            gpu_or_host_barrier();
            ++launches;
        }
        sweep.start(st);
        for (int k = H - 1; k >= 0; --k) {
            StageArgs<Real> a = stage_args(G, k, in.v + (size_t)k * nv, nt, tc);
            a.green = in.green + (size_t)k * nt;
            a.flags = in.flags + k;
            a.dep_ok = in.dep + (size_t)k * nt;
            a.t_dep = in.tdep + (size_t)k * nt;
            a.wait = in.wait + (size_t)k * nt;
            a.J_next = J.p + (size_t)(k + 1) * LV;
            a.J_next1 = a.J_next + LC;
            a.lc = LC;
            a.J_out = J.p + (size_t)k * LV;
            a.J_out1 = a.J_out + LC;
            // the kernel indexes P by the global state: shift the slab buffer
            a.P_out = P.p + (size_t)k * slab_ns - (ptrdiff_t)((size_t)plo * plane);
            a.live = count ? live.p : nullptr;
            a.src_kind = plans[k].src_kind;
            a.t0 = pr->t0;
            a.dtg = pr->dtg;
            a.j_inf = (Real)pr->j_inf;
            if (exchange == ECO_XCHG_P2P && !peer_J.empty()) {
                a.peer_base = d_peer_J.p;
                a.npeer = (int)peer_J.size();
                a.peer_off = (size_t)k * LV;
                a.lc = LC;
            }
            launch_stage<Real, 0>(a, tc, count, st, (phi - plo) * tc.nchunk);
            ++launches;
            if (nranks > 1) {
                exchange_level(k);
                launches += 2;
            }
        }
        sweep.stop(st);
        if (J_stack) {
            to_external_levels_kernel<Real><<<grid_for(ns * (H + 1)), 256, 0, st>>>(J.p, tmp.p, ns, H + 1,
                                                                                   pr->j_inf);
            ECO_CUDA(cudaGetLastError());
            ++launches;
        }
        all.stop(st);
        if (J_stack) download_big(J_stack, tmp.p, ns * (H + 1) * sizeof(double), st);
        if (P_slab) download_big(P_slab, P.p, (size_t)H * slab_ns * sizeof(int32_t), st);
        int herr = 0;
        unsigned long long nlive = 0;
        ECO_CUDA(cudaMemcpyAsync(&herr, err.p, sizeof herr, cudaMemcpyDeviceToHost, st));
        ECO_CUDA(cudaMemcpyAsync(&nlive, live.p, sizeof nlive, cudaMemcpyDeviceToHost, st));
        ECO_CUDA(cudaStreamSynchronize(st));
        if (herr) throw std::runtime_error("slab barrier timed out (a peer rank stopped)");
        if (stats) {
            stats->device_ms = all.ms();
            stats->dominant_ms = sweep.ms();
            stats->dense_updates = (int64_t)slab_ns * U * H;
            stats->live_updates = count ? (int64_t)nlive : -1;
            stats->stages = H;
            stats->kernel_launches = launches;
        }
    }
};

// eco_slab_emulate: nranks slab ranks on ONE GPU (kernel-boundary stage
// barrier, one launch per stage over every rank's tiles); every rank keeps its
// own replica of the levels, filled by its own stores and its peers' PEERS
// epilogue stores (copy 0) + the local copy-1 rebuild, as on a multi-GPU run.
template <typename Real>
void slab_emulate_impl(int nranks, const int32_t* bounds, const EcoPlant* plant, const EcoProblem* pr,
                       const EcoStepPlan* plans, int H, const double* terminal, double* J_stacks, int32_t* P_stack,
                       EcoStats* stats) {
    const int nv = pr->n_v, nx = pr->n_soc, nt = pr->n_t, U = pr->n_te * pr->n_tb;
    if (nranks < 1 || nranks > kEmulMaxRanks) throw ArgError{"emulation supports 1..8 ranks"};
    if (bounds[0] != 0 || bounds[nranks] != nv) throw ArgError{"partition does not cover the speed planes"};
    for (int g = 0; g < nranks; ++g)
        if (bounds[g + 1] <= bounds[g]) throw ArgError{"partition ranges must be non-empty and ordered"};
    const size_t ns = (size_t)nv * nx * nt, LV = level_stride(ns), LC = level_copy(ns);
    cudaStream_t st = 0;
    int64_t launches = 0;
    HorizonInputs in;
    in.upload(plant, pr, plans, H, terminal, st);
    Geometry<Real> G;
    G.dims = GeomDims{H, nv, nx, nt, U, pr->n_te, pr->n_tb, pr->delta_d, pr->a_min, pr->a_max, pr->gamma, pr->dtg};
    TablesDev tdev;
    build_geometry(G, in.plant, in.plans, in.v, in.te, in.tb, in.soc, tdev.view, st, &launches, true, false);
    DBuf<Real> rep((size_t)nranks * (H + 1) * LV);
    DBuf<int32_t> P((size_t)H * ns);
    EmulArgs<Real> e{};
    std::vector<Real*> peers;
    for (int g = 0; g < nranks; ++g) {
        e.rep[g] = rep.p + (size_t)g * (H + 1) * LV;
        e.lo[g] = bounds[g];
        for (int q = 0; q < nranks; ++q)
            if (q != g) peers.push_back(rep.p + (size_t)q * (H + 1) * LV);
        to_internal2_kernel<Real><<<grid_for(ns + 8), 256, 0, st>>>(in.terminal, e.rep[g] + (size_t)H * LV, ns,
                                                                     pr->j_inf);
        ECO_CUDA(cudaGetLastError());
    }
    e.lo[nranks] = nv;
    e.nranks = nranks;
    e.lc = LC;
    DBuf<Real*> d_peers(std::max<size_t>(1, peers.size()));
    if (!peers.empty()) d_peers.upload(peers.data(), peers.size(), st);
    e.peers = d_peers.p;
    const TileCfg tc = tile_cfg(G, nt, 0);
    auto kern = (tc.wide && w2_wpr(nt)) ? bellman_emul_kernel<Real, true, true>
                                         : tc.wide ? bellman_emul_kernel<Real, true> : bellman_emul_kernel<Real, false>;
    set_smem_attr(kern, tc.smem);
    EventTimer all;
    WriterCheck wchk(ns);
    all.start(st);
    for (int k = H - 1; k >= 0; --k) {
        wchk.arm(st);
        StageArgs<Real> a = stage_args(G, k, in.v + (size_t)k * nv, nt, tc);
        a.green = in.green + (size_t)k * nt;
        a.flags = in.flags + k;
        a.dep_ok = in.dep + (size_t)k * nt;
        a.t_dep = in.tdep + (size_t)k * nt;
        a.wait = in.wait + (size_t)k * nt;
        a.P_out = P.p + (size_t)k * ns;
        a.src_kind = plans[k].src_kind;
        a.t0 = pr->t0;
        a.dtg = pr->dtg;
        a.j_inf = (Real)pr->j_inf;
        a.lc = LC;
        e.next_off = (size_t)(k + 1) * LV;
        e.out_off = (size_t)k * LV;
        kern<<<nv * tc.nchunk, tc.S * tc.slices, tc.smem, st>>>(a, e);
        ECO_CUDA(cudaGetLastError());
        wchk.verify(st);
        ++launches;
        for (int g = 0; g < nranks; ++g) {
            shift_copy_kernel<Real><<<grid_for(ns + 8), 256, 0, st>>>(e.rep[g] + (size_t)k * LV, ns, LC);
            ECO_CUDA(cudaGetLastError());
            ++launches;
        }
    }
    all.stop(st);
    DBuf<double> tmp(ns * (H + 1));
    for (int g = 0; g < nranks; ++g) {
        to_external_levels_kernel<Real><<<grid_for(ns * (H + 1)), 256, 0, st>>>(e.rep[g], tmp.p, ns, H + 1,
                                                                               pr->j_inf);
        ECO_CUDA(cudaGetLastError());
        download_big(J_stacks + (size_t)g * (H + 1) * ns, tmp.p, ns * (H + 1) * sizeof(double), st);
    }
    if (P_stack) download_big(P_stack, P.p, (size_t)H * ns * sizeof(int32_t), st);
    ECO_CUDA(cudaStreamSynchronize(st));
    if (stats) {
        stats->device_ms = all.ms();
        stats->dominant_ms = stats->device_ms;
        stats->dense_updates = (int64_t)ns * U * H;
        stats->live_updates = -1;
        stats->stages = H;
        stats->kernel_launches = launches;
    }
}

SlabBase* make_slab(int nranks, int rank, int exchange, const int32_t* bounds, int precision, int nv, int nx, int nt,
                    int Hmax) {
    SlabBase* s;
    if (precision == ECO_FP64) s = new Slab<double>(nranks, rank, exchange, bounds, nv, nx, nt, Hmax);
    else s = new Slab<float>(nranks, rank, exchange, bounds, nv, nx, nt, Hmax);
    s->precision = precision;
    return s;
}

}  // namespace

// ================================================================== C ABI
extern "C" {

int32_t eco_abi_version(void) { return ECO_ABI_VERSION; }

const char* eco_last_error(void) { return g_err.c_str(); }

int32_t eco_release_workspace(void) {
    return run_guarded([&] {
        std::lock_guard<std::mutex> lock(workspace_mutex());
        horizon_workspace<float>().release();
        horizon_workspace<double>().release();
    });
}

int32_t eco_debug_checks(int64_t* bounds_violations, int64_t* writer_violations, int32_t reset) {
    return run_guarded([&] {
        if (!bounds_violations || !writer_violations) throw ArgError{"null pointer argument"};
#ifdef ECO_CHECKED
        ECO_CUDA(cudaDeviceSynchronize());
        unsigned long long b = 0, w = 0;
        ECO_CUDA(cudaMemcpyFromSymbol(&b, g_chk_bounds, sizeof b));
        ECO_CUDA(cudaMemcpyFromSymbol(&w, g_chk_writer, sizeof w));
        *bounds_violations = (int64_t)b;
        *writer_violations = (int64_t)w;
        if (reset) {
            const unsigned long long z = 0;
            ECO_CUDA(cudaMemcpyToSymbol(g_chk_bounds, &z, sizeof z));
            ECO_CUDA(cudaMemcpyToSymbol(g_chk_writer, &z, sizeof z));
        }
#else
        (void)reset;
        *bounds_violations = -1;
        *writer_violations = -1;
#endif
    });
}

int32_t eco_host_alloc(uint64_t bytes, void** out) {
    return run_guarded([&] {
        if (!out) throw ArgError{"null pointer argument"};
        *out = nullptr;
        if (bytes) ECO_CUDA(cudaHostAlloc(out, (size_t)bytes, cudaHostAllocPortable));
    });
}

int32_t eco_host_free(void* p) {
    return run_guarded([&] {
        if (p) ECO_CUDA(cudaFreeHost(p));
    });
}

int32_t eco_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
    return n;
}

int32_t eco_bellman_step(const EcoPlant* plant, const EcoProblem* prob, const EcoStepPlan* plan,
                         const EcoStage1Tables* tables, const double* J_next, double* J_out, int32_t* P_out,
                         int32_t precision, int32_t count_live, EcoStats* stats) {
    return run_guarded([&] {
        check_plant(plant);
        check_problem(prob);
        if (!plan || !J_next || !J_out || !P_out) throw ArgError{"null pointer argument"};
        const bool rev = (precision & ECO_REVERSE_TIES) != 0;
        precision &= ~ECO_REVERSE_TIES;
        // level 0 straight into the caller's J_out (the terminal level is J_next)
        if (precision == ECO_FP64)
            solve_horizon_impl<double>(plant, prob, plan, 1, tables, J_next, J_out, P_out, count_live, stats, rev,
                                       true);
        else
            solve_horizon_impl<float>(plant, prob, plan, 1, tables, J_next, J_out, P_out, count_live, stats, rev,
                                      true);
    });
}

int32_t eco_solve_horizon(const EcoPlant* plant, const EcoProblem* prob, const EcoStepPlan* plans, int32_t H,
                          const double* terminal, double* J_stack, int32_t* P_stack, int32_t precision,
                          int32_t count_live, EcoStats* stats) {
    return run_guarded([&] {
        check_plant(plant);
        check_problem(prob);
        if (H < 1) throw ArgError{"horizon must be >= 1"};
        if (!plans || !terminal || !J_stack || !P_stack) throw ArgError{"null pointer argument"};
        const bool rev = (precision & ECO_REVERSE_TIES) != 0;
        precision &= ~ECO_REVERSE_TIES;
        if (precision == ECO_FP64)
            solve_horizon_impl<double>(plant, prob, plans, H, nullptr, terminal, J_stack, P_stack, count_live, stats,
                                       rev);
        else
            solve_horizon_impl<float>(plant, prob, plans, H, nullptr, terminal, J_stack, P_stack, count_live, stats,
                                      rev);
    });
}

int32_t eco_solve_tables(const EcoPlant* plant, const EcoProblem* prob, const EcoStepPlan* plans,
                         const EcoStage1Tables* tables, int32_t H, const double* terminal, double* J_stack,
                         int32_t* P_stack, int32_t precision) {
    return run_guarded([&] {
        check_plant(plant);
        check_problem(prob);
        if (H < 1 || !plans || !tables || !terminal || !J_stack || !P_stack) throw ArgError{"bad arguments"};
        const bool rev = (precision & ECO_REVERSE_TIES) != 0;
        precision &= ~ECO_REVERSE_TIES;
        if (precision == ECO_FP64)
            solve_horizon_impl<double>(plant, prob, plans, H, tables, terminal, J_stack, P_stack, false, nullptr, rev);
        else
            solve_horizon_impl<float>(plant, prob, plans, H, tables, terminal, J_stack, P_stack, false, nullptr, rev);
    });
}

int32_t eco_session_create(const EcoPlant* plant, const EcoRoute* route, const EcoMpcConfig* cfg,
                           EcoSession** out) {
    return run_guarded([&] {
        check_plant(plant);
        check_cfg(cfg);
        if (!route || !out) throw ArgError{"null pointer argument"};
        *out = reinterpret_cast<EcoSession*>(make_session(plant, route, cfg));
    });
}

int32_t eco_session_upload_route(EcoSession* sess, const EcoRoute* route) {
    return run_guarded([&] {
        if (!sess || !route) throw ArgError{"null pointer argument"};
        reinterpret_cast<SessionBase*>(sess)->upload_route(route);
    });
}

int32_t eco_session_fit(EcoSession* sess, const double* field_in, double* field_out, EcoStats* stats) {
    return run_guarded([&] {
        if (!sess) throw ArgError{"null session"};
        reinterpret_cast<SessionBase*>(sess)->fit(field_in, field_out, stats);
    });
}

int32_t eco_session_run(EcoSession* sess, int32_t start_node, int32_t max_steps, const double* x_start,
                        EcoTrajRow* rows, int32_t* n_rows, int32_t* status, int32_t* status_node,
                        double* final_state, int32_t flags, EcoStats* stats) {
    return run_guarded([&] {
        if (!sess || !x_start || !rows || !n_rows || !status || !status_node || !final_state)
            throw ArgError{"null pointer argument"};
        reinterpret_cast<SessionBase*>(sess)->run(start_node, max_steps, x_start, rows, n_rows, status, status_node,
                                                  final_state, flags, stats);
    });
}

int32_t eco_session_step_times(EcoSession* sess, double* solve_ms, int32_t n) {
    return run_guarded([&] {
        if (!sess || (n > 0 && !solve_ms)) throw ArgError{"null pointer argument"};
        reinterpret_cast<SessionBase*>(sess)->step_times(solve_ms, n);
    });
}

int32_t eco_session_destroy(EcoSession* sess) {
    delete reinterpret_cast<SessionBase*>(sess);
    return ECO_OK;
}

int32_t eco_field_build(const EcoPlant* plant, const EcoRoute* route, const EcoMpcConfig* cfg, double* field_out,
                        EcoStats* stats) {
    return run_guarded([&] {
        check_plant(plant);
        check_cfg(cfg);
        if (!route || !field_out) throw ArgError{"null pointer argument"};
        EcoMpcConfig c = *cfg;
        c.use_terminal_field = 1;
        std::unique_ptr<SessionBase> s(make_session(plant, route, &c));
        s->fit(nullptr, field_out, stats);
    });
}

int32_t eco_mpc_run(const EcoPlant* plant, const EcoRoute* route, const EcoMpcConfig* cfg, const double* x_start,
                    const double* field_in, double* field_out, EcoTrajRow* rows, int32_t* n_rows, int32_t* status,
                    int32_t* status_node, double* final_state, EcoStats* stats) {
    return run_guarded([&] {
        check_plant(plant);
        check_cfg(cfg);
        if (!route || !x_start || !rows || !n_rows || !status || !status_node || !final_state)
            throw ArgError{"null pointer argument"};
        if (cfg->start_node > route->node_count - 2) throw ArgError{"start_node out of range"};
        std::unique_ptr<SessionBase> s(make_session(plant, route, cfg));
        s->fit(field_in, field_out, nullptr);
        s->run(cfg->start_node, cfg->max_steps, x_start, rows, n_rows, status, status_node, final_state,
               0, stats);
    });
}

int32_t eco_batch_create(const EcoPlant* plant, const EcoRoute* route, const EcoMpcConfig* cfg, EcoBatch** out) {
    return run_guarded([&] {
        check_plant(plant);
        check_cfg(cfg);
        if (!route || !out) throw ArgError{"null pointer argument"};
        *out = reinterpret_cast<EcoBatch*>(make_batch(plant, route, cfg));
    });
}

int32_t eco_batch_solve(EcoBatch* batch, int32_t n_scen, const EcoSignalTiming* timings, const int32_t* s,
                        const double* t_start, double* J0, int32_t* P0, int32_t flags, EcoStats* stats) {
    return run_guarded([&] {
        if (!batch) throw ArgError{"null batch"};
        if (n_scen < 0) throw ArgError{"n_scen must be >= 0"};
        if (n_scen > 0 && (!s || !t_start)) throw ArgError{"null pointer argument"};
        reinterpret_cast<BatchBase*>(batch)->solve(n_scen, timings, s, t_start, J0, P0, flags, stats);
    });
}

int32_t eco_batch_destroy(EcoBatch* batch) {
    delete reinterpret_cast<BatchBase*>(batch);
    return ECO_OK;
}

int32_t eco_solve_batch(const EcoPlant* plant, const EcoRoute* route, const EcoMpcConfig* cfg, int32_t n_scen,
                        const EcoSignalTiming* timings, const int32_t* s, const double* t_start, double* J0,
                        int32_t* P0, EcoStats* stats) {
    return run_guarded([&] {
        check_plant(plant);
        check_cfg(cfg);
        if (!route) throw ArgError{"null pointer argument"};
        if (n_scen < 0) throw ArgError{"n_scen must be >= 0"};
        if (n_scen > 0 && (!s || !t_start)) throw ArgError{"null pointer argument"};
        std::unique_ptr<BatchBase> b(make_batch(plant, route, cfg));
        b->solve(n_scen, timings, s, t_start, J0, P0, 0, stats);
    });
}

int32_t eco_slab_create(int32_t nranks, int32_t rank, int32_t exchange, const int32_t* bounds, int32_t precision,
                        int32_t n_v, int32_t n_soc, int32_t n_t, int32_t max_horizon, EcoSlab** out) {
    return run_guarded([&] {
        if (!out || !bounds) throw ArgError{"null pointer argument"};
        if (n_v < 2 || n_soc < 2 || n_t < 2 || max_horizon < 1) throw ArgError{"invalid grid / horizon"};
        if (nranks < 1) throw ArgError{"invalid rank / world size"};
        *out = reinterpret_cast<EcoSlab*>(make_slab(nranks, rank, exchange, bounds, precision, n_v, n_soc, n_t,
                                                    max_horizon));
    });
}

int32_t eco_slab_info(EcoSlab* slab, uint8_t* info) {
    return run_guarded([&] {
        if (!slab || !info) throw ArgError{"null pointer argument"};
        reinterpret_cast<SlabBase*>(slab)->info(info);
    });
}

int32_t eco_slab_connect(EcoSlab* slab, const uint8_t* all_info) {
    return run_guarded([&] {
        if (!slab || !all_info) throw ArgError{"null pointer argument"};
        reinterpret_cast<SlabBase*>(slab)->connect(all_info);
    });
}

int32_t eco_slab_solve(EcoSlab* slab, const EcoPlant* plant, const EcoProblem* prob, const EcoStepPlan* plans,
                       int32_t H, const double* terminal, double* J_stack, int32_t* P_slab, int32_t count_live,
                       EcoStats* stats) {
    return run_guarded([&] {
        check_plant(plant);
        check_problem(prob);
        if (!slab || !plans || !terminal) throw ArgError{"null pointer argument"};
        reinterpret_cast<SlabBase*>(slab)->solve(plant, prob, plans, H, terminal, J_stack, P_slab, count_live,
                                                 stats);
    });
}

int32_t eco_slab_set_host_barrier(EcoSlab* slab, void (*barrier)(void*), void* user) {
    return run_guarded([&] {
        if (!slab) throw ArgError{"null pointer argument"};
        reinterpret_cast<SlabBase*>(slab)->set_host_barrier(barrier, user);
    });
}

int32_t eco_slab_emulate(int32_t nranks, const int32_t* bounds, int32_t precision, const EcoPlant* plant,
                         const EcoProblem* prob, const EcoStepPlan* plans, int32_t H, const double* terminal,
                         double* J_stacks, int32_t* P_stack, EcoStats* stats) {
    return run_guarded([&] {
        check_plant(plant);
        check_problem(prob);
        if (!bounds || !plans || !terminal || !J_stacks || H < 1) throw ArgError{"bad arguments"};
        if (precision == ECO_FP64)
            slab_emulate_impl<double>(nranks, bounds, plant, prob, plans, H, terminal, J_stacks, P_stack, stats);
        else
            slab_emulate_impl<float>(nranks, bounds, plant, prob, plans, H, terminal, J_stacks, P_stack, stats);
    });
}

int32_t eco_slab_destroy(EcoSlab* slab) {
    delete reinterpret_cast<SlabBase*>(slab);
    return ECO_OK;
}

}  // extern "C"
