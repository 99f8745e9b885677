// eco_api.cu — the C ABI (include/eco_b200.h) over the sm_100a kernels.
//
// Host side only: argument checks, device buffers, launches, conversions
// between the caller's f64 tables (infeasible == j_inf) and the device's
// internal representation (Real, infeasible == +inf).  No CPU compute path.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <algorithm>
#include <vector>

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
    size_t n = 0;
    DBuf() = default;
    explicit DBuf(size_t count) { alloc(count); }
    void alloc(size_t count) {
        free();
        n = count;
        if (count) ECO_CUDA(cudaMalloc(&p, count * sizeof(T)));
    }
    void free() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
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

// --------------------------------------------------------- geometry store
template <typename Real>
struct Geometry {
    GeomDims dims{};
    DBuf<uint32_t> meta;
    DBuf<int32_t> zoff;
    DBuf<Real> c1, wv, wz, wx;
    DBuf<double> dt, c1d, pbat;
    DBuf<int16_t> jxlo;

    void alloc(int P, int nv, int nx, int U) {
        const size_t np = (size_t)P * nv * U;
        meta.alloc(np); zoff.alloc(np); c1.alloc(np); wv.alloc(np); wz.alloc(np);
        dt.alloc(np); c1d.alloc(np); pbat.alloc(np);
        jxlo.alloc(np * nx); wx.alloc(np * nx);
    }
    PairGeom<Real> view() {
        return PairGeom<Real>{meta.p, zoff.p, c1.p, wv.p, wz.p, dt.p, c1d.p, pbat.p, jxlo.p, wx.p};
    }
};

// Computes pair + SoC geometry for P plans (dims filled by the caller).
template <typename Real>
void build_geometry(Geometry<Real>& G, const EcoPlant* d_plant, const DevPlan* d_plans, const double* d_vaxes,
                    const double* d_te, const double* d_tb, const double* d_soc, const EcoStage1Tables& d_tab,
                    cudaStream_t st, int64_t* launches) {
    const GeomDims& g = G.dims;
    G.alloc(g.P, g.nv, g.nx, g.U);
    dim3 grid(g.nv, g.P);
    geom_pairs_kernel<Real><<<grid, 256, 0, st>>>(d_plant, d_plans, d_vaxes, d_te, d_tb, g, G.view(), d_tab);
    ECO_CUDA(cudaGetLastError());
    const size_t smem = (size_t)g.ntb * g.nx * (sizeof(double) + 1) + 16;
    if (smem > 48 * 1024)
        ECO_CUDA(cudaFuncSetAttribute(geom_soc_kernel<Real>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    geom_soc_kernel<Real><<<grid, 256, smem, st>>>(d_plant, d_vaxes, d_tb, d_soc, g, G.view(),
                                                   d_tab.ok != nullptr ? 1 : 0);
    ECO_CUDA(cudaGetLastError());
    if (launches) *launches += 2;
}

constexpr int kTile = 128;
constexpr int kSlices = 8;

template <typename Real>
StageArgs<Real> stage_args(Geometry<Real>& G, int p, const double* d_vsrc, int nt) {
    StageArgs<Real> a{};
    const GeomDims& g = G.dims;
    const size_t off = (size_t)p * g.nv * g.U;
    a.meta = G.meta.p + off;
    a.zoff = G.zoff.p + off;
    a.c1 = G.c1.p + off;
    a.wv = G.wv.p + off;
    a.wz = G.wz.p + off;
    a.dt = G.dt.p + off;
    a.c1d = G.c1d.p + off;
    a.jxlo = G.jxlo.p + off * g.nx;
    a.wx = G.wx.p + off * g.nx;
    a.v_src = d_vsrc;
    a.nv = g.nv;
    a.nx = g.nx;
    a.nt = nt;
    a.U = g.U;
    a.gamma = g.gamma;
    return a;
}

template <typename Real, int MODE>
void launch_stage(const StageArgs<Real>& a, bool count, cudaStream_t st) {
    const int plane = a.nx * a.nt;
    const int tiles = (plane + kTile - 1) / kTile;
    const unsigned grid = (unsigned)(a.nv * tiles);
    if (count)
        bellman_stage_kernel<Real, MODE, kTile, kSlices, true><<<grid, kTile * kSlices, 0, st>>>(a);
    else
        bellman_stage_kernel<Real, MODE, kTile, kSlices, false><<<grid, kTile * kSlices, 0, st>>>(a);
    ECO_CUDA(cudaGetLastError());
}

void check_problem(const EcoProblem* pr) {
    if (!pr) throw ArgError{"null problem"};
    if (pr->n_v < 2 || pr->n_soc < 2 || pr->n_t < 2 || pr->n_te < 1 || pr->n_tb < 1)
        throw ArgError{"grid sizes must be n_v,n_soc,n_t >= 2 and n_te,n_tb >= 1"};
    if (pr->n_v >= (1 << 23)) throw ArgError{"n_v too large"};
    if (pr->n_soc > 32767) throw ArgError{"n_soc must be < 32768"};
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

// --------------------------------------------------------- horizon solve
// dp.py:425-475 / dp.py:557-610: H plans, terminal -> J stack, P stack.
template <typename Real>
void solve_horizon_impl(const EcoPlant* plant, const EcoProblem* pr, const EcoStepPlan* plans, int H,
                        const EcoStage1Tables* tabs, const double* terminal, double* J_stack, int32_t* P_stack,
                        bool count, EcoStats* stats) {
    const int nv = pr->n_v, nx = pr->n_soc, nt = pr->n_t, U = pr->n_te * pr->n_tb;
    const size_t ns = (size_t)nv * nx * nt;
    cudaStream_t st = 0;
    int64_t launches = 0;
    DBuf<EcoPlant> d_plant(1);
    d_plant.upload(plant, 1, st);
    std::vector<DevPlan> hp(H);
    std::vector<double> hv((size_t)H * nv);
    std::vector<uint8_t> hgreen((size_t)H * nt), hdep((size_t)H * nt);
    std::vector<double> htdep((size_t)H * nt), hwait((size_t)H * nt);
    for (int k = 0; k < H; ++k) {
        const EcoStepPlan& s = plans[k];
        if (!s.v_src || !s.arr_green || !s.dep_ok || !s.t_dep || !s.wait) throw ArgError{"null plan array"};
        hp[k] = dev_plan(s);
        std::memcpy(&hv[(size_t)k * nv], s.v_src, sizeof(double) * nv);
        std::memcpy(&hgreen[(size_t)k * nt], s.arr_green, nt);
        std::memcpy(&hdep[(size_t)k * nt], s.dep_ok, nt);
        std::memcpy(&htdep[(size_t)k * nt], s.t_dep, sizeof(double) * nt);
        std::memcpy(&hwait[(size_t)k * nt], s.wait, sizeof(double) * nt);
    }
    DBuf<DevPlan> d_plans(H);
    DBuf<double> d_v((size_t)H * nv), d_tdep((size_t)H * nt), d_wait((size_t)H * nt);
    DBuf<uint8_t> d_green((size_t)H * nt), d_dep((size_t)H * nt);
    DBuf<double> d_te(pr->n_te), d_tb(pr->n_tb), d_soc(nx);
    d_plans.upload(hp.data(), H, st);
    d_v.upload(hv.data(), hv.size(), st);
    d_green.upload(hgreen.data(), hgreen.size(), st);
    d_dep.upload(hdep.data(), hdep.size(), st);
    d_tdep.upload(htdep.data(), htdep.size(), st);
    d_wait.upload(hwait.data(), hwait.size(), st);
    d_te.upload(pr->te_axis, pr->n_te, st);
    d_tb.upload(pr->tb_axis, pr->n_tb, st);
    d_soc.upload(pr->soc_axis, nx, st);
    TablesDev tdev;   // plant path: no tables

    EventTimer all, sweep;
    all.start(st);
    Geometry<Real> G;
    G.dims = GeomDims{H, nv, nx, U, pr->n_te, pr->n_tb, pr->delta_d, pr->a_min, pr->a_max, pr->gamma, pr->dtg};
    // toy mode: each step has its own table; geometry built per plan below
    if (!tabs) build_geometry(G, d_plant.p, d_plans.p, d_v.p, d_te.p, d_tb.p, d_soc.p, tdev.view, st, &launches);

    DBuf<Real> d_J((H + 1) * ns);
    DBuf<int32_t> d_P((size_t)H * ns);
    DBuf<double> d_tmp(ns * (H + 1));
    DBuf<unsigned long long> d_live(1);
    ECO_CUDA(cudaMemsetAsync(d_live.p, 0, sizeof(unsigned long long), st));
    d_tmp.upload(terminal, ns, st);
    to_internal_kernel<Real><<<grid_for(ns), 256, 0, st>>>(d_tmp.p, d_J.p + (size_t)H * ns, ns, pr->j_inf);
    ECO_CUDA(cudaGetLastError());
    ++launches;
    double sweep_ms = 0.0;
    std::vector<Geometry<Real>> toyG(tabs ? H : 0);
    if (tabs) {
        for (int k = 0; k < H; ++k) {
            TablesDev tk;
            tk.upload(&tabs[k], (size_t)nv * U, st);
            toyG[k].dims = GeomDims{1, nv, nx, U, pr->n_te, pr->n_tb, pr->delta_d, pr->a_min, pr->a_max,
                                    pr->gamma, pr->dtg};
            build_geometry(toyG[k], d_plant.p, d_plans.p + k, d_v.p + (size_t)k * nv, d_te.p, d_tb.p, d_soc.p,
                           tk.view, st, &launches);
            ECO_CUDA(cudaStreamSynchronize(st));   // tk freed at scope end
        }
    }
    sweep.start(st);
    for (int k = H - 1; k >= 0; --k) {
        StageArgs<Real> a = tabs ? stage_args(toyG[k], 0, d_v.p + (size_t)k * nv, nt)
                                 : stage_args(G, k, d_v.p + (size_t)k * nv, nt);
        a.green = d_green.p + (size_t)k * nt;
        a.dep_ok = d_dep.p + (size_t)k * nt;
        a.t_dep = d_tdep.p + (size_t)k * nt;
        a.wait = d_wait.p + (size_t)k * nt;
        a.J_next = d_J.p + (size_t)(k + 1) * ns;
        a.J_out = d_J.p + (size_t)k * ns;
        a.P_out = d_P.p + (size_t)k * ns;
        a.live = count ? d_live.p : nullptr;
        a.src_kind = plans[k].src_kind;
        a.t0 = pr->t0;
        a.dtg = pr->dtg;
        a.j_inf = (Real)pr->j_inf;
        launch_stage<Real, 0>(a, count, st);
        ++launches;
    }
    sweep.stop(st);
    to_external_kernel<Real><<<grid_for(ns * (H + 1)), 256, 0, st>>>(d_J.p, d_tmp.p, ns * (H + 1), pr->j_inf);
    ECO_CUDA(cudaGetLastError());
    ++launches;
    all.stop(st);
    d_tmp.download(J_stack, ns * (H + 1), st);
    d_P.download(P_stack, ns * H, st);
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
        v_min.alloc(n); v_max.alloc(n); grade.alloc(n); cos_g.alloc(n); sin_g.alloc(n);
        cycle.alloc(n); offset.alloc(n); win.alloc((size_t)n * ECO_MAX_WINDOWS * 2);
        kinds.alloc(n); nwin.alloc(n); vaxes.alloc((size_t)n * nv);
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

template <typename Real>
void field_build_impl(const EcoRoute* r, const EcoMpcConfig* c, Geometry<Real>& G, RouteDev& R,
                      const double* d_soc, DBuf<double>& d_field_ext, cudaStream_t st, int64_t* launches,
                      double* sweep_ms) {
    const int n = r->node_count, nv = c->n_v, nx = c->n_soc;
    const size_t lvl = (size_t)nv * nx;
    DBuf<Real> d_G((size_t)n * lvl);
    d_field_ext.alloc((size_t)n * lvl);
    field_init_kernel<<<1, 256, 0, st>>>(d_soc, R.vaxes.p + (size_t)(n - 1) * nv, nv, nx, c->soc_target,
                                         c->soc_weight, c->j_inf, r->kinds[n - 1] == ECO_NODE_STOP ? 1 : 0,
                                         d_field_ext.p + (size_t)(n - 1) * lvl);
    to_internal_kernel<Real><<<grid_for(lvl), 256, 0, st>>>(d_field_ext.p + (size_t)(n - 1) * lvl,
                                                            d_G.p + (size_t)(n - 1) * lvl, lvl, c->j_inf);
    ECO_CUDA(cudaGetLastError());
    *launches += 2;
    EventTimer tm;
    tm.start(st);
    for (int s = n - 2; s >= 0; --s) {
        StageArgs<Real> a = stage_args(G, s, R.vaxes.p + (size_t)s * nv, 1);
        a.J_next = d_G.p + (size_t)(s + 1) * lvl;
        a.J_out = d_G.p + (size_t)s * lvl;
        a.P_out = nullptr;
        // always-green field: a light is an ordinary launch point (mpc.py:141-142)
        a.src_kind = r->kinds[s] == ECO_NODE_SIGNAL ? ECO_NODE_PLAIN : r->kinds[s];
        a.dwell = r->stop_dwell;
        a.j_inf = (Real)c->j_inf;
        launch_stage<Real, 1>(a, false, st);
        ++*launches;
    }
    tm.stop(st);
    to_external_kernel<Real><<<grid_for((size_t)(n - 1) * lvl), 256, 0, st>>>(d_G.p, d_field_ext.p,
                                                                             (size_t)(n - 1) * lvl, c->j_inf);
    ECO_CUDA(cudaGetLastError());
    ++*launches;
    if (sweep_ms) *sweep_ms += tm.ms();
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

    void init(const EcoPlant* p, const EcoRoute* r, const EcoMpcConfig* c, cudaStream_t st, int64_t* launches) {
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
        G.dims = GeomDims{r->node_count - 1, c->n_v, c->n_soc, c->n_te * c->n_tb, c->n_te, c->n_tb,
                          r->delta_d, r->accel_min, r->accel_max, c->gamma, c->dt};
        EcoStage1Tables none{};
        build_geometry(G, plant.p, plans.p, R.vaxes.p, te.p, tb.p, soc.p, none, st, launches);
    }
};

template <typename Real>
void field_only_impl(const EcoPlant* p, const EcoRoute* r, const EcoMpcConfig* c, double* field_out,
                     EcoStats* stats) {
    cudaStream_t st = 0;
    int64_t launches = 0;
    EventTimer all;
    all.start(st);
    RouteCtx<Real> ctx;
    ctx.init(p, r, c, st, &launches);
    DBuf<double> d_field;
    double sweep_ms = 0.0;
    field_build_impl<Real>(r, c, ctx.G, ctx.R, ctx.soc.p, d_field, st, &launches, &sweep_ms);
    all.stop(st);
    d_field.download(field_out, d_field.n, st);
    ECO_CUDA(cudaStreamSynchronize(st));
    if (stats) {
        stats->device_ms = all.ms();
        stats->dominant_ms = sweep_ms;
        stats->dense_updates = (int64_t)(r->node_count - 1) * c->n_v * c->n_soc * c->n_te * c->n_tb;
        stats->live_updates = -1;
        stats->stages = r->node_count - 1;
        stats->kernel_launches = launches;
    }
}

template <typename Real>
void mpc_run_impl(const EcoPlant* p, const EcoRoute* r, const EcoMpcConfig* c, const double* x0,
                  const double* field_in, double* field_out, EcoTrajRow* rows, int32_t* n_rows, int32_t* status,
                  int32_t* status_node, double* final_state, EcoStats* stats) {
    cudaStream_t st = 0;
    int64_t launches = 0;
    const int n = r->node_count, nv = c->n_v, nx = c->n_soc, nt = c->n_t, H = c->horizon;
    const int U = c->n_te * c->n_tb;
    const size_t ns = (size_t)nv * nx * nt;
    EventTimer all, loop;
    all.start(st);
    RouteCtx<Real> ctx;
    ctx.init(p, r, c, st, &launches);
    DBuf<double> d_field;
    double sweep_ms = 0.0;
    if (c->use_terminal_field) {
        if (field_in) {
            d_field.alloc((size_t)n * nv * nx);
            d_field.upload(field_in, d_field.n, st);
        } else {
            field_build_impl<Real>(r, c, ctx.G, ctx.R, ctx.soc.p, d_field, st, &launches, &sweep_ms);
        }
    }
    DBuf<LoopState> d_state(1);
    LoopState h0{};
    h0.x[0] = x0[0]; h0.x[1] = x0[1]; h0.x[2] = x0[2];
    d_state.upload(&h0, 1, st);
    DBuf<uint8_t> green((size_t)(H + 1) * nt), dep((size_t)(H + 1) * nt);
    DBuf<double> tdep((size_t)(H + 1) * nt), wait((size_t)(H + 1) * nt), tax(nt);
    Ladders lad{green.p, dep.p, tdep.p, wait.p, tax.p};
    DBuf<Real> d_J((size_t)(H + 1) * ns);
    DBuf<int32_t> d_P(ns);
    DBuf<EcoTrajRow> d_rows(n - 1);
    const int s_begin = c->start_node;
    const int s_end = c->max_steps < 0 ? n - 1 : std::min(n - 1, s_begin + c->max_steps);
    LoopCfg lc{nv, nx, nt, c->n_te, c->n_tb, U, H, c->teleport, c->use_terminal_field, c->dt, c->gamma,
               c->soc_target, c->soc_weight, c->j_inf, ctx.te.p, ctx.tb.p, ctx.soc.p, ctx.R.vaxes.p};
    int64_t stages = 0;
    loop.start(st);
    for (int s = s_begin; s < s_end; ++s) {
        const int h = H < n - 1 - s ? H : n - 1 - s;
        mpc_prepare_kernel<Real><<<1, 256, 0, st>>>(ctx.R.view, lc, d_state.p, s, h,
                                                    c->use_terminal_field ? d_field.p : nullptr, lad,
                                                    d_J.p + (size_t)h * ns);
        ECO_CUDA(cudaGetLastError());
        ++launches;
        for (int k = h - 1; k >= 0; --k) {
            StageArgs<Real> a = stage_args(ctx.G, s + k, ctx.R.vaxes.p + (size_t)(s + k) * nv, nt);
            a.green = green.p + (size_t)(k + 1) * nt;
            a.dep_ok = dep.p + (size_t)k * nt;
            a.t_dep = tdep.p + (size_t)k * nt;
            a.wait = wait.p + (size_t)k * nt;
            a.J_next = d_J.p + (size_t)(k + 1) * ns;
            a.J_out = d_J.p + (size_t)k * ns;
            a.P_out = d_P.p;
            a.status = &d_state.p->status;
            a.src_kind = r->kinds[s + k];
            a.t0_dev = tax.p;   // ladder origin depends on the device-resident clock
            a.dtg = c->dt;
            a.j_inf = (Real)c->j_inf;
            launch_stage<Real, 0>(a, false, st);
            ++launches;
            ++stages;
        }
        mpc_decide_kernel<Real><<<1, kDecideThreads, 0, st>>>(ctx.plant.p, ctx.R.view, lc, d_state.p, s, h, lad,
                                                              d_J.p + ns, d_rows.p);
        ECO_CUDA(cudaGetLastError());
        ++launches;
    }
    loop.stop(st);
    all.stop(st);
    LoopState hs{};
    d_state.download(&hs, 1, st);
    ECO_CUDA(cudaStreamSynchronize(st));
    d_rows.download(rows, hs.n_rows, st);
    if (field_out && c->use_terminal_field) d_field.download(field_out, (size_t)n * nv * nx, st);
    ECO_CUDA(cudaStreamSynchronize(st));
    *n_rows = hs.n_rows;
    *status = hs.status;
    *status_node = hs.status_node;
    final_state[0] = hs.x[0]; final_state[1] = hs.x[1]; final_state[2] = hs.x[2];
    if (stats) {
        stats->device_ms = all.ms();
        stats->dominant_ms = loop.ms();
        stats->dense_updates = (int64_t)stages * (int64_t)ns * U;
        stats->live_updates = -1;
        stats->stages = stages;
        stats->kernel_launches = launches;
    }
}

}  // namespace

// ================================================================== C ABI
extern "C" {

int32_t eco_abi_version(void) { return ECO_ABI_VERSION; }

const char* eco_last_error(void) { return g_err.c_str(); }

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
        const size_t ns = (size_t)prob->n_v * prob->n_soc * prob->n_t;
        std::vector<double> stack(2 * ns);
        if (precision == ECO_FP64)
            solve_horizon_impl<double>(plant, prob, plan, 1, tables, J_next, stack.data(), P_out, count_live, stats);
        else
            solve_horizon_impl<float>(plant, prob, plan, 1, tables, J_next, stack.data(), P_out, count_live, stats);
        std::memcpy(J_out, stack.data(), ns * sizeof(double));
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
        if (precision == ECO_FP64)
            solve_horizon_impl<double>(plant, prob, plans, H, nullptr, terminal, J_stack, P_stack, count_live, stats);
        else
            solve_horizon_impl<float>(plant, prob, plans, H, nullptr, terminal, J_stack, P_stack, count_live, stats);
    });
}

int32_t eco_solve_tables(const EcoPlant* plant, const EcoProblem* prob, const EcoStepPlan* plans,
                         const EcoStage1Tables* tables, int32_t H, const double* terminal, double* J_stack,
                         int32_t* P_stack, int32_t precision) {
    return run_guarded([&] {
        check_plant(plant);
        check_problem(prob);
        if (H < 1 || !plans || !tables || !terminal || !J_stack || !P_stack) throw ArgError{"bad arguments"};
        if (precision == ECO_FP64)
            solve_horizon_impl<double>(plant, prob, plans, H, tables, terminal, J_stack, P_stack, false, nullptr);
        else
            solve_horizon_impl<float>(plant, prob, plans, H, tables, terminal, J_stack, P_stack, false, nullptr);
    });
}

int32_t eco_field_build(const EcoPlant* plant, const EcoRoute* route, const EcoMpcConfig* cfg, double* field_out,
                        EcoStats* stats) {
    return run_guarded([&] {
        check_plant(plant);
        check_cfg(cfg);
        if (!route || !field_out) throw ArgError{"null pointer argument"};
        if (cfg->precision == ECO_FP64) field_only_impl<double>(plant, route, cfg, field_out, stats);
        else field_only_impl<float>(plant, route, cfg, field_out, stats);
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
        if (cfg->precision == ECO_FP64)
            mpc_run_impl<double>(plant, route, cfg, x_start, field_in, field_out, rows, n_rows, status, status_node,
                                 final_state, stats);
        else
            mpc_run_impl<float>(plant, route, cfg, x_start, field_in, field_out, rows, n_rows, status, status_node,
                                final_state, stats);
    });
}

int32_t eco_solve_batch(const EcoPlant* plant, const EcoRoute* routes, int32_t n_scen, const int32_t* s,
                        const double* t_start, const EcoMpcConfig* cfg, double* J0, int32_t* P0, EcoStats* stats) {
    g_err = "eco_solve_batch: not built yet";
    return ECO_ERR_ARG;
}

}  // extern "C"
