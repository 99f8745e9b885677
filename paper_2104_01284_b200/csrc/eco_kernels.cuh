// eco_kernels.cuh — geometry and Bellman-sweep kernels.
//
// Design: the reference's per-step work splits into a part
// that does not depend on the cost-to-go (the (v,u) transition physics of
// dp_stage1_fill K:553-598, the per-(v,u,SoC) battery / SoC-cell lookup of
// dp_stage2_sweep K:657-712) and the part that does (the V gather + argmin,
// K:697-793 / K:536-545).  The first part depends only on the route node,
// so it is computed ONCE per node for all stages (and shared by the terminal
// field sweep and every receding-horizon solve of a closed loop); the per-
// stage kernel is then a pure gather + min over memoized geometry.
#pragma once

#include "eco_plant.cuh"

namespace eco {

// ---------------------------------------------------------------- layouts
// One "plan" = one spatial step m -> m+1 (StepPlan dp.py:173-188).
struct DevPlan {
    int32_t src_kind, dest_kind;
    double cos_g, sin_g, v0d, dvd;
};

// Pair record bits (per (plan, iv, u)); bit layout of PairGeom::meta.
constexpr uint32_t kOk = 1u;       // transition_tail ok (K:374-392)
constexpr uint32_t kGated = 2u;    // v_next > 0: arrival gated on green (K:496)
constexpr uint32_t kDzh = 4u;      // wz > 0: time blend uses zlo+1 (K:513)
constexpr uint32_t kDvh = 8u;      // wv > 0: speed blend uses ivlo+1
constexpr int kIvShift = 8;

template <typename Real>
struct PairGeom {                 // dense [P][n_v][U]
    uint32_t* meta;
    int32_t* zoff;
    Real* c1;
    Real* wv;
    Real* wz;
    double* dt;                   // exact dt_move (standstill relocation)
    double* c1d;                  // exact c1 (standstill hold cost in fp64 order)
    double* pbat;                 // exact battery power
    int16_t* jxlo;                // [P][n_v][U][n_soc], -1 = infeasible SoC move
    Real* wx;                     // [P][n_v][U][n_soc]
};

struct GeomDims {
    int P, nv, nx, U, nte, ntb;
    double delta_d, a_min, a_max, gamma, dtg;
};

// ------------------------------------------------------ stage-1 (v,u) pass
// K:553-598 (+ transition_tail K:374-392).  grid (nv, P), block 256.
// Table mode (tab_* != nullptr) reads the toy tables of dp_sweep_serial's
// use_tables path (K:476-493) instead of evaluating the plant.
template <typename Real>
__global__ void geom_pairs_kernel(const EcoPlant* __restrict__ plant, const DevPlan* __restrict__ plans,
                                  const double* __restrict__ vaxes, const double* __restrict__ te_axis,
                                  const double* __restrict__ tb_axis, GeomDims g, PairGeom<Real> out,
                                  EcoStage1Tables tab) {
    const int iv = blockIdx.x, p = blockIdx.y;
    const EcoPlant& P = *plant;
    const DevPlan pl = plans[p];
    const double v = vaxes[(size_t)p * g.nv + iv];
    __shared__ StepPre q;
    if (threadIdx.x == 0 && tab.ok == nullptr) q = step_pre(P, v, pl.cos_g, pl.sin_g);
    __syncthreads();
    const size_t base = ((size_t)p * g.nv + iv) * g.U;
    for (int u = threadIdx.x; u < g.U; u += blockDim.x) {
        const int ite = u / g.ntb, itb = u - ite * g.ntb;
        bool ok;
        double v2, dt, pb, c1, wv, wz;
        int ivlo, ivhi, zoff;
        if (tab.ok == nullptr) {
            StepOut o = step_eval_pre(P, v, te_axis[ite], tb_axis[itb], g.delta_d, g.a_min, g.a_max, 0.0, q);
            ok = o.feas == kFeasOk;
            if (ok && o.clamped && pl.dest_kind == ECO_NODE_PLAIN) ok = false;
            if (ok && pl.dest_kind == ECO_NODE_STOP && o.v_next > 0.0) ok = false;
            if (ok) ok = locate_uniform(o.v_next, pl.v0d, pl.dvd, g.nv, &ivlo, &ivhi, &wv);
            v2 = o.v_next; dt = o.dt_move; pb = o.p_bat;
            c1 = stage_cost(o.mf, dt, g.gamma);
            if (ok) tcell_shift(dt, g.dtg, &zoff, &wz);
        } else {
            const size_t c = (size_t)iv * g.U + u;
            ok = tab.ok[c] != 0;
            v2 = tab.v2[c]; dt = tab.dt[c]; pb = tab.pbat[c]; c1 = tab.c1[c];
            ivlo = tab.ivlo[c]; ivhi = tab.ivhi[c]; wv = tab.wv[c]; zoff = tab.zoff[c]; wz = tab.wz[c];
        }
        uint32_t m = 0;
        if (ok) {
            m = kOk | (v2 > 0.0 ? kGated : 0u) | (wz > 0.0 ? kDzh : 0u) | (ivhi != ivlo ? kDvh : 0u) |
                ((uint32_t)ivlo << kIvShift);
        }
        out.meta[base + u] = m;
        out.zoff[base + u] = ok ? zoff : 0;
        out.c1[base + u] = (Real)(ok ? c1 : 0.0);
        out.wv[base + u] = (Real)(ok ? wv : 0.0);
        out.wz[base + u] = (Real)(ok ? wz : 0.0);
        out.dt[base + u] = ok ? dt : 0.0;
        out.c1d[base + u] = ok ? c1 : 0.0;
        out.pbat[base + u] = ok ? pb : 0.0;
    }
}

// ------------------------------------------------------- SoC-cell pass
// Battery current per (v, T_bsg, SoC) shared by the torque column (K:657-672),
// then xi' = xi - dt*I/C_nom and its cell (K:498-506 / K:709-712).
// grid (nv, P), block 256; per_action_pbat = toy mode (K:676-683).
template <typename Real>
__global__ void geom_soc_kernel(const EcoPlant* __restrict__ plant, const double* __restrict__ vaxes,
                                const double* __restrict__ tb_axis, const double* __restrict__ soc_axis,
                                GeomDims g, PairGeom<Real> out, int per_action_pbat) {
    extern __shared__ double sm[];
    double* cur = sm;                                   // [ntb][nx]
    uint8_t* cur_ok = (uint8_t*)(sm + g.ntb * g.nx);    // [ntb][nx]
    const int iv = blockIdx.x, p = blockIdx.y;
    const EcoPlant& P = *plant;
    const double v = vaxes[(size_t)p * g.nv + iv];
    const double x0 = soc_axis[0];
    const double dx = (soc_axis[g.nx - 1] - soc_axis[0]) / (g.nx - 1);
    if (!per_action_pbat) {
        const Drive d = drivetrain(P, v);
        for (int i = threadIdx.x; i < g.ntb * g.nx; i += blockDim.x) {
            const int itb = i / g.nx, jx = i - itb * g.nx;
            const double pb = bsg_power(P, d.w_bsg, tb_axis[itb]);
            double c;
            cur_ok[i] = battery_current(P, pb, soc_axis[jx], &c) ? 1 : 0;
            cur[i] = c;
        }
    }
    __syncthreads();
    const size_t base = ((size_t)p * g.nv + iv) * g.U;
    for (int i = threadIdx.x; i < g.U * g.nx; i += blockDim.x) {
        const int u = i / g.nx, jx = i - u * g.nx;
        const size_t gi = (base + u) * g.nx + jx;
        int16_t lo16 = -1;
        Real wxr = (Real)0;
        if (out.meta[base + u] & kOk) {
            double c;
            bool okb;
            if (per_action_pbat) {
                okb = battery_current(P, out.pbat[base + u], soc_axis[jx], &c);
            } else {
                const int itb = u % g.ntb;
                okb = cur_ok[itb * g.nx + jx] != 0;
                c = cur[itb * g.nx + jx];
            }
            if (okb) {
                const double xi2 = soc_axis[jx] - out.dt[base + u] * c / P.c_nom;
                int lo, hi;
                double w;
                if (locate_uniform(xi2, x0, dx, g.nx, &lo, &hi, &w)) { lo16 = (int16_t)lo; wxr = (Real)w; }
            }
        }
        out.jxlo[gi] = lo16;
        out.wx[gi] = wxr;
    }
}

// ---------------------------------------------------------- stage sweep
// Internal cost-to-go representation: +inf marks infeasible (the reference's
// j_inf).  A gather touching an infeasible corner then yields inf or NaN and
// can never pass the strict F < best test — the absorbing rule of
// bilin2_abs / interp3_abs (K:325-361) without per-corner tests.
template <typename Real>
struct StageArgs {
    // geometry of this stage's plan
    const uint32_t* meta;
    const int32_t* zoff;
    const Real* c1;
    const Real* wv;
    const Real* wz;
    const double* dt;
    const double* c1d;
    const int16_t* jxlo;
    const Real* wx;
    const double* v_src;
    // ladders (n_t): destination green mask, source standstill arrays
    const uint8_t* green;
    const uint8_t* dep_ok;
    const double* t_dep;
    const double* wait;
    const Real* J_next;
    Real* J_out;
    int32_t* P_out;               // nullptr in field mode
    unsigned long long* live;     // nullptr unless counting
    const int32_t* status;        // closed loop: skip when nonzero (nullable)
    const double* t0_dev;         // closed loop: ladder origin on the device (nullable)
    int nv, nx, nt, U;
    int src_kind;
    double t0, dtg, gamma, dwell;
    Real j_inf;
};

// a + w*(b - a).  Double: unfused (the library builds with -fmad=false), the
// reference's exact expression tree.  Float: one FMA.
__device__ __forceinline__ double lerp(double a, double b, double w) { return a + w * (b - a); }
__device__ __forceinline__ float lerp(float a, float b, float w) { return __fmaf_rn(w, b - a, a); }

// MODE 0: (v, soc, t) step (dp_sweep_serial K:421-546 / dp_stage2_sweep).
// MODE 1: (v, soc) terminal-field step (field_sweep K:801-865): no time
//         axis, stop-sign dwell charged at the time price.
template <typename Real, int MODE, int TILE, int SLICES, bool COUNT>
__global__ void __launch_bounds__(TILE * SLICES)
bellman_stage_kernel(StageArgs<Real> a) {
    __shared__ Real s_best[SLICES][TILE];
    __shared__ int32_t s_arg[SLICES][TILE];
    if (a.status && *a.status != 0) return;
    const int plane = a.nx * a.nt;
    const int tiles_per_plane = (plane + TILE - 1) / TILE;
    const int iv = blockIdx.x / tiles_per_plane;
    const int f = (blockIdx.x - iv * tiles_per_plane) * TILE + (threadIdx.x % TILE);
    const int slice = threadIdx.x / TILE;
    const bool active = f < plane;
    const int jx = active ? f / a.nt : 0;
    const int z = active ? f - jx * a.nt : 0;
    const double v = a.v_src[iv];
    const bool skip = (a.src_kind == ECO_NODE_STOP && v > 0.0);   // K:458-459
    const bool standstill = v == 0.0;
    const int nt = a.nt, nx = a.nx;

    Real best = a.j_inf;
    int32_t bu = -1;
    unsigned long long nlive = 0;

    if (active && !skip) {
        const size_t pbase = (size_t)iv * a.U;
        // stop-sign dwell of the field sweep (K:825) / per-z hold of the 3-D sweep
        const double hold_field = (MODE == 1 && a.src_kind == ECO_NODE_STOP && standstill)
                                      ? (1.0 - a.gamma) * a.dwell : 0.0;
        uint8_t dep = 1;
        double hold_z = 0.0, tdep_z = 0.0;
        if (MODE == 0 && standstill) { dep = a.dep_ok[z]; hold_z = a.wait[z]; tdep_z = a.t_dep[z]; }
        if (dep) {
            for (int u = slice; u < a.U; u += SLICES) {
                const uint32_t m = __ldg(a.meta + pbase + u);
                if (!(m & kOk)) continue;
                const size_t gi = (pbase + u) * nx + jx;
                const int jxlo = __ldg(a.jxlo + gi);
                if (jxlo < 0) continue;
                const Real wx = __ldg(a.wx + gi);
                const int jxhi = jxlo + (wx > (Real)0 ? 1 : 0);
                const int ivlo = (int)(m >> kIvShift);
                const int ivhi = ivlo + ((m & kDvh) ? 1 : 0);
                const Real wv = __ldg(a.wv + pbase + u);
                int zlo = 0, zhi = 0;
                Real wz = (Real)0;
                double hold = 0.0;
                if (MODE == 0) {
                    const int zoff = __ldg(a.zoff + pbase + u);
                    if (standstill && hold_z > 0.0) {      // red wait / stop dwell relocation K:523-527
                        const double t2 = tdep_z + __ldg(a.dt + pbase + u);
                        double w;
                        const double t0 = a.t0_dev ? a.t0_dev[0] : a.t0;
                        if (!locate_uniform(t2, t0, a.dtg, nt, &zlo, &zhi, &w)) continue;
                        wz = (Real)w;
                        hold = hold_z;
                    } else {                                // constant ladder shift K:508-515
                        zlo = z + zoff;
                        zhi = zlo + ((m & kDzh) ? 1 : 0);
                        if (zhi > nt - 1) continue;
                        wz = __ldg(a.wz + pbase + u);
                    }
                    if ((m & kGated) && a.green[zlo] == 0) continue;   // K:516 / K:534
                } else {
                    hold = hold_field;
                }
                if (COUNT) ++nlive;
                const Real* J = a.J_next;
                const size_t r00 = ((size_t)ivlo * nx + jxlo) * nt, r10 = ((size_t)ivhi * nx + jxlo) * nt;
                const size_t r01 = ((size_t)ivlo * nx + jxhi) * nt, r11 = ((size_t)ivhi * nx + jxhi) * nt;
                // bilin2_abs nesting (K:335-337): v inside, then soc; then t (K:361)
                const Real lo0 = lerp(__ldg(J + r00 + zlo), __ldg(J + r10 + zlo), wv);
                const Real hi0 = lerp(__ldg(J + r01 + zlo), __ldg(J + r11 + zlo), wv);
                Real jn = lerp(lo0, hi0, wx);
                if (zhi != zlo) {
                    const Real lo1 = lerp(__ldg(J + r00 + zhi), __ldg(J + r10 + zhi), wv);
                    const Real hi1 = lerp(__ldg(J + r01 + zhi), __ldg(J + r11 + zhi), wv);
                    jn = lerp(jn, lerp(lo1, hi1, wx), wz);
                }
                // F = c1 + (1-gamma)*hold + Jn, left to right (K:542 / K:862)
                Real F;
                if (hold > 0.0) {
                    const double c = __ldg(a.c1d + pbase + u) + (MODE == 0 ? (1.0 - a.gamma) * hold : hold);
                    F = (Real)c + jn;
                } else {
                    F = __ldg(a.c1 + pbase + u) + jn;
                }
                if (F < best) { best = F; bu = u; }
            }
        }
    }
    if (COUNT && a.live) {
        unsigned long long w = nlive;
        for (int o = 16; o > 0; o >>= 1) w += __shfl_down_sync(0xffffffffu, w, o);
        if ((threadIdx.x & 31) == 0 && w) atomicAdd(a.live, w);
    }
    s_best[slice][threadIdx.x % TILE] = best;
    s_arg[slice][threadIdx.x % TILE] = bu;
    __syncthreads();
    if (slice == 0 && active) {
        for (int s = 1; s < SLICES; ++s) {
            const int32_t u2 = s_arg[s][threadIdx.x];
            if (u2 < 0) continue;
            const Real b2 = s_best[s][threadIdx.x];
            if (bu < 0 || b2 < best || (b2 == best && u2 < bu)) { best = b2; bu = u2; }
        }
        const size_t o = (size_t)iv * plane + f;
        a.J_out[o] = bu < 0 ? (Real)INFINITY : best;
        if (MODE == 0) a.P_out[o] = bu;
    }
}

}  // namespace eco
