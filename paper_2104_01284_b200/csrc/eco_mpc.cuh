// eco_mpc.cuh — device-resident receding-horizon loop pieces.
//
//   ladders / seed   <- build_context        dp.py:255-341  (ladders at x.t; terminal level)
//   candidates/pick  <- _argmin_at_state     mpc.py:189-278
//                       + _max_braking_decision mpc.py:490-510
//                       + propagate_state_full  plant.py:341-439
//                       + simulate_closed_loop  mpc.py:549-594 (row log, mismatch check)
//
// The state x = (v, soc, t) never leaves the device during a run.  Per route
// node: the candidates (and the next node's terminal level) beside the h
// stage sweeps, then one pick, which also builds the next node's ladders.
#pragma once

#include "eco_kernels.cuh"

namespace eco {

__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

struct DevRoute {               // device copies of EcoRoute arrays
    int n;
    double delta_d, accel_min, accel_max, stop_dwell;
    const double* v_min;
    const double* v_max;
    const double* grade;
    const double* cos_g;
    const double* sin_g;
    const int8_t* kinds;
    const double* sig_cycle;
    const double* sig_offset;
    const int32_t* sig_nwin;
    const double* sig_win;
};

struct LoopState {              // lives in device memory for the whole run
    double x[3];                // v, soc, t
    int32_t status;             // ECO_RUN_* (3 = prediction mismatch)
    int32_t status_node;
    int32_t n_rows;
    int32_t pad;
    unsigned long long prep_ns;     // globaltimer at this step's prepare entry
    unsigned long long sweep_ns;    // summed prepare-entry -> pick-entry clocks
};

struct Ladders {                // [H+1][nt] per receding-horizon solve
    uint8_t* green;
    uint8_t* dep_ok;
    double* t_dep;
    double* wait;
    double* t_axis;             // [nt]
    int* flags;                 // [H] kStageAny* of stage k (nullable)
};

// kStageAny* bits of stages 0..h-1 from ladders [h+1][nt] (stage k arrives at
// node k + 1, departs node k); one block, after the ladders are complete.
__device__ __forceinline__ void ladder_flags(const uint8_t* green, const uint8_t* dep, const double* wait, int nt,
                                             int h, int* flags) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int k = w; k < h; k += nw) {
        int red = 0, hold = 0;
        for (int z = lane; z < nt; z += 32) {
            red |= green[(size_t)(k + 1) * nt + z] == 0;
            hold |= (dep[(size_t)k * nt + z] == 0) | (wait[(size_t)k * nt + z] > 0.0);
        }
        red = __any_sync(0xffffffffu, red);
        hold = __any_sync(0xffffffffu, hold);
        if (lane == 0) flags[k] = (red ? kStageAnyRed : 0) | (hold ? kStageAnyHold : 0);
    }
}

struct LoopCfg {
    int nv, nx, nt, nte, ntb, U, H, teleport, use_field;
    double dt, gamma, soc_target, soc_weight, j_inf;
    const double* te_axis;
    const double* tb_axis;
    const double* soc_axis;     // [nx]
    const double* vaxes;        // [n][nv] node speed axes
};

// _node_time_arrays dp.py:217-252 for one node on the ladder; the signal
// phase plan (cycle, offset, green windows) is passed explicitly
__device__ __forceinline__ void ladder_entry(int kind, double cycle, double offset, const double* win, int nwin,
                                             double dwell, double tz, int teleport, uint8_t* green, uint8_t* dep,
                                             double* tdep, double* wait, int z) {
    uint8_t g = 1, d = 1;
    double td = tz, w = 0.0;
    if (kind == ECO_NODE_SIGNAL) {
        if (!sig_is_green(cycle, offset, win, nwin, tz)) {
            g = 0;
            if (teleport) {
                const double ng = sig_next_green(cycle, offset, win, nwin, tz);
                td = ng;
                w = ng - tz;
            } else {
                d = 0;
            }
        }
    } else if (kind == ECO_NODE_STOP) {
        td = tz + dwell;
        w = dwell;
    }
    green[z] = g; dep[z] = d; tdep[z] = td; wait[z] = w;
}

__device__ __forceinline__ void node_ladder(const DevRoute& r, int node, const double* t_axis, int nt, int teleport,
                                            uint8_t* green, uint8_t* dep, double* tdep, double* wait, int z) {
    (void)nt;
    ladder_entry(r.kinds[node], r.sig_cycle[node], r.sig_offset[node],
                 r.sig_win + (size_t)node * ECO_MAX_WINDOWS * 2, r.sig_nwin[node], r.stop_dwell, t_axis[z], teleport,
                 green, dep, tdep, wait, z);
}

// terminal seed dp.py:322-334: min(base + w*(xi - xi*)^2, j_inf), j_inf where
// base >= j_inf, constant along t; written in the internal (+inf) form.
template <typename Real>
__device__ __forceinline__ Real terminal_value(double base, double soc, double target, double weight, double j_inf) {
    const double d = soc - target;
    const double q = weight * (d * d);
    double val;
    if (base >= j_inf) val = j_inf;
    else { val = base + q; if (!(val < j_inf)) val = j_inf; }
    return val >= j_inf ? (Real)INFINITY : (Real)val;
}

// build_context (dp.py:255-341) on the device, in two x-independent /
// x-dependent halves.
//
// build_ladders: the time ladder at clock t (GridSpec.t_axis dp.py:75-77),
// the node ladders of nodes s..s+h (dp.py:217-252) and the per-stage flags;
// one block.  Run by the pick kernel for the next step (the clock is known
// once the decision is applied) and by mpc_ladders_kernel for a run's first
// step.
__device__ void build_ladders(const DevRoute& r, const LoopCfg& c, double t, int s, int h, const Ladders& lad) {
    __shared__ double t_axis[1024];
    const double t0 = c.dt * floor(t / c.dt);
    const int nt = c.nt;
    for (int z = threadIdx.x; z < nt; z += blockDim.x) {
        const double tz = t0 + c.dt * (double)z;
        lad.t_axis[z] = tz;
        if (z < 1024) t_axis[z] = tz;
    }
    __syncthreads();
    const double* tax = nt <= 1024 ? t_axis : lad.t_axis;
    for (int i = threadIdx.x; i < (h + 1) * nt; i += blockDim.x) {
        const int k = i / nt, z = i - k * nt;
        node_ladder(r, s + k, tax, nt, c.teleport, lad.green + k * nt, lad.dep_ok + k * nt, lad.t_dep + k * nt,
                    lad.wait + k * nt, z);
    }
    if (lad.flags) {
        __syncthreads();
        ladder_flags(lad.green, lad.dep_ok, lad.wait, nt, h, lad.flags);
    }
}

// The first step's ladders.  The per-step solve clock starts when a step's
// ladders are in place (prep_ns) and stops at the pick's entry: device
// timestamps instead of event nodes, which cost ~20 us per step in the graph.
__global__ void mpc_ladders_kernel(DevRoute r, LoopCfg c, LoopState* st, int s, int h, Ladders lad) {
    if (st->status != 0) return;
    build_ladders(r, c, st->x[2], s, h, lad);
    if (threadIdx.x == 0) st->prep_ns = globaltimer_ns();
}

// The terminal level J_h of the solve at node s (dp.py:322-334): the field
// slice at node s + h plus the SoC penalty, replicated along t, both level
// copies.  Independent of the vehicle state, so it runs for step s + 1 on the
// side branch of step s (double-buffered levels).
template <typename Real>
__global__ void mpc_seed_kernel(LoopCfg c, int s, int h, const double* field, Real* Jh, Real* Jh1) {
    const int nt = c.nt;
    const int ncell = c.nv * c.nx;
    const int total = ncell * nt;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
        const int cell = i / nt;
        const int jx = cell - (cell / c.nx) * c.nx;
        const double base = (c.use_field && field) ? field[(size_t)(s + h) * ncell + cell] : 0.0;
        const Real val = terminal_value<Real>(base, c.soc_axis[jx], c.soc_target, c.soc_weight, c.j_inf);
        Jh[i] = val;
        if (i > 0) Jh1[i - 1] = val;      // shifted copy (see level_copy in eco_api.cu)
    }
    if (blockIdx.x == 0)
        for (int i = total - 1 + threadIdx.x; i < total + 8; i += blockDim.x) {
            Jh1[i] = (Real)INFINITY;
            if (i >= total) Jh[i] = (Real)INFINITY;
        }
}

// interp3_abs (K:340-361) on an internal table at a continuous query,
// CostToGoTable.interpolate dp.py:115-134: returns j_inf when infeasible.
template <typename Real>
__device__ double table_interp(const Real* J, const double* va, int nv, const double* xa, int nx,
                               const double* ta, int nt, double j_inf, double v, double x, double t) {
    const double v0 = va[0], dv = (va[nv - 1] - v0) / (nv - 1);
    const double x0 = xa[0], dx = (xa[nx - 1] - x0) / (nx - 1);
    const double t0 = ta[0], dtg = (ta[nt - 1] - t0) / (nt - 1);
    int a0, a1, b0, b1, c0, c1;
    double wa, wb, wc;
    const bool ok = locate_uniform(v, v0, dv, nv, &a0, &a1, &wa) && locate_uniform(x, x0, dx, nx, &b0, &b1, &wb) &&
                    locate_uniform(t, t0, dtg, nt, &c0, &c1, &wc);
    if (!ok) return j_inf;
    auto at = [&](int i, int j, int k) -> double {
        const Real r = J[((size_t)i * nx + j) * nt + k];
        return r;  // +inf stays +inf
    };
    auto bil = [&](int k) -> double {
        const double c00 = at(a0, b0, k), c01 = at(a0, b1, k), c10 = at(a1, b0, k), c11 = at(a1, b1, k);
        if (c00 >= j_inf || c01 >= j_inf || c10 >= j_inf || c11 >= j_inf) return j_inf;
        const double lo = c00 + wa * (c10 - c00);
        const double hi = c01 + wa * (c11 - c01);
        return lo + wb * (hi - lo);
    };
    const double r0 = bil(c0);
    if (r0 >= j_inf) return j_inf;
    if (c1 == c0) return r0;
    const double r1 = bil(c1);
    if (r1 >= j_inf) return j_inf;
    return r0 + wc * (r1 - r0);
}

constexpr int kDecideThreads = 1024;


// The MPC decision (mpc.py:189-278 + 490-510, plant.py:341-439), in two
// kernels.  Everything of the exact-state argmin that does not read the
// solve's tables -- the source-node wait, the plant step of every candidate
// action, its battery current and the floor-sample green gate -- runs in
// mpc_candidates_kernel on a side branch of the MPC step, concurrently with
// the H stage sweeps; mpc_pick_kernel then interpolates J_1 (the solve's
// tables[1]) at each admissible candidate's successor, reduces (f, u)
// lexicographically (= the first win in scan order, mpc.py:269) and applies
// the winner.  For an admissible winner propagate_state_full is its
// candidate evaluation: the same step_eval arithmetic with brake 0 (the
// comfort box only gates feasibility, which it passed), the same battery
// current and departure clock -- so the plant step is the prediction exactly
// (mpc.py:575-582 holds by construction) and is not re-run.
struct DecideCand {            // one candidate action (64 B)
    double pre;                // stage cost + (1 - gamma) * wait
    double v2, soc2, t2, dt_move, mf, accel;
    double ok;                 // 1: admissible before the table lookup
};
struct DecideHead {            // per-step header (block 0, thread 0)
    double wait, t_base;
    int src_ok, gear;
};

__device__ __forceinline__ int decide_source(const DevRoute& r, const LoopCfg& c, int s, int src, double v, double t,
                                             double* wait_out, double* t_base_out) {
    double wait = 0.0, t_base = t;
    int ok = 1;
    if (src == ECO_NODE_STOP) {
        if (v > 0.0) ok = 0;
        wait = r.stop_dwell;
        t_base = t + wait;
    } else if (src == ECO_NODE_SIGNAL && v == 0.0) {
        const double* win = r.sig_win + (size_t)s * ECO_MAX_WINDOWS * 2;
        if (!sig_is_green(r.sig_cycle[s], r.sig_offset[s], win, r.sig_nwin[s], t)) {
            if (!c.teleport) ok = 0;
            t_base = sig_next_green(r.sig_cycle[s], r.sig_offset[s], win, r.sig_nwin[s], t);
            wait = t_base - t;
        }
    }
    *wait_out = wait;
    *t_base_out = t_base;
    return ok;
}

constexpr int kCandThreads = 128;

__global__ void __launch_bounds__(kCandThreads)
mpc_candidates_kernel(const EcoPlant* __restrict__ plant, DevRoute r, LoopCfg c, const LoopState* st, int s,
                      Ladders lad, DecideCand* cand, DecideHead* head) {
    if (st->status != 0) return;
    const EcoPlant& P = *plant;
    const double v = st->x[0], soc = st->x[1], t = st->x[2];
    const int src = r.kinds[s], dst = r.kinds[s + 1];
    double wait, t_base;
    const int src_ok = decide_source(r, c, s, src, v, t, &wait, &t_base);
    const StepPre q = step_pre(P, v, r.cos_g[s], r.sin_g[s]);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        head->wait = wait; head->t_base = t_base; head->src_ok = src_ok; head->gear = q.d.gear;
    }
    const int u = blockIdx.x * blockDim.x + threadIdx.x;
    if (u >= c.U) return;
    DecideCand k{};
    k.ok = 0.0;
    if (src_ok) {
        const int ite = u / c.ntb, itb = u - ite * c.ntb;
        const double te = c.te_axis[ite], tb = c.tb_axis[itb];
        if (!(te > q.te_hi || te < q.te_lo || tb > q.tb_hi || tb < q.tb_lo)) {
            const StepOut o = step_eval_pre(P, v, te, tb, r.delta_d, r.accel_min, r.accel_max, 0.0, q);
            double cur;
            if (o.feas == kFeasOk && !(o.clamped && dst == ECO_NODE_PLAIN) && !(dst == ECO_NODE_STOP && o.v_next > 0.0) &&
                battery_current(P, o.p_bat, soc, &cur)) {
                const double soc2 = soc - o.dt_move * cur / P.c_nom;
                const double t2 = t_base + o.dt_move;
                bool gate = true;
                if (o.v_next > 0.0) {            // floor-sample green gate mpc.py:256-261
                    int zlo, zhi;
                    double w;
                    if (locate_uniform(t2, lad.t_axis[0], c.dt, c.nt, &zlo, &zhi, &w) && lad.green[c.nt + zlo] == 0)
                        gate = false;
                }
                if (gate) {
                    k.pre = stage_cost(o.mf, o.dt_move, c.gamma) + (1.0 - c.gamma) * wait;
                    k.v2 = o.v_next; k.soc2 = soc2; k.t2 = t2;
                    k.dt_move = o.dt_move; k.mf = o.mf; k.accel = o.accel;
                    k.ok = 1.0;
                }
            }
        }
    }
    cand[u] = k;
}

__device__ __forceinline__ bool decide_better(double f2, int u2, double f, int u) {
    return u2 >= 0 && (u < 0 || f2 < f || (f2 == f && u2 < u));
}

// Applies the decision (thread 0): the winner's plant step, or the
// max-brake fallback (mpc.py:490-510) and propagate_state_full; writes the
// trajectory row and the next state, or a failure status.
__device__ void decide_apply(const EcoPlant* __restrict__ plant, const DevRoute& r, const LoopCfg& c, LoopState* st,
                             int s, int h, int bestu, double bestf, const DecideCand* __restrict__ cand,
                             const DecideHead* __restrict__ head, EcoTrajRow* rows) {
    const double v = st->x[0], soc = st->x[1], t = st->x[2];
    const int src = r.kinds[s], dst = r.kinds[s + 1];
    EcoTrajRow row{};
    row.s = s; row.v = v; row.soc = soc; row.t = t; row.horizon = h;
    if (bestu >= 0) {
        // the winner's candidate evaluation is its plant step (see above)
        const DecideCand* k = cand + bestu;
        row.cost_to_go = bestf;
        row.t_eng = c.te_axis[bestu / c.ntb]; row.t_bsg = c.tb_axis[bestu % c.ntb]; row.brake_force = 0.0;
        row.gear = head->gear;
        row.wait_s = head->wait; row.dt_move_s = k->dt_move; row.fuel_inc_g = k->mf * k->dt_move;
        row.accel = k->accel;
        rows[st->n_rows] = row;
        st->n_rows += 1;
        st->x[0] = k->v2; st->x[1] = k->soc2; st->x[2] = k->t2;
        return;
    }
    // _max_braking_decision mpc.py:490-510, then propagate_state_full (rare path)
    const EcoPlant& P = *plant;
    const StepPre q = step_pre(P, v, r.cos_g[s], r.sin_g[s]);
    if (v <= 0.0) { st->status = ECO_RUN_INFEASIBLE; st->status_node = s; return; }
    double a_target;
    if (dst == ECO_NODE_PLAIN) {
        const double a_stop = -(v * v) / (2.0 * r.delta_d) * (1.0 - 1.0e-2);
        a_target = r.accel_min >= a_stop ? r.accel_min : a_stop;
    } else {
        a_target = r.accel_min;
    }
    const double f_road = road_load(P, v, r.cos_g[s], r.sin_g[s]);
    const double b = -(P.mass * a_target + f_road);
    const double brake = b > 0.0 ? b : 0.0;
    row.cost_to_go = __longlong_as_double(0x7ff8000000000000ULL);   // NaN (ControlDecision default)
    row.fallback = 1;
    const double te = 0.0, tb = 0.0;
    if (!(q.te_lo <= te && te <= q.te_hi) || !(q.tb_lo <= tb && tb <= q.tb_hi) || brake < 0.0) {
        st->status = ECO_RUN_PLANT; st->status_node = s; return;
    }
    double wait_p = 0.0, tb_p = t;
    if (v == 0.0) {
        if (src == ECO_NODE_SIGNAL) {
            const double* win = r.sig_win + (size_t)s * ECO_MAX_WINDOWS * 2;
            if (!sig_is_green(r.sig_cycle[s], r.sig_offset[s], win, r.sig_nwin[s], t)) {
                if (!c.teleport) { st->status = ECO_RUN_PLANT; st->status_node = s; return; }
                tb_p = sig_next_green(r.sig_cycle[s], r.sig_offset[s], win, r.sig_nwin[s], t);
                wait_p = tb_p - t;
            }
        } else if (src == ECO_NODE_STOP) {
            wait_p = r.stop_dwell;
            tb_p = t + wait_p;
        }
    }
    const StepOut o = step_eval_pre(P, v, te, tb, r.delta_d, -INFINITY, INFINITY, brake, q);
    if (o.feas == kFeasNoMotion || (o.clamped && dst == ECO_NODE_PLAIN) || (dst == ECO_NODE_STOP && o.v_next > 0.0)) {
        st->status = ECO_RUN_PLANT; st->status_node = s; return;
    }
    double cur;
    if (!battery_current(P, o.p_bat, soc, &cur)) { st->status = ECO_RUN_PLANT; st->status_node = s; return; }
    row.t_eng = te; row.t_bsg = tb; row.brake_force = brake;
    row.gear = q.d.gear;
    row.wait_s = wait_p; row.dt_move_s = o.dt_move; row.fuel_inc_g = o.mf * o.dt_move; row.accel = o.accel;
    rows[st->n_rows] = row;
    st->n_rows += 1;
    st->x[0] = o.v_next; st->x[1] = soc - o.dt_move * cur / P.c_nom; st->x[2] = tb_p + o.dt_move;
}

template <typename Real>
__global__ void __launch_bounds__(kDecideThreads)
mpc_pick_kernel(const EcoPlant* __restrict__ plant, DevRoute r, LoopCfg c, LoopState* st, int s, int h,
                const Real* J1, const DecideCand* __restrict__ cand, const DecideHead* __restrict__ head,
                Ladders lad, EcoTrajRow* rows, unsigned long long* step_ns, int s_next, int h_next) {
    // launched programmatically after the last stage sweep: resident during
    // its tail, then waits for J_1.  The next step's first stage may start
    // its prologue early: it reads the ladders built at the end of this
    // kernel only after its own grid dependency wait.
    pdl_launch_dependents();
    pdl_wait();
    if (st->status != 0) return;
    if (threadIdx.x == 0) {                      // per-step solve clock (see mpc_ladders_kernel)
        const unsigned long long dt = globaltimer_ns() - st->prep_ns;
        st->sweep_ns += dt;
        step_ns[st->n_rows] = dt;
    }
    const double* v1 = c.vaxes + (size_t)(s + 1) * c.nv;
    double bestf = 0.0;
    int bestu = -1;
    for (int u = threadIdx.x; u < c.U; u += blockDim.x) {
        const DecideCand* k = cand + u;
        if (k->ok == 0.0) continue;
        const double jn = table_interp<Real>(J1, v1, c.nv, c.soc_axis, c.nx, lad.t_axis, c.nt, c.j_inf, k->v2,
                                             k->soc2, k->t2);
        if (!(jn < c.j_inf)) continue;
        const double f = k->pre + jn;
        if (bestu < 0 || f < bestf) { bestf = f; bestu = u; }
    }
    for (int o = 16; o > 0; o >>= 1) {
        const double f2 = __shfl_down_sync(0xffffffffu, bestf, o);
        const int u2 = __shfl_down_sync(0xffffffffu, bestu, o);
        if (decide_better(f2, u2, bestf, bestu)) { bestf = f2; bestu = u2; }
    }
    __shared__ double s_f[kDecideThreads / 32];
    __shared__ int s_u[kDecideThreads / 32];
    const int nw = (int)(blockDim.x >> 5), lane = threadIdx.x & 31;
    if (lane == 0) { s_f[threadIdx.x >> 5] = bestf; s_u[threadIdx.x >> 5] = bestu; }
    __syncthreads();
    if (threadIdx.x < 32) {
        bestf = lane < nw ? s_f[lane] : 0.0;
        bestu = lane < nw ? s_u[lane] : -1;
        for (int o = 16; o > 0; o >>= 1) {
            const double f2 = __shfl_down_sync(0xffffffffu, bestf, o);
            const int u2 = __shfl_down_sync(0xffffffffu, bestu, o);
            if (decide_better(f2, u2, bestf, bestu)) { bestf = f2; bestu = u2; }
        }
        if (threadIdx.x == 0) decide_apply(plant, r, c, st, s, h, bestu, bestf, cand, head, rows);
    }
    if (s_next < 0) return;
    // the next step's ladders at the new clock (build_context's x-dependent half)
    __syncthreads();
    if (st->status != 0) return;
    build_ladders(r, c, st->x[2], s_next, h_next, lad);
    if (threadIdx.x == 0) st->prep_ns = globaltimer_ns();
}

// Batch scenarios (C4): per scenario b the time ladder at t_start[b]
// (GridSpec.t_axis dp.py:75-77), the node ladders of nodes s_b..s_b+h_b with
// the scenario's own signal timings, and the terminal level J_{h_b} in buffer
// h_b & 1 (dp.py:322-334).  grid (blocks, B).
template <typename Real>
__global__ void batch_prepare_kernel(DevRoute r, LoopCfg c, const int32_t* __restrict__ sig_of_node, int n_sig,
                                     const EcoSignalTiming* __restrict__ timings, const int32_t* __restrict__ s_arr,
                                     const int32_t* __restrict__ h_arr, const double* __restrict__ t_start, int Hmax,
                                     const double* __restrict__ field, uint8_t* green, uint8_t* dep, double* tdep,
                                     double* wait, double* t_axis, Real* J, size_t LV, size_t LC, int* flags) {
    const int b = blockIdx.y;
    const int s = s_arr[b], h = h_arr[b];
    const int nt = c.nt;
    const double t0 = c.dt * floor(t_start[b] / c.dt);
    double* tax = t_axis + (size_t)b * nt;
    const size_t lad = (size_t)b * (Hmax + 1) * nt;
    if (blockIdx.x == 0) {
        for (int i = threadIdx.x; i < (h + 1) * nt; i += blockDim.x) {
            const int k = i / nt, z = i - k * nt;
            const int node = s + k;
            const double tz = t0 + c.dt * (double)z;
            if (k == 0) tax[z] = tz;
            const int si = sig_of_node[node];
            const EcoSignalTiming* tm = si >= 0 ? timings + (size_t)b * n_sig + si : nullptr;
            ladder_entry(r.kinds[node], tm ? tm->cycle : 1.0, tm ? tm->offset : 0.0, tm ? &tm->win[0][0] : nullptr,
                         tm ? tm->nwin : 0, r.stop_dwell, tz, c.teleport, green + lad, dep + lad, tdep + lad,
                         wait + lad, i);
        }
        if (flags) {
            __syncthreads();
            ladder_flags(green + lad, dep + lad, wait + lad, nt, h, flags + (size_t)b * Hmax);
        }
    }
    const int ncell = c.nv * c.nx;
    const int total = ncell * nt;
    Real* Jh = J + (size_t)b * 2 * LV + (h & 1) * LV;
    Real* Jh1 = Jh + LC;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
        const int cell = i / nt;
        const int jx = cell - (cell / c.nx) * c.nx;
        const double base = (c.use_field && field) ? field[(size_t)(s + h) * ncell + cell] : 0.0;
        const Real val = terminal_value<Real>(base, c.soc_axis[jx], c.soc_target, c.soc_weight, c.j_inf);
        Jh[i] = val;
        if (i > 0) Jh1[i - 1] = val;
    }
    if (blockIdx.x == 0) {
        // pads of both buffers (the other buffer's are written here too: the
        // stage kernel never writes past the level)
        for (int q = 0; q < 2; ++q) {
            Real* L0 = J + (size_t)b * 2 * LV + q * LV;
            Real* L1 = L0 + LC;
            for (int i = total - 1 + threadIdx.x; i < total + 8; i += blockDim.x) {
                L1[i] = (Real)INFINITY;
                if (i >= total) L0[i] = (Real)INFINITY;
            }
        }
    }
}

}  // namespace eco
