/*
 * eco_b200.h — C ABI of the B200 eco-driving DP solver.
 *
 * Plain C: POD structs, raw pointers and sizes, integer status codes, no
 * exceptions and no torch types.  Every entry point replaces one call site
 * of the reference package `ecodrive` (paths relative to
 * /root/reference/pkg/src/ecodrive/):
 *
 *   eco_bellman_step   <- backward_step           dp.py:365-404
 *                         (= _kernels.dp_sweep_serial _kernels.py:421-546,
 *                          = parallel_step           parallel.py:152-158;
 *                          tables != NULL is the use_tables / toy_mode path
 *                          of _kernels.py:476-493 and solve_toy dp.py:557-610)
 *   eco_solve_horizon  <- solve_horizon           dp.py:425-475
 *   eco_field_build    <- build_terminal_cost     mpc.py:96-158
 *                         (loop of _kernels.field_sweep _kernels.py:801-865)
 *   eco_mpc_run        <- EcoDrivingMPC.fit + simulate_closed_loop
 *                                                  mpc.py:379-391, 513-596
 *   eco_batch_*, eco_solve_batch
 *                      <- run_bench inner loop    bench.py:136-148
 *                         (many independent build_context + solve_horizon)
 *
 * Conventions (dp.py:383-384, _kernels.py:540-545): infeasible cost-to-go is
 * exactly j_inf, infeasible policy entries are -1, policy values are flat
 * action indices ite * n_tb + itb.  All host arrays are C-contiguous,
 * row-major (v, soc, t) with t fastest.  Outputs are written by the callee.
 *
 * Precision: ECO_FP64 computes the value path in IEEE double with unfused
 * arithmetic (bitwise equal to the reference); ECO_FP32 keeps the transition
 * geometry in double and the cost-to-go gather / argmin in float.
 */
#ifndef ECO_B200_H
#define ECO_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ECO_ABI_VERSION 6

#define ECO_MAX_GEARS 16
#define ECO_MAX_AXIS 32
#define ECO_MAX_MAP (ECO_MAX_AXIS * ECO_MAX_AXIS)
#define ECO_MAX_WINDOWS 8

/* status codes */
#define ECO_OK 0
#define ECO_ERR_ARG 1      /* invalid argument (sizes, null pointers) */
#define ECO_ERR_CUDA 2     /* CUDA runtime failure; see eco_last_error() */
#define ECO_ERR_NODEV 3    /* no CUDA device visible */

/* precision selector */
#define ECO_FP32 0
#define ECO_FP64 1
/* OR-ed into the precision argument of eco_bellman_step / eco_solve_horizon /
 * eco_solve_tables: ties go to the HIGHEST flat action index instead of the
 * lowest (perturb_ties / reverse_ties, dp.py:365-404, _kernels.py:630-632 and
 * 738-740: the negative control of the backend-diff harness; costs are
 * unchanged, tied policy entries flip). */
#define ECO_REVERSE_TIES 0x100

/* node kinds (route.py:29-31) */
#define ECO_NODE_PLAIN 0
#define ECO_NODE_SIGNAL 1
#define ECO_NODE_STOP 2

/* Packed plant: the fields of PlantPack (_kernels.py:31-53) with fixed-capacity
 * arrays.  shift_v holds n_gears - 1 entries; maps are row-major. */
typedef struct EcoPlant {
    double mass, c0, c1, c2, wheel_radius, final_drive;
    double idle_speed, belt_ratio;
    double r0, c_nom, soc_min, soc_max, p_bat_max;
    int32_t n_gears, n_eng, n_fuel_w, n_fuel_t;
    int32_t n_bsg, n_eff_w, n_eff_t, n_voc;
    double gear_ratios[ECO_MAX_GEARS];
    double gear_eff[ECO_MAX_GEARS];
    double shift_v[ECO_MAX_GEARS];
    double eng_w[ECO_MAX_AXIS], eng_tmin[ECO_MAX_AXIS], eng_tmax[ECO_MAX_AXIS];
    double fuel_w[ECO_MAX_AXIS], fuel_t[ECO_MAX_AXIS];
    double bsg_w[ECO_MAX_AXIS], bsg_tmin[ECO_MAX_AXIS], bsg_tmax[ECO_MAX_AXIS];
    double eff_w[ECO_MAX_AXIS], eff_t[ECO_MAX_AXIS];
    double voc_soc[ECO_MAX_AXIS], voc_v[ECO_MAX_AXIS];
    double fuel_vals[ECO_MAX_MAP];
    double eff_vals[ECO_MAX_MAP];
} EcoPlant;

/* Grid and per-solve scalars shared by every step (GridSpec dp.py:41-83,
 * SolveContext dp.py:191-214, PenaltyConfig dp.py:86-98). */
typedef struct EcoProblem {
    int32_t n_v, n_soc, n_t, n_te, n_tb;
    int32_t reserved;
    double delta_d, a_min, a_max;   /* route spacing and comfort box */
    double gamma, j_inf;
    double t0, dtg;                  /* time ladder t_z = t_axis[z], spacing */
    const double* te_axis;           /* n_te */
    const double* tb_axis;           /* n_tb */
    const double* soc_axis;          /* n_soc */
    const double* t_axis;            /* n_t */
} EcoProblem;

/* One spatial step m -> m+1 (StepPlan dp.py:173-188). */
typedef struct EcoStepPlan {
    int32_t node, src_kind, dest_kind, reserved;
    double grade, v0_dest, dv_dest;
    double cos_grade, sin_grade;  /* host libm cos/sin(grade): road_load K:134-142 */
    const double* v_src;      /* n_v source speed axis */
    const uint8_t* arr_green; /* n_t destination green mask */
    const uint8_t* dep_ok;    /* n_t source standstill departure allowed */
    const double* t_dep;      /* n_t */
    const double* wait;       /* n_t */
} EcoStepPlan;

/* Table-driven (v, u) transition quantities, shape (n_v, n_te, n_tb) each:
 * the s1* arguments of dp_sweep_serial (_kernels.py:424), used by toy
 * instances (dp.py:482-610). */
typedef struct EcoStage1Tables {
    const uint8_t* ok;
    const double* v2;
    const double* dt;
    const double* pbat;
    const double* c1;
    const int32_t* ivlo;
    const int32_t* ivhi;
    const double* wv;
    const int32_t* zoff;
    const double* wz;
} EcoStage1Tables;

/* Route with SPaT (Route route.py:102-184, SignalTiming route.py:34-86). */
typedef struct EcoRoute {
    int32_t node_count;
    int32_t reserved;
    double delta_d, accel_min, accel_max, stop_dwell;
    const double* v_min;      /* node_count */
    const double* v_max;      /* node_count */
    const double* grade;      /* node_count */
    const double* cos_grade;  /* node_count, host libm cos(grade) */
    const double* sin_grade;  /* node_count, host libm sin(grade) */
    const int8_t* kinds;      /* node_count, ECO_NODE_* */
    /* per node (meaningful where kinds == ECO_NODE_SIGNAL) */
    const double* sig_cycle;  /* node_count */
    const double* sig_offset; /* node_count */
    const int32_t* sig_nwin;  /* node_count */
    const double* sig_win;    /* node_count * ECO_MAX_WINDOWS * 2 ([start,end)) */
} EcoRoute;

/* Controller settings (EcoDrivingMPC.__init__ mpc.py:354-377). */
typedef struct EcoMpcConfig {
    int32_t n_v, n_soc, n_t, n_te, n_tb;
    int32_t horizon;
    int32_t teleport;             /* 1: red wait allowed (default) */
    int32_t use_terminal_field;   /* 1: offline field (default) */
    int32_t precision;            /* ECO_FP32 / ECO_FP64 */
    int32_t start_node;           /* closed loop starts at this node (0 = route start) */
    int32_t max_steps;            /* < 0: drive to the end of the route */
    int32_t reserved;
    double dt;                    /* ladder spacing */
    double gamma, soc_target, soc_weight, j_inf;
    const double* te_axis;        /* n_te */
    const double* tb_axis;        /* n_tb */
} EcoMpcConfig;

/* One closed-loop step (TrajectoryStep mpc.py:418-435). */
typedef struct EcoTrajRow {
    int32_t s, gear, fallback, horizon;
    double v, soc, t, t_eng, t_bsg, brake_force;
    double wait_s, dt_move_s, fuel_inc_g, accel, cost_to_go;
} EcoTrajRow;

/* Diagnostics returned by the solvers. */
typedef struct EcoStats {
    double device_ms;          /* CUDA-event time of the device work */
    double dominant_ms;        /* CUDA-event time of the Bellman sweeps only */
    int64_t dense_updates;     /* N_s * n_te * n_tb * stages */
    int64_t live_updates;      /* candidates that reached the value gather (counted when requested) */
    int64_t stages;            /* Bellman stages executed */
    int64_t kernel_launches;   /* kernels launched by this call */
} EcoStats;

/* closed-loop status codes */
#define ECO_RUN_OK 0
#define ECO_RUN_INFEASIBLE 1   /* no admissible action and max-brake impossible */
#define ECO_RUN_PLANT 2        /* plant step raised (zero mean velocity, power, rule) */

int32_t eco_abi_version(void);
const char* eco_last_error(void);
int32_t eco_device_count(void);

/* The stateless solvers (eco_bellman_step, eco_solve_horizon) keep their
 * device buffers in a grow-only workspace so repeated calls on one grid
 * allocate nothing (not thread-safe: one solving thread per process).
 * This frees it. */
int32_t eco_release_workspace(void);

/* Page-locked host buffers for solver outputs: J / P stacks written into
 * them arrive by direct DMA (no staging copy), and level by level while the
 * remaining stages still sweep.  Any output pointer may also be ordinary
 * pageable memory. */
int32_t eco_host_alloc(uint64_t bytes, void** out);
/* Checked builds (-DECO_CHECKED, paper_2104_01284_b200/_eco_b200_checked.so):
 * violations counted since the last reset -- gathers of J_{k+1} / of a tile's
 * shared-memory band outside their buffers, and stage outputs not written
 * exactly once (the single-writer rule).  Regular builds
 * report -1 for both. */
int32_t eco_debug_checks(int64_t* bounds_violations, int64_t* writer_violations, int32_t reset);
int32_t eco_host_free(void* p);

/* One backward Bellman step (backward_step, dp.py:365-404).  J_next, J_out
 * are (n_v, n_soc, n_t) f64, P_out int32.  tables may be NULL (plant path). */
int32_t eco_bellman_step(const EcoPlant* plant, const EcoProblem* prob,
                         const EcoStepPlan* plan, const EcoStage1Tables* tables,
                         const double* J_next, double* J_out, int32_t* P_out,
                         int32_t precision, int32_t count_live, EcoStats* stats);

/* Whole-horizon backward recursion (solve_horizon, dp.py:425-475).
 * plans[0..H-1]; terminal (n_v, n_soc, n_t); J_stack (H+1) levels with
 * index 0 = start node; P_stack H levels. */
int32_t eco_solve_horizon(const EcoPlant* plant, const EcoProblem* prob,
                          const EcoStepPlan* plans, int32_t H,
                          const double* terminal, double* J_stack,
                          int32_t* P_stack, int32_t precision,
                          int32_t count_live, EcoStats* stats);

/* Table-driven horizon solve (solve_toy, dp.py:557-610): tables[k] holds the
 * (n_v, n_te, n_tb) transition quantities of step k; battery power is read per
 * action (toy_mode of dp_stage2_sweep, _kernels.py:676-683). */
int32_t eco_solve_tables(const EcoPlant* plant, const EcoProblem* prob,
                         const EcoStepPlan* plans, const EcoStage1Tables* tables,
                         int32_t H, const double* terminal, double* J_stack,
                         int32_t* P_stack, int32_t precision);

/* Offline terminal field (build_terminal_cost, mpc.py:96-158):
 * field_out (node_count, n_v, n_soc) f64. */
int32_t eco_field_build(const EcoPlant* plant, const EcoRoute* route,
                        const EcoMpcConfig* cfg, double* field_out,
                        EcoStats* stats);

/* Closed loop (EcoDrivingMPC.fit + simulate_closed_loop, mpc.py:379-596) on
 * the device.  rows has room for node_count - 1 entries; *n_rows receives the
 * number of steps taken, *status an ECO_RUN_* code, final_state (v, soc, t).
 * field_in may hold a precomputed field (node_count, n_v, n_soc); when NULL
 * and cfg->use_terminal_field, the field is built on the device first.
 * field_out (nullable) receives the field used. */
int32_t eco_mpc_run(const EcoPlant* plant, const EcoRoute* route,
                    const EcoMpcConfig* cfg, const double* x_start,
                    const double* field_in, double* field_out,
                    EcoTrajRow* rows, int32_t* n_rows, int32_t* status,
                    int32_t* status_node, double* final_state, EcoStats* stats);

/* Sessions: a route-resident solver for serving many closed loops.
 * create  — upload plant / route, allocate all device buffers (no compute);
 * fit     — route-level transition geometry + terminal field
 *           (EcoDrivingMPC.fit, mpc.py:379-391); field_in != NULL uploads a
 *           precomputed field instead of building it; field_out optional;
 * run     — closed loop from start_node for max_steps nodes (< 0: to the end)
 *           (simulate_closed_loop, mpc.py:513-596); flags: ECO_RUN_COUNT_LIVE
 *           counts gathers (slower).  stats->dominant_ms is always the summed
 *           per-step solve clock (device timestamps, prepare entry -> decision
 *           entry); ECO_RUN_TIME_SWEEPS is accepted for compatibility. */
typedef struct EcoSession EcoSession;
#define ECO_RUN_COUNT_LIVE 1
#define ECO_RUN_TIME_SWEEPS 2
int32_t eco_session_create(const EcoPlant* plant, const EcoRoute* route,
                           const EcoMpcConfig* cfg, EcoSession** out);
/* new data for the session's route (same node count): speed limits,
 * grades, node kinds, signal programs; the next fit rebuilds geometry and
 * field from it (EcoDrivingMPC.fit(route, spat) mpc.py:379-391 on a new
 * route / SPaT of the same shape). */
int32_t eco_session_upload_route(EcoSession* sess, const EcoRoute* route);
int32_t eco_session_fit(EcoSession* sess, const double* field_in,
                        double* field_out, EcoStats* stats);
int32_t eco_session_run(EcoSession* sess, int32_t start_node, int32_t max_steps,
                        const double* x_start, EcoTrajRow* rows, int32_t* n_rows,
                        int32_t* status, int32_t* status_node,
                        double* final_state, int32_t flags, EcoStats* stats);
/* per-step solve clocks (ms, device timestamps: context in place -> decision
 * entry) of the last eco_session_run's first n steps (n <= the steps that
 * run took): ClosedLoopTrajectory.solver_wall_s (mpc.py:438-487), written by
 * write_timing_csv (io.py:115-124). */
int32_t eco_session_step_times(EcoSession* sess, double* solve_ms, int32_t n);
int32_t eco_session_destroy(EcoSession* sess);

/* Phase plan of one signal (SignalTiming route.py:50-86): green windows
 * [win[i][0], win[i][1]) within a cycle, shifted by offset. */
typedef struct EcoSignalTiming {
    double cycle, offset;
    int32_t nwin, reserved;
    double win[ECO_MAX_WINDOWS][2];
} EcoSignalTiming;

/* Batch of independent horizon solves sharing one route geometry (C4, the
 * inner loop of run_bench bench.py:136-148 over build_context dp.py:255-341 +
 * solve_horizon dp.py:425-475).  The route supplies the geometry (speed
 * limits, grades, node kinds); its signal arrays are ignored.  Scenario i
 * starts at node s[i] and clock t_start[i]; its signals are
 * timings[i * n_signal_nodes + j] for the j-th signal node of the route (in
 * node order).  The horizon is cfg->horizon clipped at the route end.
 * cfg->use_terminal_field selects the offline field (built once per batch
 * object) or zeros (terminal_field=None).  J0 (n_scen, n_v, n_soc, n_t) f64
 * and P0 (int32) receive each scenario's start-node level when non-NULL.
 * create/solve/destroy keep the route geometry resident across solves;
 * eco_solve_batch is the one-shot form.  flags: ECO_RUN_COUNT_LIVE. */
typedef struct EcoBatch EcoBatch;
int32_t eco_batch_create(const EcoPlant* plant, const EcoRoute* route,
                         const EcoMpcConfig* cfg, EcoBatch** out);
int32_t eco_batch_solve(EcoBatch* batch, int32_t n_scen,
                        const EcoSignalTiming* timings, const int32_t* s,
                        const double* t_start, double* J0, int32_t* P0,
                        int32_t flags, EcoStats* stats);
int32_t eco_batch_destroy(EcoBatch* batch);
int32_t eco_solve_batch(const EcoPlant* plant, const EcoRoute* route,
                        const EcoMpcConfig* cfg, int32_t n_scen,
                        const EcoSignalTiming* timings, const int32_t* s,
                        const double* t_start, double* J0, int32_t* P0,
                        EcoStats* stats);

/* Slab-partitioned horizon solve across GPUs (C5; the GPU form
 * of the reference's v-plane WorkPartition, parallel.py:59-106).  One process
 * per GPU; rank r of nranks computes the speed planes [bounds[r],
 * bounds[r + 1]) of every level (bounds: nranks + 1 plane edges, the host's
 * make_partition parallel.py:87-101) and after each stage the slabs are
 * exchanged so every rank holds the full level for the next stage:
 *   ECO_XCHG_P2P   the stage kernel stores its slab into every peer's replica
 *                  over NVLink (CUDA IPC) + a GPU-side flag barrier;
 *   ECO_XCHG_NCCL  grouped ncclBroadcast of each slab (the library baseline).
 * Protocol: create -> info (ECO_SLAB_INFO_BYTES per rank) -> all-gather the
 * infos on the host (any transport) -> connect(all infos, rank order) ->
 * solve (collective: every rank calls it with the same problem).  solve
 * writes the full J stack (H + 1 levels, NULL to skip) and this rank's
 * policy slab P_slab (H, hi - lo, n_soc, n_t) (NULL to skip). */
typedef struct EcoSlab EcoSlab;
#define ECO_XCHG_P2P 0
#define ECO_XCHG_NCCL 1
#define ECO_SLAB_INFO_BYTES 256
int32_t eco_slab_create(int32_t nranks, int32_t rank, int32_t exchange,
                        const int32_t* bounds, int32_t precision,
                        int32_t n_v, int32_t n_soc, int32_t n_t,
                        int32_t max_horizon, EcoSlab** out);
int32_t eco_slab_info(EcoSlab* slab, uint8_t* info);
int32_t eco_slab_connect(EcoSlab* slab, const uint8_t* all_info);
int32_t eco_slab_solve(EcoSlab* slab, const EcoPlant* plant,
                       const EcoProblem* prob, const EcoStepPlan* plans,
                       int32_t H, const double* terminal, double* J_stack,
                       int32_t* P_slab, int32_t count_live, EcoStats* stats);
int32_t eco_slab_destroy(EcoSlab* slab);
/* ECO_XCHG_P2P with several ranks on ONE GPU (tests): replace the GPU-side
 * stage barrier by a stream sync + barrier(user) on the host (e.g. a gloo
 * barrier), so no kernel waits on another process's kernels.  NULL restores
 * the GPU barrier. */
int32_t eco_slab_set_host_barrier(EcoSlab* slab, void (*barrier)(void*), void* user);
/* The slab decomposition of nranks ranks emulated on ONE GPU (tests of the
 * exchange where fewer GPUs than ranks are available): one launch per stage
 * covers every rank's tiles, each rank keeps its own replica of the levels,
 * filled through the same peer-store epilogue and local copy-1 rebuild as the
 * multi-GPU path.  J_stacks receives every rank's replica, (nranks, H + 1,
 * n_v, n_soc, n_t) f64; P_stack (nullable) the policy stack assembled from
 * the slabs.  nranks <= 8. */
int32_t eco_slab_emulate(int32_t nranks, const int32_t* bounds, int32_t precision, const EcoPlant* plant,
                         const EcoProblem* prob, const EcoStepPlan* plans, int32_t H, const double* terminal,
                         double* J_stacks, int32_t* P_stack, EcoStats* stats);

#ifdef __cplusplus
}
#endif
#endif /* ECO_B200_H */
