#!/usr/bin/env python3
"""Benchmark: receding-horizon eco-driving DP on B200 (BASELINE.json metric).

Default workload at N=1 (BASELINE.json configs[2], SURVEY §8d C3 — the largest
single-GPU configuration, the north star's "finest named grid"): one
receding-horizon DP solve of the synthetic 700-node urban route with SPaT at
urban node s = 60, clock t = 30 s, fine grid 350 x 260 x 400 states (dt =
0.2 s) x 23 x 30 controls, H = 20, gamma = 0.5.  One *step* = one solve:
the J-independent transition geometry of the 20 spatial steps (the
reference's stage 1) + 20 Bellman stage sweeps (5.02e11 dense updates).

  value   dense Bellman updates/s, device time of the solves (CUDA events on
          the solver's stream around the device work of each call: inputs
          already in HBM, outputs left there), summed over the K steps;
  e2e     the same metric through the public API (solve_horizon -> a
          SolveResult with all 21 f64 J levels and 20 int32 policy levels on
          the host) with the host context in and the 9 GB of tables out,
          wall-clocked with a device synchronize on both sides.

`--impl reference`: the reference algorithm's CPU implementation (the pinned
C restatement in oracle/, kind "port", all host threads) on the SAME C3
solve: step i runs stage H-1-(i mod H) of the horizon, chained from the
terminal level, so K = 20 timed steps are exactly one full C3 solve.

N > 1 GPUs: independent replicas of the solve ("replicas only" for C3;
the slab-partitioned single grid is C5): value = sum over ranks / max time.

Other workloads (`--workload`):
  c2  BASELINE configs[1]: the closed-loop MPC over the urban route, default
      grid 35 x 26 x 40 x 23 x 30, H = 20, terminal field on; one step = fit +
      699 receding-horizon solves (13,790 stages).  Replicas for N > 1.
  c4  BASELINE configs[3]: 4096 independent urban scenarios (route seed i,
      bench_schedule(route_i, 20, 1, seed=i)[0]), C2 grid, H = 20, no terminal
      field; sharded over ranks in contiguous blocks (strong scaling, no
      inter-GPU communication).  One step = one batch solve of the shard.
  c5  BASELINE configs[4]: the C3 solve with its speed planes split into N
      slabs, one per GPU (strong scaling); after every stage the slabs are
      exchanged (--exchange p2p: NVLink stores from the stage kernel's
      epilogue + GPU flag barrier; nccl: grouped ncclBroadcast).
  n1  the north-star Target: the closed loop at the C3 grid (fit with the
      terminal field + the first --loop-steps receding-horizon solves).
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "Bellman state×control updates/sec; ms per receding-horizon DP solve"
UNIT = "updates/s"
FLOPS_PER_LIVE = 23          # 7 lerps x 3 + add + min per gathered candidate


def env_rank():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), \
        int(os.environ.get("LOCAL_RANK", "0"))


def measured_peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    return json.loads(p.read_text()) if p.exists() else {}


def fp32_peak_tflops(sm_count: int, sm_mhz: float) -> float:
    """CUDA-core FP32 peak: 128 FMA lanes/SM x 2 flops x SMs x clock."""
    return 2.0 * 128 * sm_count * sm_mhz * 1e6 / 1e12


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        sm, mx, reasons = [], None, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for name, flag in zip(names, parts[5:9]):
                if flag.lower() in ("active", "1", "yes"):
                    reasons.add(name)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------------ workload

def c2_inputs():
    from paper_2104_01284_b200 import GridSpec, PenaltyConfig, StateVector, load_fixture_route, make_vehicle
    vehicle = make_vehicle()
    route, spat = load_fixture_route("urban", seed=0)
    return vehicle, route, spat, GridSpec(), PenaltyConfig(), StateVector(v=0.0, soc=0.5, t=0.0)


def dense_updates(route, grids, horizon, stages_loop):
    n_u = grids.n_t_eng * grids.n_t_bsg
    field = (route.node_count - 1) * grids.n_v * grids.n_soc * n_u
    loop = stages_loop * grids.n_v * grids.n_soc * grids.n_t * n_u
    return field, loop


def run_ours(args, rank, world, local_rank):
    import torch
    from paper_2104_01284_b200 import EcoDrivingMPC, simulate_closed_loop
    from paper_2104_01284_b200.mpc import MpcSession

    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    backend = "b200-fp64" if args.precision == "fp64" else "b200"
    vehicle, route, spat, grids, pen, x0 = c2_inputs()
    kw = dict(gamma=0.5, grids=grids, penalty=pen, horizon=20, backend=backend)
    sess = MpcSession(vehicle, route, spat, **kw)

    def step():
        _, fst = sess.fit(want_field=False)
        rows, status, _, fin, rst = sess.run(x0)
        assert status == 0 and len(rows) == route.node_count - 1, (status, len(rows))
        return fst, rst, rows

    for _ in range(args.warmup):
        step()
    # one counting pass (outside the timed region): U_live of the whole loop
    _, lst = sess.fit(want_field=False)
    live = sess.run(x0, count_live=True, time_sweeps=False)[4]["live_updates"]

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sweep_ms, loop_ms, stages, fit_dense = 0.0, 0.0, 0, 0
    with ClockSampler(local_rank) as clk:
        barrier()
        e0.record(stream)
        for _ in range(args.steps):
            fst, rst, rows = step()
            sweep_ms += rst["dominant_ms"]
            loop_ms += rst["device_ms"]
            stages += rst["stages"]
            fit_dense += fst["dense_updates"]
        e1.record(stream)
        barrier()
    ms = e0.elapsed_time(e1)
    t_max = ms
    if dist is not None:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_max = float(t.item())
    field_u, loop_u = dense_updates(route, grids, 20, stages // args.steps)
    per_step = field_u + loop_u
    value = per_step * args.steps * world / (t_max / 1e3)
    fuel = float(rows["fuel_inc_g"].sum())
    t_end = float(rows["t"][-1] + rows["wait_s"][-1] + rows["dt_move_s"][-1])

    # ------------------------------------------------ e2e through the public API
    def api_step():
        mpc = EcoDrivingMPC(vehicle, **kw).fit(route, spat)
        traj = simulate_closed_loop(route, spat, mpc, x0)
        assert traj.completed
        return mpc, traj

    api_step()
    barrier()
    a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a0.record(stream)
    for _ in range(args.steps):
        mpc, traj = api_step()
    a1.record(stream)
    barrier()
    e2e_ms = a0.elapsed_time(a1)
    if dist is not None:
        t = torch.tensor([e2e_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    h2d = mpc.upload_bytes_ + 3 * 8          # route / SPaT arrays re-sent by every fit + x0
    d2h = traj.n_steps * (120 + 8) + 3 * 8 + mpc.terminal_field_.values.nbytes + 4 * 3   # rows + step clocks

    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return None
    peaks = measured_peaks()
    props = torch.cuda.get_device_properties(local_rank)
    sm_max = float(peaks.get("sm_max_mhz", 1965.0))
    peak = fp32_peak_tflops(props.multi_processor_count, sm_max)
    if args.precision == "fp64":
        peak /= 2.0     # B200: FP64 at half the FP32 rate
    sweep_avg_s = sweep_ms / args.steps / 1e3
    achieved = FLOPS_PER_LIVE * live / sweep_avg_s / 1e12
    traffic, tsrc = measured_traffic(f"c2_{args.precision}")
    launches_per_step = rst["kernel_launches"] + fst["kernel_launches"]
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t_max / args.steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32" if args.precision == "fp32" else "f64",
        "data": "synthetic (reference fixture generators: urban route seed 0, synthetic 48V P0 vehicle)",
        "config": {"workload": "C2: closed-loop MPC, urban 700-node route with SPaT, default grid 35x26x40 "
                               "states x 23x30 controls, H=20, terminal field on (fit + 699 solves per step)",
                   "parallelism": f"replicas x{world}" if world > 1 else "single GPU",
                   "l2": "working set (route geometry ~2.6 GB) exceeds L2; no flush between steps",
                   "precision": args.precision},
        "ms_per_solve": loop_ms / args.steps / (route.node_count - 1),
        "sweep_ms_per_stage": sweep_ms / max(stages, 1),
        "dense_updates_per_step": per_step,
        "live_updates_per_step": live,
        "closed_loop": {"fuel_g": fuel, "travel_time_s": t_end - x0.t, "steps": int(len(rows))},
        "gpu_launches": int(launches_per_step * args.steps),
        "e2e": {"value": per_step * args.steps * world / (e2e_ms / 1e3), "unit": UNIT,
                "ms_per_step": e2e_ms / args.steps, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)},
        "roofline": {"bound": "fp32", "kernel": "bellman_stage_kernel", "achieved": achieved, "peak": peak,
                     "unit": "TFLOP/s", "frac": achieved / peak, "traffic": traffic, "traffic_source": tsrc,
                     "peak_source": f"CUDA-core FP32 = 2 x 128 x {props.multi_processor_count} SMs x "
                                    f"{sm_max:.0f} MHz (sm_max_mhz of MEASURED_PEAKS.json)"
                                    + (" / 2 for FP64" if args.precision == "fp64" else ""),
                     "algorithmic": f"{FLOPS_PER_LIVE} flop x {live} live gathers per step / summed sweep time"},
        "clocks": clk.summary(),
    }
    if not args.no_cpu_baseline and world == 1:      # the CPU sample runs at N = 1 only
        out["cpu_baseline"] = cpu_baseline(args.cpu_seconds)
    if dist is not None:
        dist.destroy_process_group()
    return out


# ------------------------------------------------------------ CPU reference

def cpu_sample(max_steps: int):
    """Oracle (pinned C restatement of the reference, all host threads) on the
    C2 workload: terminal field + the first max_steps receding-horizon steps."""
    from oracle import oracle as O
    vehicle, route, spat, grids, pen, x0 = c2_inputs()
    threads = O.threads_available()
    t0 = time.perf_counter()
    fld = O.field_build(vehicle, route, spat, grids, pen, 0.5)
    t1 = time.perf_counter()
    r = O.mpc_run(vehicle, route, spat, grids, pen, 0.5, 20, (x0.v, x0.soc, x0.t), fld, parallel=True,
                  threads=threads, max_steps=max_steps)
    t2 = time.perf_counter()
    stages = int(r["rows"]["horizon"].sum())
    field_u, loop_u = dense_updates(route, grids, 20, stages)
    return dict(updates=field_u + loop_u, seconds=t2 - t0, fit_s=t1 - t0, loop_s=t2 - t1,
                steps=len(r["rows"]), threads=threads)


def cpu_baseline(budget_s: float) -> dict:
    probe = cpu_sample(5)
    per_step = max(probe["loop_s"] / 5, 1e-3)
    m = int(min(699, max(5, (budget_s - probe["fit_s"]) / per_step)))
    s = cpu_sample(m)
    return {"value": s["updates"] / s["seconds"], "unit": UNIT, "cores": s["threads"], "kind": "port",
            "sample": f"C2 urban: terminal field ({699} (v,soc) sweeps) + first {s['steps']} MPC steps, "
                      f"oracle/eco_oracle.c two-stage sweep, {s['threads']} OpenMP threads",
            "seconds": s["seconds"], "ms_per_solve": s["loop_s"] * 1e3 / s["steps"]}


def run_reference(args, rank, world):
    if rank != 0:
        return None
    if args.workload == "c3":
        return run_reference_c3(args, world)
    if args.workload in ("c4", "c5"):
        return run_reference_other(args, world)
    budget = args.cpu_seconds
    probe = cpu_sample(3)
    per_step = max(probe["loop_s"] / 3, 1e-3)
    m = int(min(699, max(3, (budget - probe["fit_s"]) / per_step)))
    for _ in range(args.warmup):
        cpu_sample(min(m, 3))
    times, ups, last = [], [], None
    for _ in range(args.steps):
        last = cpu_sample(m)
        times.append(last["seconds"])
        ups.append(last["updates"])
    value = sum(ups) / sum(times)
    return {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * sum(times) / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
        "config": {"workload": "C2: closed-loop MPC, urban route, default grid, H=20 (bounded sample)"},
        "ms_per_solve": 1e3 * last["loop_s"] / last["steps"],
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": last["threads"], "kind": "port",
                         "sample": f"terminal field + first {last['steps']} MPC steps per step "
                                   f"(oracle/eco_oracle.c, the pinned restatement of the reference kernels)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


# ------------------------------------------------------------ C4 / C3

def _dist_init(world, local_rank):
    import torch
    torch.cuda.set_device(local_rank)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        return dist
    return None


def _max_over_ranks(dist, ms):
    if dist is None:
        return ms
    import torch
    t = torch.tensor([ms], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _roofline(args, local_rank, live, sweep_s, kernel, traffic=None, traffic_src=None, algorithmic_bytes=None):
    import torch
    peaks = measured_peaks()
    props = torch.cuda.get_device_properties(local_rank)
    sm_max = float(peaks.get("sm_max_mhz", 1965.0))
    peak = fp32_peak_tflops(props.multi_processor_count, sm_max)
    if args.precision == "fp64":
        peak /= 2.0
    achieved = FLOPS_PER_LIVE * live / sweep_s / 1e12
    out = {"bound": "fp32", "kernel": kernel, "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
           "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src,
           "peak_source": f"CUDA-core FP32 = 2 x 128 x {props.multi_processor_count} SMs x {sm_max:.0f} MHz"
                          + (" / 2 for FP64" if args.precision == "fp64" else "")
                          + " (FP32 is not in MEASURED_PEAKS.json; its sm_max_mhz is)",
           "algorithmic": f"{FLOPS_PER_LIVE} flop x {live} live gathers / summed sweep time (all stage launches "
                          f"of a solve)"}
    if algorithmic_bytes:
        out["algorithmic_bytes_per_launch"] = int(algorithmic_bytes)
    return out


def c4_inputs(n):
    from paper_2104_01284_b200 import GridSpec, PenaltyConfig, make_vehicle
    from paper_2104_01284_b200 import _abi
    from paper_2104_01284_b200.fixtures import bench_schedule, make_route_urban
    from paper_2104_01284_b200.route import load_route
    routes = [load_route(make_route_urban(seed=i)) for i in range(n)]
    sched = [bench_schedule(r, 20, 1, seed=i)[0] for i, (r, _) in enumerate(routes)]
    tim = _abi.signal_timings(routes[0][0], [sp for _, sp in routes])
    return make_vehicle(), routes, sched, tim, GridSpec(), PenaltyConfig()


def run_c4(args, rank, world, local_rank):
    import torch
    from paper_2104_01284_b200.batch import BatchSolver, shard
    dist = _dist_init(world, local_rank)
    backend = "b200-fp64" if args.precision == "fp64" else "b200"
    vehicle, routes, sched, tim, grids, pen = c4_inputs(args.scenarios)
    mine = shard(len(sched), rank, world)
    my_sched = [sched[i] for i in mine]
    my_spats = [routes[i][1] for i in mine]
    my_tim = tim[mine.start:mine.stop]
    bs = BatchSolver(vehicle, routes[0][0], grids=grids, penalty=pen, gamma=0.5, horizon=20, backend=backend)
    fit = bs.solve(my_spats, my_sched, return_tables=False, timings=my_tim).stats     # geometry build
    for _ in range(args.warmup):
        bs.solve(my_spats, my_sched, return_tables=False, timings=my_tim)
    live = bs.solve(my_spats, my_sched, return_tables=False, count_live=True, timings=my_tim).stats["live_updates"]
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    sweep_ms, dense, launches = 0.0, 0, 0
    with ClockSampler(local_rank) as clk:
        barrier()
        e0.record(stream)
        for _ in range(args.steps):
            st = bs.solve(my_spats, my_sched, return_tables=False, timings=my_tim).stats
            sweep_ms += st["dominant_ms"]
            dense += st["dense_updates"]
            launches += st["kernel_launches"]
        e1.record(stream)
        barrier()
    t_max = _max_over_ranks(dist, e0.elapsed_time(e1))
    total_dense = dense * world if dist is None else None
    if dist is not None:
        t = torch.tensor([float(dense)], device="cuda", dtype=torch.float64)
        dist.all_reduce(t)
        total_dense = float(t.item())
    # e2e: public API, host timings in, J0 / P0 of every scenario out
    bs.solve(my_spats, my_sched, timings=my_tim)
    barrier()
    a0 = time.perf_counter()
    for _ in range(args.steps):
        res = bs.solve(my_spats, my_sched)
    barrier()
    e2e_ms = _max_over_ranks(dist, (time.perf_counter() - a0) * 1e3)
    bs.close()
    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return None
    out = {
        "metric": METRIC, "value": total_dense / (t_max / 1e3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t_max / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32" if args.precision == "fp32" else "f64",
        "data": "synthetic (reference fixture generators: urban route seeds 0..N-1, bench_schedule per seed)",
        "config": {"workload": f"C4: batch of {args.scenarios} independent urban scenarios (own SPaT phasing, "
                               "start node and clock each), default grid 35x26x40 x 23x30, H=20, terminal_field=None",
                   "parallelism": f"scenario shards x{world} (no inter-GPU communication)",
                   "l2": "per-step working set (2.4 GB of levels + 2 GB geometry) exceeds L2; no flush",
                   "precision": args.precision},
        "ms_per_solve": t_max / args.steps / (args.scenarios / world),
        "geometry_ms": fit["device_ms"] - fit["dominant_ms"],
        "geometry": "the route geometry (one plan per spatial step, shared by every scenario) is built once per "
                    "BatchSolver, before the timed region, and excluded from value and e2e; geometry_ms is its "
                    "device time",
        "dense_updates_per_step": total_dense / args.steps, "live_updates_per_step_rank0": live,
        "gpu_launches": int(launches),
        "e2e": {"value": total_dense / (e2e_ms / 1e3), "unit": UNIT, "ms_per_step": e2e_ms / args.steps,
                "h2d_bytes_per_step": int(res.stats["h2d_bytes"]), "d2h_bytes_per_step": int(res.stats["d2h_bytes"])},
        "roofline": _roofline(args, local_rank, live, sweep_ms / args.steps / 1e3, "bellman_batch_kernel",
                              *measured_traffic(f"c4_{args.precision}")),
        "clocks": clk.summary(),
    }
    if not args.no_cpu_baseline and world == 1:
        out["cpu_baseline"] = c4_cpu_baseline(args.cpu_seconds)
    if dist is not None:
        dist.destroy_process_group()
    return out


def c4_cpu_sample(n_solves, threads=0):
    from oracle import oracle as O
    from paper_2104_01284_b200 import build_context
    vehicle, routes, sched, _, grids, pen = c4_inputs(n_solves)
    ctxs = [build_context(vehicle, r, sp, s, t, grids=grids, penalty=pen, gamma=0.5, horizon=20)
            for (r, sp), (s, t) in zip(routes, sched)]
    threads = threads or O.threads_available()
    t0 = time.perf_counter()
    for c in ctxs:
        O.solve_context(c, parallel=True, threads=threads)
    sec = time.perf_counter() - t0
    ups = sum(c.horizon for c in ctxs) * grids.n_v * grids.n_soc * grids.n_t * grids.n_t_eng * grids.n_t_bsg
    return dict(updates=ups, seconds=sec, solves=n_solves, threads=threads)


def c4_cpu_baseline(budget_s):
    probe = c4_cpu_sample(2)
    n = int(max(2, min(4096, budget_s / max(probe["seconds"] / 2, 1e-3))))
    s = c4_cpu_sample(n)
    return {"value": s["updates"] / s["seconds"], "unit": UNIT, "cores": s["threads"], "kind": "port",
            "sample": f"first {n} of the C4 scenarios solved one after another (oracle/eco_oracle.c two-stage "
                      f"sweep, {s['threads']} OpenMP threads)", "seconds": s["seconds"],
            "ms_per_solve": 1e3 * s["seconds"] / n}


C3_WORKLOAD = ("C3: one receding-horizon DP solve, urban 700-node route with SPaT, node s=60, t=30 s, fine grid "
               "350x260x400 states (dt=0.2 s) x 23x30 controls, H=20, gamma=0.5 (5.02e11 dense updates per solve)")
C3_CONFIG = {"workload": C3_WORKLOAD,
             "l2": "each level (145.6 MB f32 / 291 MB f64) exceeds the 126 MB L2: inputs larger than L2, no flush"}


def c3_context(H=20):
    from paper_2104_01284_b200 import (GridSpec, PenaltyConfig, build_context, load_fixture_route, make_vehicle)
    route, spat = load_fixture_route("urban", seed=0)
    grids = GridSpec(n_v=350, n_soc=260, n_t=400, dt=0.2)
    return build_context(make_vehicle(), route, spat, 60, 30.0, grids=grids, penalty=PenaltyConfig(), gamma=0.5,
                         horizon=H)


def so_digest() -> str:
    """Identity of the library build: the kernel sources + header + nvcc flags
    (the .so bytes themselves embed nvcc's per-run temp-file names)."""
    import hashlib
    import __graft_entry__ as ge
    h = hashlib.sha256(" ".join(ge.NVCC_FLAGS).encode())
    for f in sorted(ge.CSRC.glob("*.cu*")) + [ROOT / "include" / "eco_b200.h"]:
        h.update(f.name.encode())
        h.update(f.read_bytes())
    return h.hexdigest()[:16]


def measured_traffic(key: str):
    """DRAM bytes per launch of the dominant kernel from the committed ncu
    capture of THIS build (profiles/traffic.json records the library digest
    it was taken on); None when the capture belongs to another build."""
    tf = ROOT / "profiles" / "traffic.json"
    if not tf.exists():
        return None, "no capture committed"
    d = json.loads(tf.read_text())
    ent = d.get(key)
    if not ent:
        return None, f"no capture for {key}"
    if ent.get("so_digest") != so_digest():
        return None, f"capture {ent.get('file')} was taken on another build ({ent.get('so_digest')})"
    return ent["dram_bytes"], ent.get("file")


def run_c3(args, rank, world, local_rank):
    import torch
    from paper_2104_01284_b200 import solve_horizon
    from paper_2104_01284_b200.dp import solve_stacks
    dist = _dist_init(world, local_rank)
    backend = "b200-fp64" if args.precision == "fp64" else "b200"
    ctx = c3_context()
    for _ in range(args.warmup):
        solve_stacks(ctx, backend)
    live = solve_stacks(ctx, backend, count_live=True)[2]["live_updates"]

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    dev_ms, sweep_ms, dense, launches = 0.0, 0.0, 0, 0
    with ClockSampler(local_rank) as clk:
        barrier()
        w0 = time.perf_counter()
        for _ in range(args.steps):
            J, P, st = solve_stacks(ctx, backend)
            del J, P
            dev_ms += st["device_ms"]
            sweep_ms += st["dominant_ms"]
            dense += st["dense_updates"]
            launches += st["kernel_launches"]
        barrier()
        wall_ms = (time.perf_counter() - w0) * 1e3
    t_max = _max_over_ranks(dist, dev_ms)
    sweep_max = _max_over_ranks(dist, sweep_ms)
    # e2e: the public API, host context in, SolveResult (all levels) out
    res = solve_horizon(ctx, backend=backend)
    del res
    barrier()
    a0 = time.perf_counter()
    for _ in range(args.steps):
        res = solve_horizon(ctx, backend=backend)
        del res           # the previous result's pinned blocks go back to the pool
    barrier()
    e2e_ms = _max_over_ranks(dist, (time.perf_counter() - a0) * 1e3)
    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return None
    g = ctx.grids
    ns = g.n_v * g.n_soc * g.n_t
    traffic, tsrc = measured_traffic(f"c3_{args.precision}")
    out = {
        "metric": METRIC, "value": dense * world / (t_max / 1e3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t_max / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32" if args.precision == "fp32" else "f64",
        "data": "synthetic (reference fixture generators: urban route seed 0, synthetic 48V P0 vehicle)",
        "config": dict(C3_CONFIG),
        "parallelism": f"replicas x{world}" if world > 1 else "single GPU", "precision": args.precision,
        "timing": "value: CUDA events on the solver's stream around each solve's device work (geometry of the 20 "
                  "steps + 20 stage sweeps + output conversion), summed over the K steps; wall clock of the same "
                  "K steps with sync on both sides in wall_ms (includes the 291 MB terminal H2D per call)",
        "wall_ms": wall_ms,
        "ms_per_solve": t_max / args.steps, "sweep_ms_per_solve": sweep_max / args.steps,
        "dense_updates_per_step": dense / args.steps, "live_updates_per_step": live,
        "gpu_launches": int(launches),
        "e2e": {"value": dense * world / (e2e_ms / 1e3), "unit": UNIT, "ms_per_step": e2e_ms / args.steps,
                "h2d_bytes_per_step": int(ns * 8 + 20 * (g.n_v * 8 + g.n_t * (1 + 1 + 8 + 8))),
                # fp32: each J level crosses PCIe as f32 and is widened to
                # the f64 table by host threads; fp64: f64 levels
                "d2h_bytes_per_step": int(21 * ns * (4 if args.precision == "fp32" else 8) + 20 * ns * 4),
                "api": "paper_2104_01284_b200.solve_horizon(ctx, backend) -> SolveResult with all 21 f64 J and "
                       "20 int32 P levels on the host (9.0 GB; pinned output pool)"},
        "roofline": _roofline(args, local_rank, live, sweep_max / args.steps / 1e3, "bellman_wide2_kernel",
                              traffic, tsrc, algorithmic_bytes=ns * 4 + 3 * ns * 4),
        "clocks": clk.summary(),
    }
    if not args.no_cpu_baseline and world == 1:
        out["cpu_baseline"] = c3_cpu_baseline(args.cpu_seconds)
    if dist is not None:
        dist.destroy_process_group()
    return out


def c3_stage_chain(ctx, n_steps, threads, J=None, k=None):
    """Oracle stages of the C3 solve, chained: stage H-1 from the terminal,
    then H-2 from its output, ... (restarting at the terminal after stage 0).
    Returns (per-stage seconds, per-stage dense updates, state)."""
    from oracle import oracle as O
    g = ctx.grids
    ups = g.n_v * g.n_soc * g.n_t * g.n_t_eng * g.n_t_bsg
    H = ctx.horizon
    times = []
    if J is None:
        J, k = np.asarray(ctx.terminal, dtype=np.float64), H - 1
    for _ in range(n_steps):
        t0 = time.perf_counter()
        Jk, _, _ = O.sweep(ctx, k, J, parallel=True, threads=threads)
        times.append(time.perf_counter() - t0)
        J, k = Jk, k - 1
        if k < 0:
            J, k = np.asarray(ctx.terminal, dtype=np.float64), H - 1
    return times, [ups] * n_steps, (J, k)


def c3_cpu_baseline(budget_s):
    from oracle import oracle as O
    ctx = c3_context()
    threads = O.threads_available()
    t1, _, st = c3_stage_chain(ctx, 1, threads)
    n = int(max(1, min(ctx.horizon - 1, budget_s / max(t1[0], 1e-3))))
    times, ups, _ = c3_stage_chain(ctx, n, threads, *st)
    times = t1 + times
    ups = [ups[0]] * len(times)
    return {"value": sum(ups) / sum(times), "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"the first {len(times)} of the 20 stages of the same C3 solve, chained from the terminal "
                      f"level (oracle/eco_oracle.c two-stage sweep, {threads} OpenMP threads)",
            "seconds": sum(times), "ms_per_solve_est": 1e3 * sum(times) / len(times) * ctx.horizon}


def run_reference_c3(args, world):
    """--impl reference for the default C3 line: the oracle port on the same
    solve, one stage per step, chained (K = 20 steps = the whole solve)."""
    from oracle import oracle as O
    ctx = c3_context()
    threads = O.threads_available()
    _, _, st = c3_stage_chain(ctx, args.warmup, threads)        # warm-up: the first W stages
    times, ups, _ = c3_stage_chain(ctx, args.steps, threads)    # timed: restart at the terminal
    value = sum(ups) / sum(times)
    H = ctx.horizon
    return {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * sum(times) / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (reference fixture generators: "
        "urban route seed 0, synthetic 48V P0 vehicle)", "impl": "reference", "config": dict(C3_CONFIG),
        "ms_per_solve": 1e3 * sum(times) / len(times) * H,
        "stages_timed": len(times),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"the C3 solve itself: step i = stage {H - 1}-(i mod {H}) chained from the "
                                   f"terminal level, so the {args.steps} timed steps cover "
                                   f"{args.steps / H:g} full H={H} solve(s) (oracle/eco_oracle.c, the pinned C "
                                   f"restatement of the reference's two-stage numba sweep, {threads} OpenMP threads)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def run_reference_other(args, world):
    """--impl reference for C4 / C3: the oracle on a bounded sample."""
    from oracle import oracle as O
    times, ups, sample = [], [], ""
    if args.workload == "c4":
        probe = c4_cpu_sample(2)
        n = int(max(2, min(4096, args.cpu_seconds / max(probe["seconds"] / 2, 1e-3))))
        for _ in range(args.warmup):
            c4_cpu_sample(2)
        for _ in range(args.steps):
            s = c4_cpu_sample(n)
            times.append(s["seconds"])
            ups.append(s["updates"])
        sample = f"first {n} C4 scenarios per step, solved one after another"
        workload = f"C4: batch of {args.scenarios} urban scenarios, default grid, H=20 (bounded sample)"
    else:
        ctx = c3_context(H=1)
        ns = ctx.grids.n_v * ctx.grids.n_soc * ctx.grids.n_t
        for _ in range(args.steps):
            t0 = time.perf_counter()
            O.solve_context(ctx, parallel=True)
            times.append(time.perf_counter() - t0)
            ups.append(ns * ctx.grids.n_t_eng * ctx.grids.n_t_bsg)
        sample = "one C3 Bellman stage per step"
        workload = "C3: fine grid 350x260x400 x 23x30, urban s=60 t=30 (bounded sample)"
    value = sum(ups) / sum(times)
    threads = O.threads_available()
    return {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * sum(times) / args.steps, "higher_is_better": True,
        "scaling": "strong" if args.workload == "c4" else "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "impl": "reference", "config": {"workload": workload},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": sample + f" (oracle/eco_oracle.c two-stage sweep, {threads} OpenMP threads)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def run_c5(args, rank, world, local_rank):
    import torch
    from paper_2104_01284_b200.slab import SlabSolver
    dist = _dist_init(world, local_rank)
    backend = "b200-fp64" if args.precision == "fp64" else "b200"
    ctx = c3_context()
    g = ctx.grids
    ss = SlabSolver(g.n_v, g.n_soc, g.n_t, ctx.horizon, backend=backend, exchange=args.exchange, rank=rank,
                    world=world)
    for _ in range(args.warmup):
        ss.solve(ctx, return_P=False)
    live = ss.solve(ctx, return_P=False, count_live=True).stats["live_updates"]

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    dev_ms, sweep_ms, launches = 0.0, 0.0, 0
    with ClockSampler(local_rank) as clk:
        barrier()
        for _ in range(args.steps):
            st = ss.solve(ctx, return_P=False).stats
            dev_ms += st["device_ms"]
            sweep_ms += st["dominant_ms"]
            launches += st["kernel_launches"]
        barrier()
    t_max = _max_over_ranks(dist, dev_ms)
    sweep_max = _max_over_ranks(dist, sweep_ms)
    live_all = live
    if dist is not None:
        t = torch.tensor([float(live)], device="cuda", dtype=torch.float64)
        dist.all_reduce(t)
        live_all = float(t.item())
    # e2e: the public slab API with host context in, this rank's policy slab out
    barrier()
    a0 = time.perf_counter()
    for _ in range(args.steps):
        res = ss.solve(ctx)
    barrier()
    e2e_ms = _max_over_ranks(dist, (time.perf_counter() - a0) * 1e3)
    ss.close()
    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return None
    ns = g.n_v * g.n_soc * g.n_t
    dense = ns * g.n_t_eng * g.n_t_bsg * ctx.horizon          # whole grid, all ranks together
    out = {
        "metric": METRIC, "value": dense * args.steps / (t_max / 1e3), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_max / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32" if args.precision == "fp32" else "f64",
        "data": "synthetic (urban route seed 0)",
        "config": {"workload": "C5: the C3 solve (350x260x400 x 23x30, H=20) with its speed planes split into "
                               f"{world} slab(s) (make_partition), per-stage exchange of the level",
                   "parallelism": f"v-slabs x{world}, exchange={args.exchange}", "precision": args.precision,
                   "l2": "levels of 291 MB exceed L2; no flush"},
        "ms_per_solve": t_max / args.steps, "sweep_ms_per_solve": sweep_max / args.steps,
        "live_updates_per_step": live_all, "gpu_launches": int(launches),
        "e2e": {"value": dense * args.steps / (e2e_ms / 1e3), "unit": UNIT, "ms_per_step": e2e_ms / args.steps,
                "h2d_bytes_per_step": int(ns * 8), "d2h_bytes_per_step": int(res.P.nbytes)},
        "roofline": _roofline(args, local_rank, live_all / world, sweep_max / args.steps / 1e3,
                              "bellman_wide2_kernel", *measured_traffic(f"c5_{args.precision}")),
        "clocks": clk.summary(),
    }
    if dist is not None:
        dist.destroy_process_group()
    return out



def run_n1(args, rank, world, local_rank):
    """North-star Target: the receding-horizon closed loop at the C3 grid.
    EcoDrivingMPC.fit (chunked terminal field over the 700-node route) once,
    then each step = the first --loop-steps nodes of the closed loop from
    x0 = (0, 0.5, 0): per node a full H=20 C3 solve (ring of plan slots), the
    exact-state decision and the plant step, all on the device."""
    import torch
    from paper_2104_01284_b200 import GridSpec, PenaltyConfig, StateVector, load_fixture_route, make_vehicle
    from paper_2104_01284_b200.mpc import MpcSession
    dist = _dist_init(world, local_rank)
    backend = "b200-fp64" if args.precision == "fp64" else "b200"
    route, spat = load_fixture_route("urban", seed=0)
    grids = GridSpec(n_v=350, n_soc=260, n_t=400, dt=0.2)
    sess = MpcSession(make_vehicle(), route, spat, gamma=0.5, grids=grids, penalty=PenaltyConfig(), horizon=20,
                      backend=backend)
    _, fst = sess.fit(want_field=False)
    x0 = StateVector(0.0, 0.5, 0.0)
    M = args.loop_steps
    for _ in range(args.warmup):
        sess.run(x0, 0, M)
    live = sess.run(x0, 0, M, count_live=True)[4]["live_updates"]

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    dev_ms, sweep_ms, dense, launches = 0.0, 0.0, 0, 0
    with ClockSampler(local_rank) as clk:
        barrier()
        for _ in range(args.steps):
            rows, status, _, fin, st = sess.run(x0, 0, M)
            assert status == 0 and len(rows) == M
            dev_ms += st["device_ms"]
            sweep_ms += st["dominant_ms"]
            dense += st["dense_updates"]
            launches += st["kernel_launches"]
        barrier()
    t_max = _max_over_ranks(dist, dev_ms)
    sess.close()
    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return None
    out = {
        "metric": METRIC, "value": dense * world / (t_max / 1e3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t_max / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32" if args.precision == "fp32" else "f64",
        "data": "synthetic (reference fixture generators: urban route seed 0, synthetic 48V P0 vehicle)",
        "config": {"workload": f"N1 (north-star Target): closed-loop MPC on the urban route at the C3 grid "
                               f"350x260x400 (dt=0.2) x 23x30, H=20, terminal field on; one step = the first {M} "
                               f"nodes from x0=(0, 0.5, 0) (one full C3 solve + decision + plant step per node)",
                   "l2": "levels of 145.6 MB exceed L2; no flush"},
        "precision": args.precision,
        "fit_ms": fst["device_ms"], "fit_field_sweep_ms": fst["dominant_ms"],
        "ms_per_solve": t_max / args.steps / M, "sweep_ms_per_solve": sweep_ms / args.steps / M,
        "live_updates_per_step": live, "gpu_launches": int(launches),
        "final_state": [float(x) for x in fin],
        "roofline": _roofline(args, local_rank, live, sweep_ms / args.steps / 1e3, "bellman_wide2_kernel",
                              *measured_traffic(f"c3_{args.precision}")),
        "clocks": clk.summary(),
    }
    if dist is not None:
        dist.destroy_process_group()
    return out


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--precision", choices=["fp32", "fp64"], default="fp32")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="CPU baseline sample budget")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--workload", choices=["c2", "c3", "c4", "c5", "n1"], default="c3")
    ap.add_argument("--exchange", choices=["p2p", "nccl"], default="p2p", help="C5 slab exchange")
    ap.add_argument("--scenarios", type=int, default=4096, help="C4 batch size (all ranks together)")
    ap.add_argument("--loop-steps", type=int, default=20, help="n1: closed-loop nodes per step")
    args = ap.parse_args()
    rank, world, local_rank = env_rank()
    if world != args.gpus and world == 1:
        world = 1
    if args.impl == "reference":
        out = run_reference(args, rank, world)
    elif args.workload == "c4":
        out = run_c4(args, rank, world, local_rank)
    elif args.workload == "c3":
        out = run_c3(args, rank, world, local_rank)
    elif args.workload == "c5":
        out = run_c5(args, rank, world, local_rank)
    elif args.workload == "n1":
        out = run_n1(args, rank, world, local_rank)
    else:
        out = run_ours(args, rank, world, local_rank)
    if out is not None:
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
