"""Trajectory / summary files: byte-identical to the reference's writers
(io.py) on the golden short-route closed loop (rows from the reference run),
plus read-back round trips."""

import math

import numpy as np
import pytest
from conftest import GOLDEN, golden_npz

from paper_2104_01284_b200 import StateVector
from paper_2104_01284_b200.io import (TRAJECTORY_COLUMNS, comparison_summary, read_trajectory_csv, summarize,
                                      write_summary_json, write_timing_csv, write_trajectory_csv)
from paper_2104_01284_b200.mpc import ClosedLoopTrajectory, TrajectoryStep

FIELDS = ("s", "v", "soc", "t", "t_eng", "t_bsg", "brake_force", "gear", "wait_s", "dt_move_s", "fuel_inc_g",
          "accel", "cost_to_go", "fallback")


def golden_traj(backend="parallel"):
    g = golden_npz("loop_short_small.npz")
    steps = []
    for row in g["rows"]:
        d = {k: float(x) for k, x in zip(FIELDS, row)}     # Python floats, as the loop produces
        d["s"], d["gear"], d["fallback"] = int(d["s"]), int(d["gear"]), bool(d["fallback"])
        steps.append(TrajectoryStep(**d))
    v, soc, t = map(float, g["final"])
    return ClosedLoopTrajectory(route_name="short-1p2km", controller="mpc", backend=backend, delta_d=10.0,
                                x_start=StateVector(v=0.0, soc=0.5, t=0.0), steps=steps,
                                solver_wall_s=[1e-3] * len(steps), final_state=StateVector(v=v, soc=soc, t=t))


def test_trajectory_csv_byte_identical_to_reference(tmp_path):
    out = tmp_path / "traj.csv"
    write_trajectory_csv(out, golden_traj())
    assert out.read_bytes() == (GOLDEN / "loop_short_small_traj.csv").read_bytes()


def test_summary_json_byte_identical_to_reference(tmp_path):
    out = tmp_path / "summary.json"
    write_summary_json(out, summarize(golden_traj()))
    assert out.read_bytes() == (GOLDEN / "loop_short_small_summary.json").read_bytes()


def test_trajectory_round_trip(tmp_path):
    tr = golden_traj()
    out = tmp_path / "traj.csv"
    write_trajectory_csv(out, tr)
    f = read_trajectory_csv(out)
    assert len(f.steps) == len(tr.steps) and f.final["step"] == tr.steps[-1].s + 1
    for r, st in zip(f.steps, tr.steps):
        assert r["v_mps"] == st.v and r["cost_to_go"] == st.cost_to_go or math.isnan(st.cost_to_go)
        assert r["gear"] == st.gear and r["fallback"] == st.fallback
    assert f.fuel_g == pytest.approx(tr.fuel_g, rel=0, abs=1e-12)
    assert f.travel_time_s == tr.final_state.t - tr.steps[0].t
    assert f.soc_end == tr.final_state.soc


def test_bad_header_rejected(tmp_path):
    p = tmp_path / "bad.csv"
    p.write_text("a,b\n1,2\n")
    with pytest.raises(ValueError):
        read_trajectory_csv(p)


def test_timing_and_comparison(tmp_path):
    tr = golden_traj()
    p = tmp_path / "timing.csv"
    write_timing_csv(p, tr)
    lines = p.read_text().splitlines()
    assert lines[0] == "step,solver_wall_ms" and len(lines) == len(tr.steps) + 1
    a, b = summarize(tr), dict(summarize(tr))
    b["fuel_g"] *= 2.0
    c = comparison_summary(a, b)
    assert c["fuel_ratio"] == 0.5 and c["fuel_saving_pct"] == 50.0 and c["time_ratio"] == 1.0
    assert TRAJECTORY_COLUMNS[0] == "step" and len(TRAJECTORY_COLUMNS) == 14
