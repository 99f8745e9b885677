"""Command line (cli.py, mirroring the reference's ecodrive CLI): option and
config validation on CPU (exit code 1 for every configuration error, as
the reference's test_io_cli.py checks), the three subcommands on the GPU."""

import json

import pytest

from paper_2104_01284_b200.cli import EXIT_CONFIG, EXIT_OK, build_parser, load_config, main

SMALL_CFG = {"grid": {"n_v": 12, "n_soc": 8, "n_t": 40, "n_t_eng": 8, "n_t_bsg": 10}, "horizon_steps": 8}


@pytest.mark.parametrize("argv", [
    ["run", "--backend", "serial"],                 # a CPU backend name
    ["run", "--gamma", "1.5"],
    ["run", "--route", "/nonexistent/route.json"],
    ["run", "--controller", "baseline"],
    ["run", "--vehicle", "v.json"],
    ["run", "--horizon", "0"],
    ["bench", "--reps", "10"],
    ["bench", "--backends", "b200,parallel"],
    ["diff-backends", "--against", "serial"],
    ["frobnicate"],
    [],
])
def test_configuration_errors_exit_1(argv, tmp_path, capsys):
    assert main(argv + ["--out", str(tmp_path)] if argv and argv[0] != "frobnicate" else argv) == EXIT_CONFIG
    assert "error" in capsys.readouterr().err


def test_config_file_merge_and_checks(tmp_path):
    p = tmp_path / "cfg.json"
    p.write_text(json.dumps({"gamma": 0.3, "time_step_s": 1.0, "grid": {"n_t": 80}, "backend": "b200-fp64",
                             "soc_init": 0.6, "soc_weight": 900.0}))
    args = build_parser().parse_args(["run", "--config", str(p), "--horizon", "12"])
    cfg = load_config(args.config, args)
    assert (cfg.gamma, cfg.grid.dt, cfg.grid.n_t, cfg.backend, cfg.horizon) == (0.3, 1.0, 80, "b200-fp64", 12)
    assert cfg.soc_init == 0.6 and cfg.penalty.soc_weight == 900.0
    p.write_text(json.dumps({"time_step_s": 2.0, "horizon_time_s": 50.0}))
    assert main(["run", "--config", str(p)]) == EXIT_CONFIG
    p.write_text("{not json")
    assert main(["run", "--config", str(p)]) == EXIT_CONFIG
    assert main(["run", "--config", str(tmp_path / "missing.json")]) == EXIT_CONFIG


@pytest.mark.gpu
def test_cli_run_diff_bench(tmp_path, capsys):
    cfg = tmp_path / "small.json"
    cfg.write_text(json.dumps(SMALL_CFG))
    out = tmp_path / "out"
    base = ["--route", "short", "--seed", "2", "--config", str(cfg), "--out", str(out)]
    assert main(["run", "--backend", "b200-fp64"] + base) == EXIT_OK
    name = "short-1p2km"                           # the fixture route's name
    for f in (f"trajectory_mpc_{name}.csv", f"timing_mpc_{name}.csv", f"summary_{name}.json"):
        assert (out / f).is_file()
    summary = json.loads((out / f"summary_{name}.json").read_text())
    assert summary["runs"]["mpc"]["status"] == "ok" and summary["backend"] == "b200-fp64"
    assert main(["diff-backends", "--backend", "b200-fp64", "--against", "b200-fp64"] + base) == EXIT_OK
    assert "policy mismatches total: 0" in capsys.readouterr().out
    assert main(["bench", "--reps", "30", "--warmup", "2"] + base) == EXIT_OK
    txt = capsys.readouterr().out
    assert "b200-fp64" in txt and "speedup (b200 mean / b200-fp64 mean)" in txt
    assert (out / f"bench_{name}.csv").is_file() and (out / f"diff_backends_{name}.csv").is_file()
