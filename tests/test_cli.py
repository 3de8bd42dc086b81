"""GPU-backed command line: the reference's ``solve`` flags, defaults, config
layering, output files and exit codes (pkg/src/timemg/cli.py:232-290,
402-416), and the GPU ``bench`` scaling study (bench.py:77-137)."""

import csv
import json
import os

import numpy as np
import pytest

from paper_1409_5254_b200 import cli


def test_usage_errors_exit_2(tmp_path):
    assert cli.main([]) == 2
    assert cli.main(["solve", "--omega", "fast"]) == 2
    cfg = tmp_path / "c.json"
    cfg.write_text(json.dumps({"no_such_key": 1}))
    assert cli.main(["solve", "--config", str(cfg)]) == 2


def test_defaults_and_layering(tmp_path):
    p = cli.build_parser()
    cfg = tmp_path / "c.json"
    cfg.write_text(json.dumps({"steps": 128, "nu1": 1}))
    a = p.parse_args(["solve", "--config", str(cfg), "--nu1", "3"])
    m = cli.settings("solve", vars(a))
    assert m["steps"] == 128 and m["nu1"] == 3 and m["nu2"] == 2 and m["omega"] == "optimal"
    assert m["pt"] == 0 and m["eps"] == 1e-8 and m["max_iters"] == 250 and m["format"] == "csv"
    assert m["u0"] == 1.0 and m["f"] == "zero" and m["tau"] is None and m["levels"] == "max"
    b = cli.settings("bench", vars(p.parse_args(["bench", "--pt", "0,1", "--reps", "5"])))
    assert b["pt"] == [0, 1] and b["reps"] == 5 and b["mode"] == "strong"
    assert b["total_steps"] == 1 << 17 and b["steps_per_worker"] == 1 << 15


def test_bench_usage_errors():
    assert cli.main(["bench", "--workers", "1,3"]) == 2
    assert cli.main(["bench", "--workers", "2,1"]) == 2
    assert cli.main(["bench", "--reps", "2"]) == 2
    assert cli.main(["bench", "--workers", "1,2"]) == 2  # one process: no second GPU rank


@pytest.mark.gpu
def test_cli_solve_matches_oracle(tmp_path, oracle_mod):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_1409_5254_b200 as tmg
    out = tmp_path / "o"
    rc = cli.main(["solve", "--pt", "1", "--steps", "4096", "--f", "sin", "--f-param", "3",
                   "--nu1", "1", "--nu2", "1", "--out", str(out), "--compare-sequential"])
    assert rc == 0
    stats = json.load(open(out / "solve_stats.json"))
    basis = tmg.BasisSpec(1)
    tau = 1.0 / 4096
    hier = tmg.TimeHierarchy.build(basis, tau, 4096)
    rhs = tmg.rhs_moments(lambda t: np.sin(3.0 * t), basis, tau, 4096, u0=1.0)
    om = [tmg.optimal_omega(tmg.alpha(basis, l.tau)) for l in hier.levels]
    u_ref, norms, iters = oracle_mod.iterate(hier, om, rhs, tmg.random_initial_guess(hier, 42), 1, 1,
                                             1e-8, 250)
    assert stats["iterations"] == iters and stats["residual_norms"] == norms and stats["converged"]
    rows = list(csv.DictReader(open(out / "solve_solution.csv")))
    got = np.array([[float(r["c0"]), float(r["c1"])] for r in rows])
    assert np.array_equal(got, u_ref)  # csv round-trips float64 repr exactly
    res = list(csv.reader(open(out / "solve_residuals.csv")))
    assert res[0] == ["iteration", "residual_norm"] and len(res) == iters + 2


@pytest.mark.gpu
def test_cli_bench_gpu(tmp_path):
    out = tmp_path / "b"
    rc = cli.main(["bench", "--total-steps", "16384", "--pt", "0,1", "--reps", "3",
                   "--out", str(out), "--format", "json"])
    assert rc == 0
    rows = json.load(open(out / "bench_strong.json"))
    assert [r["p_t"] for r in rows] == [0, 1] and all(r["workers"] == 1 for r in rows)
    assert all(r["iterations"] > 0 and r["median_time"] > 0 and len(r["samples"]) == 3
               for r in rows)
