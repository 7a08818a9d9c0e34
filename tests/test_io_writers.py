"""Result writers, run-configuration reader and benchmark CSV of the reference (io.hpp:307-531),
exercised on CPU with oracle results (the writers are host-side and result-type agnostic)."""
import csv
import json

import numpy as np
import pytest

import paper_2301_03989_b200 as ps
from paper_2301_03989_b200 import io


@pytest.fixture(scope="module")
def result(oracle):
    base = ps.reference_state()
    states = ps.make_clone_batch(base, 3, 1e-5)
    period = ps.osculating_period(base, ps.MU_SUN)
    plan = ps.plan_segments(base, 0.0, 1.3 * period, ps.MU_SUN, "per_orbit", 16)
    cfg = ps.reference_force_config("two_body", n_nodes=16)
    return oracle.run_batch(states, cfg, plan, "grouped", 2)


def test_samples_csv(tmp_path, result):
    p = tmp_path / "samples.csv"
    io.write_samples_csv(p, result)
    rows = list(csv.reader(open(p)))
    assert rows[0] == ["trajectory_id", "node_index", "t_s", "x_km", "y_km", "z_km", "vx_kms", "vy_kms", "vz_kms"]
    M, R = result.trajectories.shape[:2]
    assert len(rows) == 1 + M * R
    i, j = 2, R - 1
    row = rows[1 + i * R + j]
    assert row[:2] == [str(i), str(j)]
    assert float(row[2]) == result.times[j]  # 17 significant digits: exact round trip
    assert np.array_equal(np.array(row[3:], dtype=float), result.trajectories[i, j])
    err = np.full((R, M), 1e-13)
    io.write_samples_csv(p, result, oracle_errors=err)
    rows = list(csv.reader(open(p)))
    assert rows[0][-1] == "oracle_rel_err" and float(rows[5][-1]) == 1e-13


def test_report_json(tmp_path, result):
    p = tmp_path / "report.json"
    io.write_report_json(p, result, metadata={"mode": "grouped"}, oracle_max_per_trajectory=[1e-12, 3e-12, 2e-12])
    d = json.load(open(p))
    assert d["metadata"] == {"mode": "grouped"}
    assert d["group_sizes"] == [int(g) for g in result.group_sizes]
    assert d["segment_boundaries"] == list(result.segments.boundaries)
    S, P = len(result.reports), len(result.reports[0])
    assert len(d["iteration_reports"]) == S * P
    r = d["iteration_reports"][-1]
    assert (r["segment"], r["group"]) == (S - 1, P - 1)
    assert r["iterations"] == result.reports[S - 1][P - 1].iterations and r["converged"] is True
    assert d["oracle_check"]["max"] == 3e-12


def test_error_history_csv(tmp_path, result):
    p = tmp_path / "hist.csv"
    io.write_error_history_csv(p, result)
    rows = list(csv.reader(open(p)))
    assert rows[0] == ["segment", "group", "iteration", "error"]
    n = sum(len(result.reports[s][g].per_iteration_errors) for s in range(len(result.reports))
            for g in range(len(result.reports[s])))
    assert len(rows) == 1 + n and rows[1][:3] == ["0", "0", "1"]


def test_read_config_json(tmp_path):
    p = tmp_path / "run.json"
    p.write_text(json.dumps({"nodes": 128, "tolerance": 1e-11, "segments": "per-orbit", "mode": "independent",
                             "span_periods": 2.5, "output": {"samples": "s.csv"},
                             "benchmark": {"repeat": 3, "threads": [1, 4], "modes": ["independent", "grouped"]}}))
    s = io.read_config_json(p)
    assert s.config.n_nodes == 128 and s.config.tolerance == 1e-11 and s.config.segment_policy == "per_orbit"
    assert s.mode == "independent" and s.span_periods == 2.5 and s.output.samples == "s.csv"
    assert s.output.report == "report.json" and s.benchmark.threads == [1, 4] and s.benchmark.repeat == 3
    # validation and messages (io.hpp:358-431)
    for bad, msg in [({"nodes": 2}, "nodes must be at least 3"), ({"tolerance": 0}, "tolerance must be positive"),
                     ({"span_s": 10, "span_periods": 1}, "not both"), ({"bogus": 1}, "unknown key 'bogus'"),
                     ({"start": "hot"}, "start mode must be"), ({"segments": "x"}, "segment policy must be")]:
        p.write_text(json.dumps(bad))
        with pytest.raises(io.ParseError, match=msg):
            io.read_config_json(p)


def test_benchmark_csv_and_summary(tmp_path):
    rep = ps.BenchmarkReport(machine="test", repeat=2, rows=[
        ps.BenchmarkRow("independent", 1, 16, 0.5, 1.0, 22, 0.0),
        ps.BenchmarkRow("augmented_parallel", 4, 1, 0.25, 2.0, 23, 1.5e-13)])
    p = tmp_path / "bench.csv"
    io.write_benchmark_csv(p, rep)
    rows = list(csv.reader(open(p)))
    assert rows[0] == ["mode", "threads", "groups", "wall_time_s", "speedup", "max_iterations", "max_discrepancy"]
    assert rows[2][:6] == ["augmented_parallel", "4", "1", "0.25", "2", "23"]
    assert float(rows[2][6]) == 1.5e-13  # 17 significant digits (io.hpp format_double)
    s = io.benchmark_summary(rep)
    assert s.startswith("machine: test, median of 2 run(s)\n") and "augmented_parallel" in s.splitlines()[3]


def test_writers_create_parent_dirs_and_map_open_failures(tmp_path, result):
    """open_output (io.hpp:75-84): parent directories are created; an unopenable path is a
    ParseError 'cannot open ... for writing'."""
    p = tmp_path / "a" / "b" / "report.json"
    io.write_report_json(p, result)
    assert p.exists()
    blocker = tmp_path / "file"
    blocker.write_text("x")
    with pytest.raises(io.ParseError, match="cannot open .* for writing"):
        io.write_samples_csv(blocker / "samples.csv", result)


def test_report_json_non_finite_is_null(tmp_path, result):
    """nlohmann::json writes non-finite doubles as null; the file stays valid JSON."""
    p = tmp_path / "r.json"
    io.write_report_json(p, result, metadata={"inf": float("inf"), "nan": float("nan"), "ok": 1.5})
    text = p.read_text()
    assert "Infinity" not in text and "NaN" not in text
    d = json.loads(text)
    assert d["metadata"] == {"inf": None, "nan": None, "ok": 1.5}


@pytest.mark.parametrize("text", ["+1", "1_0", "0x10", "1e", "", "e5", "1.2.3", "1 2"])
def test_number_grammar_is_from_chars(text):
    """parse_double (io.hpp:35-48) = std::from_chars: no '+', no '_', no hex."""
    with pytest.raises(io.ParseError, match="cannot parse number"):
        io._parse_double(text, "ctx")


def test_number_grammar_accepts_from_chars_forms():
    for t, v in (("-1.5e3", -1500.0), (" 2.0\r", 2.0), (".5", 0.5), ("5.", 5.0), ("-inf", float("-inf"))):
        assert io._parse_double(t, "ctx") == v
