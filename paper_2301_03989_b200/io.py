"""Input formats of the batch path: the initial-condition CSV and the
ephemeris system JSON of the reference (io.hpp:117-305), so a real ephemeris exported in
the reference's schema (analytic elements or tabulated Chebyshev segments) feeds the
device path unchanged — tabulated bodies are evaluated per node by Clenshaw on the GPU
(k_ephemeris).  Validation and messages follow the reference; numbers are written with
17 significant digits (value-exact round trip, io.hpp:29-33).
"""
from __future__ import annotations

import json
import math
import os
import re
from dataclasses import dataclass, field
from typing import List

import numpy as np

from .api import BodySpec, Error

BATCH_CSV_HEADER = "epoch_s,x_km,y_km,z_km,vx_kms,vy_kms,vz_kms"  # io.hpp:120-121


class ParseError(Error):
    """pswarm::ParseError (errors.hpp)."""


def format_double(x: float) -> str:
    return format(float(x), ".17g")


# std::from_chars(double, chars_format::general) grammar (io.hpp:35-48): optional '-', decimal
# mantissa, optional exponent, or inf / infinity / nan[(chars)] — no '+', no '_', no hex
_NUMBER = re.compile(r"-?(?:(?:[0-9]+\.?[0-9]*|\.[0-9]+)(?:[eE][+-]?[0-9]+)?|(?i:inf(?:inity)?|nan(?:\([0-9A-Za-z_]*\))?))")


def _parse_double(text: str, ctx: str) -> float:
    t = text.lstrip(" \t").rstrip(" \t\r")  # io.hpp:36-43
    if not _NUMBER.fullmatch(t):
        raise ParseError(f"{ctx}: cannot parse number '{t}'")
    return float(t.split("(")[0]) if t.lower().lstrip("-").startswith("nan") else float(t)


def _open_output(path):
    """open_output (io.hpp:75-84): creates the parent directories; failures raise ParseError."""
    path = os.fspath(path)
    try:
        parent = os.path.dirname(path)
        if parent:
            os.makedirs(parent, exist_ok=True)
        return open(path, "w")
    except OSError:
        raise ParseError(f"cannot open '{path}' for writing") from None


def _json_value(x):
    """nlohmann::json serialises non-finite doubles as null (io.hpp:479-480 dump)."""
    if isinstance(x, float) and not math.isfinite(x):
        return None
    if isinstance(x, dict):
        return {k: _json_value(v) for k, v in x.items()}
    if isinstance(x, (list, tuple)):
        return [_json_value(v) for v in x]
    return x


def _dump_json(root, f):
    json.dump(_json_value(root), f, indent=2, allow_nan=False)
    f.write("\n")


def read_batch_csv(path) -> np.ndarray:
    """read_batch_csv (io.hpp:123-160) -> states [M, 7] = (epoch, r, v)."""
    try:
        f = open(path, newline="")
    except OSError:
        raise ParseError(f"cannot open '{path}'") from None
    with f:
        first = f.readline().rstrip("\n").rstrip("\r")
        if first != BATCH_CSV_HEADER:
            raise ParseError(f"'{path}': first line must be '{BATCH_CSV_HEADER}'")
        rows = []
        for row, line in enumerate(f, start=1):
            line = line.rstrip("\n").rstrip("\r")
            if not line:
                continue
            fields = line.split(",")
            if len(fields) != 7:
                raise ParseError(f"'{path}' row {row}: expected 7 fields, got {len(fields)}")
            ctx = f"'{path}' row {row}"
            vals = [_parse_double(x, ctx) for x in fields]
            if not all(math.isfinite(v) for v in vals):
                raise ParseError(f"{ctx}: non-finite state")
            rows.append(vals)
    if not rows:
        raise ParseError(f"'{path}': no initial conditions")
    return np.asarray(rows, dtype=np.float64)


def write_batch_csv(path, states) -> None:
    """write_batch_csv (io.hpp:162-178)."""
    st = np.asarray(states, dtype=np.float64).reshape(-1, 7)
    with _open_output(path) as f:
        f.write(BATCH_CSV_HEADER + "\n")
        for s in st:
            f.write(",".join(format_double(x) for x in s) + "\n")


@dataclass
class SystemModel:
    """SystemModel (io.hpp:183-188)."""
    frame: str = "heliocentric-ecliptic-J2000"
    central_name: str = "sun"
    central_mu: float = 0.0
    bodies: List[BodySpec] = field(default_factory=list)


def _check_keys(obj, allowed, where):
    if not isinstance(obj, dict):
        raise ParseError(f"{where}: expected an object")
    for k in obj:
        if k not in allowed:
            raise ParseError(f"{where}: unknown key '{k}'")


def read_system_json(path) -> SystemModel:
    """read_system_json (io.hpp:190-274)."""
    where = f"'{path}'"
    try:
        with open(path) as f:
            root = json.load(f)
    except OSError:
        raise ParseError(f"cannot open '{path}'") from None
    except json.JSONDecodeError as e:
        raise ParseError(f"{where}: {e}") from None
    try:
        _check_keys(root, {"header", "central", "bodies"}, where)
        header = root["header"]
        _check_keys(header, {"frame", "units"}, where + " header")
        units = header["units"]
        _check_keys(units, {"length", "time", "mu"}, where + " units")
        if units["length"] != "km" or units["time"] != "s" or units["mu"] != "km3/s2":
            raise ParseError(where + ": units must be km, s, km3/s2")
        model = SystemModel(frame=str(header["frame"]))
        central = root["central"]
        _check_keys(central, {"name", "mu"}, where + " central")
        model.central_name = str(central["name"])
        model.central_mu = float(central["mu"])
        if not model.central_mu > 0.0:
            raise ParseError(where + ": central mu must be positive")
        for jb in root.get("bodies", []):
            _check_keys(jb, {"name", "mu", "elements", "chebyshev"}, where + " body")
            name, mu = str(jb["name"]), float(jb["mu"])
            if not mu > 0.0:
                raise ParseError(f"{where}: body '{name}' mu must be positive")
            if ("elements" in jb) == ("chebyshev" in jb):
                raise ParseError(f"{where}: body '{name}' needs exactly one of elements/chebyshev")
            if "elements" in jb:
                je = jb["elements"]
                keys = ("a", "e", "i", "raan", "argp", "M0", "epoch")
                _check_keys(je, set(keys), f"{where} elements of '{name}'")
                el = [float(je[k]) for k in keys]
                if not el[0] > 0.0 or el[1] < 0.0 or el[1] >= 1.0:
                    raise ParseError(f"{where}: body '{name}' elements must describe a bound conic")
                model.bodies.append(BodySpec(name, mu, tuple(el)))
            else:
                segs = []
                for js in jb["chebyshev"]:
                    _check_keys(js, {"t_start", "t_end", "coeffs_x", "coeffs_y", "coeffs_z"},
                                f"{where} chebyshev segment of '{name}'")
                    cx, cy, cz = (np.asarray(js[k], dtype=np.float64) for k in ("coeffs_x", "coeffs_y", "coeffs_z"))
                    if cx.size == 0 or cx.size != cy.size or cx.size != cz.size:
                        raise ParseError(f"{where}: body '{name}' needs equal, non-empty coefficient arrays")
                    segs.append((float(js["t_start"]), float(js["t_end"]), cx, cy, cz))
                if not segs:
                    raise ParseError(f"{where}: body '{name}' has no segments")
                model.bodies.append(BodySpec(name, mu, None, segments=segs))
        return model
    except (KeyError, TypeError, ValueError) as e:
        raise ParseError(f"{where}: {e}") from None


def write_system_json(path, model: SystemModel) -> None:
    """write_system_json (io.hpp:276-305)."""
    root = {"header": {"frame": model.frame, "units": {"length": "km", "time": "s", "mu": "km3/s2"}},
            "central": {"name": model.central_name, "mu": model.central_mu}, "bodies": []}
    for b in model.bodies:
        jb = {"name": b.name, "mu": b.mu}
        if b.segments is None:
            a, e, i, raan, argp, m0, epoch = b.elements
            jb["elements"] = {"a": a, "e": e, "i": i, "raan": raan, "argp": argp, "M0": m0, "epoch": epoch}
        else:
            jb["chebyshev"] = [{"t_start": t0, "t_end": t1, "coeffs_x": list(map(float, cx)),
                                "coeffs_y": list(map(float, cy)), "coeffs_z": list(map(float, cz))}
                               for t0, t1, cx, cy, cz in b.segments]
        root["bodies"].append(jb)
    with _open_output(path) as f:
        _dump_json(root, f)


# ---------------------------------------------------------------------------
# Run configuration (JSON), io.hpp:307-431

@dataclass
class OutputSpec:
    samples: str = "samples.csv"
    report: str = "report.json"
    error_history: str = ""  # empty disables the per-iteration dump


@dataclass
class BenchmarkSpec:
    repeat: int = 5
    threads: List[int] = field(default_factory=lambda: [1])
    modes: List[str] = field(default_factory=lambda: ["independent", "augmented_parallel"])


@dataclass
class RunSettings:
    config: object = None  # api.PropagationConfig
    mode: str = "grouped"
    threads: int = 0
    span_s: float = 0.0
    span_periods: float = 0.87
    output: OutputSpec = field(default_factory=OutputSpec)
    benchmark: BenchmarkSpec = field(default_factory=BenchmarkSpec)


_START = {"warm": "warm", "cold": "cold"}
_ERRMODE = {"relative": "relative", "absolute": "absolute"}
_POLICY = {"single": "single", "per-orbit": "per_orbit"}
_FORCE = {"two_body": "two_body", "n_body": "n_body"}


def _pick(table, name, what):
    if name not in table:
        raise ParseError(f"{what} must be {' or '.join(repr(k) for k in table)}, got '{name}'")
    return table[name]


def read_config_json(path) -> RunSettings:
    """read_config_json (io.hpp:358-431): the run configuration file of the reference CLI,
    same keys, defaults, validation and messages."""
    from .api import PropagationConfig, parse_run_mode
    where = f"'{path}'"
    try:
        with open(path) as f:
            root = json.load(f)
    except OSError:
        raise ParseError(f"cannot open '{path}'") from None
    except json.JSONDecodeError as e:
        raise ParseError(f"{where}: {e}") from None
    s = RunSettings(config=PropagationConfig(force_kind="n_body"))
    try:
        _check_keys(root, {"nodes", "tolerance", "error_mode", "max_iterations", "start", "segments",
                           "max_segment_periods", "force_model", "proximity_floor_km", "mode", "groups",
                           "threads", "timeout_s", "span_s", "span_periods", "output", "benchmark"}, where)
        c = s.config
        c.n_nodes = int(root.get("nodes", 200))
        c.tolerance = float(root.get("tolerance", 1e-12))
        c.error_mode = _pick(_ERRMODE, root.get("error_mode", "relative"), "error mode")
        c.max_iterations = int(root.get("max_iterations", 100))
        c.start_mode = _pick(_START, root.get("start", "warm"), "start mode")
        c.segment_policy = _pick(_POLICY, root.get("segments", "single"), "segment policy")
        c.max_segment_periods = float(root.get("max_segment_periods", 1.0))
        c.force_kind = _pick(_FORCE, root.get("force_model", "n_body"), "force model")
        c.proximity_floor_km = float(root.get("proximity_floor_km", 1.0))
        c.p_groups = int(root.get("groups", 1))
        c.timeout_s = float(root.get("timeout_s", 0.0))
        try:
            s.mode = parse_run_mode(root.get("mode", "grouped"))
        except Exception as e:
            raise ParseError(str(e)) from None
        s.threads = int(root.get("threads", 0))
        if "span_s" in root and "span_periods" in root:
            raise ParseError(where + ": give span_s or span_periods, not both")
        s.span_s = float(root.get("span_s", 0.0))
        s.span_periods = float(root.get("span_periods", 0.0 if s.span_s != 0.0 else 0.87))
        if "output" in root:
            jo = root["output"]
            _check_keys(jo, {"samples", "report", "error_history"}, where + " output")
            s.output.samples = str(jo.get("samples", s.output.samples))
            s.output.report = str(jo.get("report", s.output.report))
            s.output.error_history = str(jo.get("error_history", s.output.error_history))
        if "benchmark" in root:
            jb = root["benchmark"]
            _check_keys(jb, {"repeat", "threads", "modes"}, where + " benchmark")
            s.benchmark.repeat = int(jb.get("repeat", s.benchmark.repeat))
            if "threads" in jb:
                s.benchmark.threads = [int(t) for t in jb["threads"]]
            if "modes" in jb:
                s.benchmark.modes = [parse_run_mode(str(m)) for m in jb["modes"]]
    except ParseError:
        raise
    except (KeyError, TypeError, ValueError) as e:
        raise ParseError(f"{where}: {e}") from None
    if s.config.n_nodes < 3:
        raise ParseError(where + ": nodes must be at least 3")
    if not s.config.tolerance > 0.0:
        raise ParseError(where + ": tolerance must be positive")
    if s.config.max_iterations < 1:
        raise ParseError(where + ": max_iterations must be positive")
    if s.span_s == 0.0 and s.span_periods == 0.0:
        raise ParseError(where + ": need a non-zero span_s or span_periods")
    return s


# ---------------------------------------------------------------------------
# Result writers, io.hpp:436-496

def write_samples_csv(path, result, oracle_errors=None) -> None:
    """write_samples_csv (io.hpp:436-459): one row per (trajectory, node); oracle_errors
    [R, M] (per-node RKF7(8) discrepancies, Context.oracle_check) adds a column."""
    traj = result.trajectories
    if traj is None:
        raise ParseError("write_samples_csv: the result carries no node samples (run with samples=True)")
    times = np.asarray(result.times)
    with _open_output(path) as f:
        f.write("trajectory_id,node_index,t_s,x_km,y_km,z_km,vx_kms,vy_kms,vz_kms")
        f.write(",oracle_rel_err\n" if oracle_errors is not None else "\n")
        for i in range(traj.shape[0]):
            for j in range(traj.shape[1]):
                row = [str(i), str(j), format_double(times[j])] + [format_double(x) for x in traj[i, j]]
                if oracle_errors is not None:
                    row.append(format_double(oracle_errors[j, i]))
                f.write(",".join(row) + "\n")


def write_report_json(path, result, metadata=None, oracle_max_per_trajectory=None) -> None:
    """write_report_json (io.hpp:461-486)."""
    root = {"metadata": metadata if metadata is not None else {},
            "group_sizes": [int(g) for g in result.group_sizes],
            "segment_boundaries": [float(b) for b in result.segments.boundaries],
            "warnings": list(result.warnings)}
    reports = []
    for seg, row in enumerate(result.reports):
        for g in range(len(row)):
            rep = row[g]
            reports.append({"segment": seg, "group": g, "iterations": int(rep.iterations),
                            "converged": bool(rep.converged), "final_error": float(rep.final_error)})
    root["iteration_reports"] = reports
    if oracle_max_per_trajectory is not None:
        v = [float(x) for x in oracle_max_per_trajectory]
        root["oracle_check"] = {"per_trajectory_max": v, "max": max(v)}
    with _open_output(path) as f:
        _dump_json(root, f)


def write_error_history_csv(path, result) -> None:
    """write_error_history_csv (io.hpp:488-503); needs a run with history=True."""
    with _open_output(path) as f:
        f.write("segment,group,iteration,error\n")
        for seg, row in enumerate(result.reports):
            for g in range(len(row)):
                for it, e in enumerate(row[g].per_iteration_errors):
                    f.write(f"{seg},{g},{it + 1},{format_double(e)}\n")


def write_benchmark_csv(path, report) -> None:
    """write_benchmark_csv (io.hpp:505-515) of api.run_benchmark's report."""
    with _open_output(path) as f:
        f.write("mode,threads,groups,wall_time_s,speedup,max_iterations,max_discrepancy\n")
        for r in report.rows:
            f.write(f"{r.mode},{r.threads},{r.groups},{format_double(r.wall_time_s)},{format_double(r.speedup)},"
                    f"{r.max_iterations},{format_double(r.max_discrepancy)}\n")


def benchmark_summary(report) -> str:
    """benchmark_summary (io.hpp:517-531)."""
    out = [f"machine: {report.machine}, median of {report.repeat} run(s)\n",
           "mode                   threads  groups  wall_time_s  speedup  max_iter  max_discrepancy\n"]
    for r in report.rows:
        out.append("%-22s %7u %7d %12.4f %8.3f %9d %16.3e\n" % (r.mode, r.threads, r.groups, r.wall_time_s,
                                                               r.speedup, r.max_iterations, r.max_discrepancy))
    return "".join(out)
