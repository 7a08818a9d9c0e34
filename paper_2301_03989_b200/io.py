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
from dataclasses import dataclass, field
from typing import List

import numpy as np

from .api import BodySpec, Error

BATCH_CSV_HEADER = "epoch_s,x_km,y_km,z_km,vx_kms,vy_kms,vz_kms"  # io.hpp:120-121


class ParseError(Error):
    """pswarm::ParseError (errors.hpp)."""


def format_double(x: float) -> str:
    return format(float(x), ".17g")


def _parse_double(text: str, ctx: str) -> float:
    t = text.strip(" \t\r")
    try:
        return float(t)
    except ValueError:
        raise ParseError(f"{ctx}: cannot parse number '{t}'") from None


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
    with open(path, "w") as f:
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
    with open(path, "w") as f:
        json.dump(root, f, indent=2)
        f.write("\n")
