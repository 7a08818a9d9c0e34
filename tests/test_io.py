"""Input formats (io.hpp:117-305): IC CSV and ephemeris system JSON round trips,
the reference's validation rules, and a tabulated (Chebyshev) system read from JSON driving
the propagation exactly like the in-memory bodies."""
import json
import math

import numpy as np
import pytest

import paper_2301_03989_b200 as ps
from paper_2301_03989_b200 import io


def _tabulated(body, t0, t1, span, n=16):
    segs, a = [], t0
    while a < t1:
        b = min(a + span, t1)
        tau = -np.cos(np.pi * np.arange(n) / (n - 1))
        t = 0.5 * (b - a) * tau + 0.5 * (b + a)
        pos = np.array([ps.elements_to_state(body.elements, ps.MU_SUN, x)[1:4] for x in t])
        cs = [np.polynomial.chebyshev.chebfit(tau, pos[:, c], n - 1) for c in range(3)]
        segs.append((a, b, cs[0], cs[1], cs[2]))
        a = b
    return ps.BodySpec(body.name + "-tab", body.mu, None, segments=segs)


def test_batch_csv_round_trip_exact(tmp_path):
    states = ps.make_clone_batch(ps.reference_state(), 50, 1e-5)
    p = tmp_path / "ics.csv"
    io.write_batch_csv(p, states)
    assert open(p).readline().strip() == io.BATCH_CSV_HEADER
    assert np.array_equal(io.read_batch_csv(p), states)


@pytest.mark.parametrize("text,msg", [
    ("epoch,x\n", "first line must be"),
    (io.BATCH_CSV_HEADER + "\n0,1,2,3,4,5\n", "expected 7 fields, got 6"),
    (io.BATCH_CSV_HEADER + "\n0,1,2,3,4,5,nan\n", "non-finite state"),
    (io.BATCH_CSV_HEADER + "\n0,1,2,3,4,5,x7\n", "cannot parse number 'x7'"),
    (io.BATCH_CSV_HEADER + "\n\n", "no initial conditions"),
])
def test_batch_csv_errors(tmp_path, text, msg):
    p = tmp_path / "bad.csv"
    p.write_text(text)
    with pytest.raises(io.ParseError, match=msg):
        io.read_batch_csv(p)


def test_system_json_round_trip(tmp_path):
    bodies = ps.planets8()[:3] + [_tabulated(ps.reference_bodies()[1], 0.0, 4.0e7, 2.0e7)]
    model = io.SystemModel(central_mu=ps.MU_SUN, bodies=bodies)
    p = tmp_path / "system.json"
    io.write_system_json(p, model)
    back = io.read_system_json(p)
    assert back.central_mu == ps.MU_SUN and back.central_name == "sun"
    assert [b.name for b in back.bodies] == [b.name for b in bodies]
    for a, b in zip(back.bodies, bodies):
        assert a.mu == b.mu
        if b.segments is None:
            assert tuple(a.elements) == tuple(b.elements)
        else:
            for sa, sb in zip(a.segments, b.segments):
                assert sa[0] == sb[0] and sa[1] == sb[1]
                assert all(np.array_equal(sa[k], sb[k]) for k in (2, 3, 4))


def _system(**over):
    root = {"header": {"frame": "heliocentric-ecliptic-J2000", "units": {"length": "km", "time": "s", "mu": "km3/s2"}},
            "central": {"name": "sun", "mu": ps.MU_SUN},
            "bodies": [{"name": "b", "mu": 1.0, "elements": {"a": 1e8, "e": 0.1, "i": 0, "raan": 0, "argp": 0,
                                                             "M0": 0, "epoch": 0}}]}
    for k, v in over.items():
        root[k] = v
    return root


@pytest.mark.parametrize("mutate,msg", [
    (lambda r: r["header"]["units"].update(length="m"), "units must be km, s, km3/s2"),
    (lambda r: r["central"].update(mu=-1.0), "central mu must be positive"),
    (lambda r: r["bodies"][0].update(mu=0.0), "mu must be positive"),
    (lambda r: r["bodies"][0]["elements"].update(e=1.2), "bound conic"),
    (lambda r: r["bodies"][0].update(chebyshev=[]), "exactly one of elements/chebyshev"),
    (lambda r: r.update(extra=1), "unknown key 'extra'"),
    (lambda r: r["bodies"][0].pop("elements") and r["bodies"][0].update(chebyshev=[]), "has no segments"),
])
def test_system_json_errors(tmp_path, mutate, msg):
    root = _system()
    mutate(root)
    p = tmp_path / "sys.json"
    p.write_text(json.dumps(root))
    with pytest.raises(io.ParseError, match=msg):
        io.read_system_json(p)


def test_tabulated_system_from_json_drives_oracle_identically(tmp_path, oracle):
    base = ps.reference_state()
    period = ps.osculating_period(base, ps.MU_SUN)
    bodies = [_tabulated(b, -1.0, 0.5 * period + 1.0, 25 * 86400.0) for b in ps.reference_bodies()]
    p = tmp_path / "system.json"
    io.write_system_json(p, io.SystemModel(central_mu=ps.MU_SUN, bodies=bodies))
    loaded = io.read_system_json(p).bodies
    states = ps.make_clone_batch(base, 4, 1e-5)
    plan = ps.plan_segments(base, 0.0, 0.5 * period, ps.MU_SUN, "single", 64)
    a = oracle.run_batch(states, ps.reference_force_config("n_body", bodies=bodies, n_nodes=64), plan, "independent", 2)
    b = oracle.run_batch(states, ps.reference_force_config("n_body", bodies=loaded, n_nodes=64), plan, "independent", 2)
    assert np.array_equal(a.trajectories, b.trajectories)
    assert not math.isnan(a.trajectories.sum())


@pytest.mark.gpu
def test_tabulated_system_from_json_on_device(tmp_path, ctx, oracle):
    base = ps.reference_state()
    period = ps.osculating_period(base, ps.MU_SUN)
    bodies = [_tabulated(b, -1.0, 0.87 * period + 1.0, 25 * 86400.0) for b in ps.planets8()]
    p = tmp_path / "system.json"
    io.write_system_json(p, io.SystemModel(central_mu=ps.MU_SUN, bodies=bodies))
    cfg = ps.reference_force_config("n_body", bodies=io.read_system_json(p).bodies, n_nodes=200)
    states = ps.make_clone_batch(base, 32, 1e-5)
    plan = ps.plan_segments(base, 0.0, 0.87 * period, ps.MU_SUN, "single", 200)
    got = ctx.run_batch(states, cfg, plan, "independent")
    want = oracle.run_batch(states, cfg, plan, "independent", 8)
    assert ps.max_state_discrepancy(got.trajectories, want.trajectories) <= 1e-10
    assert int(np.abs(got.iterations.astype(int) - want.iterations.astype(int)).max()) <= 1
