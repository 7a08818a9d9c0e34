"""Device RKF7(8) verifier (pswarm_oracle_check; oracle.hpp:63-183, cli.hpp:238-261):
the batched --oracle-check must reproduce the CPU oracle's RK samples, confirm the PC
path at the reference's acceptance bar (criterion 3: <= 1e-9, acceptance.cpp:148-172)
and raise the reference's OracleError on bad inputs."""
import numpy as np
import pytest

import paper_2301_03989_b200 as ps

pytestmark = pytest.mark.gpu


def _setup(m, kind="n_body", bodies="reference", frac=0.87, n=200):
    base = ps.reference_state()
    states = ps.make_clone_batch(base, m, 1e-5)
    period = ps.osculating_period(base, ps.MU_SUN)
    plan = ps.plan_segments(base, 0.0, frac * period, ps.MU_SUN, "single", n)
    blist = {"reference": ps.reference_bodies, "planets8": ps.planets8, "none": list}[bodies]()
    cfg = ps.reference_force_config(kind, bodies=blist, n_nodes=n)
    return states, plan, cfg


@pytest.mark.parametrize("kind,bodies", [("n_body", "planets8"), ("n_body_1pn", "planets8"), ("two_body", "none")])
def test_rk_samples_match_cpu_oracle(ctx, oracle, kind, bodies):
    states, plan, cfg = _setup(4, kind, bodies)
    res = ctx.run_batch(states, cfg, plan, "independent")
    rk, _, _ = ctx.oracle_check(states, cfg, res.times)
    for i in range(4):
        want = oracle.rk_sample(states[i], cfg, res.times)
        assert ps.max_state_discrepancy(rk[i:i + 1], want[None]) <= 1e-11


def test_oracle_check_confirms_pc_at_acceptance_bar(ctx):
    """64 clones, Sun + 2 planets (acceptance.cpp:135-172): PC vs RKF78 <= 1e-9."""
    states, plan, cfg = _setup(64)
    res = ctx.run_batch(states, cfg, plan, "independent")
    rk, node, mx = ctx.oracle_check(states, cfg, res.times, candidate=res.trajectories)
    assert mx.max() <= 1e-9, mx.max()
    assert node.shape == (64, res.times.size) and np.allclose(node.max(axis=1), mx)
    assert ps.max_state_discrepancy(res.trajectories, rk) <= 1e-9


def test_oracle_check_two_body_closed_form(ctx, oracle):
    el = [1.3e8, 0.2, 0.05, 0.4, 0.9, 0.0, 0.0]
    base = ps.elements_to_state(el, ps.MU_SUN, 0.0)
    states = ps.make_clone_batch(base, 8, 1e-5)
    times = np.linspace(0.0, ps.osculating_period(base, ps.MU_SUN), 17)
    cfg = ps.reference_force_config("two_body")
    rk, _, _ = ctx.oracle_check(states, cfg, times)
    for i in range(8):
        for j in range(0, 17, 4):
            k = oracle.kepler_propagate(states[i], ps.MU_SUN, times[j])
            assert np.linalg.norm(rk[i, j, :3] - k[1:4]) / np.linalg.norm(k[1:4]) <= 1e-11


def test_oracle_check_errors(ctx):
    states, plan, cfg = _setup(2)
    times = np.array([0.0, 1.0e5])
    with pytest.raises(ps.OracleError, match="tolerances must be positive"):
        ctx.oracle_check(states, cfg, times, rel_tol=0.0)
    with pytest.raises(ps.OracleError, match="must begin at the state epoch"):
        ctx.oracle_check(states, cfg, times + 1.0)
    with pytest.raises(ps.OracleError, match="exceeded 3 steps"):
        ctx.oracle_check(states, cfg, np.array([0.0, 3.0e7]), max_steps=3)
