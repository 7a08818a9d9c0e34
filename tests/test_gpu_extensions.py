"""Parity of the device path on the BASELINE extensions the reference does not have
(SPEC.md:17, :189, :350): the relativistic n_body_1pn force model (config 5) and the
hot start (config 3).  Their oracle is the repo's own CPU extension of the
restatement, pinned by oracle/ext_tests.cpp (Schwarzschild limit, perihelion advance,
PC vs RKF7(8) <= 1e-9) — parity here is GPU vs that oracle, same bars as the
reference path: 1e-10 relative on every node sample, iterations within +-1.
"""
import numpy as np
import pytest

import paper_2301_03989_b200 as ps

pytestmark = pytest.mark.gpu


def _parity(got, want, tol=1e-10):
    assert got.iterations.shape == want.iterations.shape
    disc = ps.max_state_discrepancy(got.trajectories, want.trajectories)
    diter = int(np.abs(got.iterations.astype(int) - want.iterations.astype(int)).max())
    assert disc <= tol, disc
    assert diter <= 1, diter
    return disc


def _rel_setup(m, n, frac, bodies="planets8", spread=1e-5, policy="single"):
    base = ps.reference_state()
    states = ps.make_clone_batch(base, m, spread)
    period = ps.osculating_period(base, ps.MU_SUN)
    plan = ps.plan_segments(base, 0.0, frac * period, ps.MU_SUN, policy, n)
    blist = [] if bodies == "none" else (ps.reference_bodies() if bodies == "reference" else ps.planets8())
    cfg = ps.reference_force_config("n_body_1pn", bodies=blist, n_nodes=n)
    return states, plan, cfg


@pytest.mark.parametrize("n", [64, 128, 200, 256])
@pytest.mark.parametrize("unified,kernel", [(1, "k_pc_uni"), (0, "k_pc_ws_fold")])
def test_c5_relativistic_node_sweep(ctx, oracle, n, unified, kernel):
    """C5: Sun + 8 planets with the EIH 1PN correction, node sweep: the unified folded kernel
    (auto choice for this force-bound model up to N = 200) and the warp-specialised one."""
    states, plan, cfg = _rel_setup(24, n, 0.87)
    ctx.set_option("unified", unified)
    try:
        got = ctx.run_batch(states, cfg, plan, "independent")
        assert ctx.kernel_name().split(".")[0] == kernel
    finally:
        ctx.set_option("unified", 2)
    want = oracle.run_batch(states, cfg, plan, "independent", 8)
    _parity(got, want)
    assert got.converged.all()
    # the relativistic term is resolved: it moves the solution far above the parity bar
    newt = ctx.run_batch(states, ps.reference_force_config("n_body", bodies=cfg.bodies, n_nodes=n), plan,
                         "independent")
    assert ps.max_state_discrepancy(got.trajectories, newt.trajectories) > 1e-9


def test_relativistic_sun_only(ctx, oracle):
    """Schwarzschild limit (no perturbing bodies): only the Sun row of the node table."""
    states, plan, cfg = _rel_setup(16, 200, 1.0, bodies="none")
    got = ctx.run_batch(states, cfg, plan, "independent")
    want = oracle.run_batch(states, cfg, plan, "independent", 8)
    _parity(got, want)


@pytest.mark.parametrize("mode,p,m", [("grouped", 4, 32), ("augmented", 1, 24)])
def test_relativistic_group_modes(ctx, oracle, mode, p, m):
    """Generic slot kernel (groups of 8) and the wide-group path on the 1PN model."""
    states, plan, cfg = _rel_setup(m, 128, 0.6, bodies="reference")
    cfg.p_groups = p
    got = ctx.run_batch(states, cfg, plan, mode)
    want = oracle.run_batch(states, cfg, plan, mode, 4)
    _parity(got, want)


def _tabulate(body, t0, t1, span, n=24):
    """Chebyshev segments of an analytic body on Lobatto nodes (fit_chebyshev_segment,
    ephemeris.hpp:112-152, restated with numpy for the test input)."""
    segs = []
    a = t0
    while a < t1:
        b = min(a + span, t1)
        tau = -np.cos(np.pi * np.arange(n) / (n - 1))
        t = 0.5 * (b - a) * tau + 0.5 * (b + a)
        pos = np.array([ps.elements_to_state(body.elements, ps.MU_SUN, x)[1:4] for x in t])
        cs = [np.polynomial.chebyshev.chebfit(tau, pos[:, c], n - 1) for c in range(3)]
        segs.append((a, b, cs[0], cs[1], cs[2]))
        a = b
    return ps.BodySpec(body.name, body.mu, body.elements, segments=segs)


def test_relativistic_tabulated_ephemeris(ctx, oracle):
    """Tabulated (Chebyshev) bodies: positions by Clenshaw and velocities by the
    derivative series on the device, against the oracle's derivative coefficients."""
    base = ps.reference_state()
    period = ps.osculating_period(base, ps.MU_SUN)
    states = ps.make_clone_batch(base, 16, 1e-5)
    plan = ps.plan_segments(base, 0.0, 0.5 * period, ps.MU_SUN, "single", 128)
    bodies = [_tabulate(b, -1.0, 0.5 * period + 1.0, 20 * 86400.0) for b in ps.reference_bodies()]
    cfg = ps.reference_force_config("n_body_1pn", bodies=bodies, n_nodes=128)
    got = ctx.run_batch(states, cfg, plan, "independent")
    want = oracle.run_batch(states, cfg, plan, "independent", 8)
    _parity(got, want)


def _hot_setup(m, frac, bodies="reference", kind="n_body", n=200):
    base = ps.reference_state()
    states = ps.make_clone_batch(base, m, 1e-5)
    period = ps.osculating_period(base, ps.MU_SUN)
    plan = ps.plan_segments(base, 0.0, frac * period, ps.MU_SUN, "per_orbit", n)
    blist = [] if bodies == "none" else (ps.reference_bodies() if bodies == "reference" else ps.planets8())
    cfg = ps.reference_force_config(kind, bodies=blist, n_nodes=n, start_mode="hot")
    return states, plan, cfg


def test_c3_hot_start_multisegment(ctx, oracle):
    """C3 restart semantics with hot starts: per-orbit segments 1/1/1/0.5 periods (the
    truncated last segment falls back to warm), parity with the oracle and the same fixed
    point as the reference's warm restart."""
    states, plan, cfg = _hot_setup(32, 3.5)
    assert len(plan.boundaries) == 5
    got = ctx.run_batch(states, cfg, plan, "independent")
    want = oracle.run_batch(states, cfg, plan, "independent", 8)
    _parity(got, want)
    cfg.start_mode = "warm"
    warm = ctx.run_batch(states, cfg, plan, "independent")
    assert ps.max_state_discrepancy(got.trajectories, warm.trajectories) <= 1e-10
    assert np.array_equal(got.iterations[0], warm.iterations[0])  # segment 0 is warm


def test_hot_start_pays_on_periodic_correction(ctx, oracle):
    """Sun-only 1PN: the relativistic correction repeats every orbit, so the hot start
    cuts the iterations of later segments (oracle/ext_tests.cpp pins the same)."""
    states, plan, cfg = _hot_setup(16, 3.0, bodies="none", kind="n_body_1pn")
    got = ctx.run_batch(states, cfg, plan, "independent")
    want = oracle.run_batch(states, cfg, plan, "independent", 8)
    _parity(got, want)
    cfg.start_mode = "warm"
    warm = ctx.run_batch(states, cfg, plan, "independent")
    assert 10 * got.iterations[2].sum() < 7 * warm.iterations[2].sum()


@pytest.mark.parametrize("mode,p,m", [("grouped", 4, 32), ("augmented", 1, 24)])
def test_hot_start_group_modes(ctx, oracle, mode, p, m):
    """Hot start on the generic slot kernel (groups of 8) and the wide-group path."""
    states, plan, cfg = _hot_setup(m, 2.0, n=128)
    cfg.p_groups = p
    got = ctx.run_batch(states, cfg, plan, mode)
    want = oracle.run_batch(states, cfg, plan, mode, 4)
    _parity(got, want)


@pytest.mark.parametrize("n", [33, 50, 99, 201])
def test_relativistic_dense_node_counts(ctx, oracle, n):
    """1PN at N % 8 != 0 (dense warp-specialised / generic kernels) against the oracle."""
    states, plan, cfg = _rel_setup(12, n, 0.5)
    got = ctx.run_batch(states, cfg, plan, "independent")
    assert ctx.kernel_name().split(".")[0] in ("k_pc_ws", "k_pc_segment")
    want = oracle.run_batch(states, cfg, plan, "independent", 8)
    _parity(got, want)


@pytest.mark.parametrize("n", [136, 216, 232])
@pytest.mark.parametrize("kind", ["n_body", "n_body_1pn"])
def test_hot_start_folded_tile_plans(ctx, oracle, n, kind):
    """Hot start (EXTENSION) over per-orbit segments with the folded tile plans that use
    extra units (136), none (216) and b0 from the DMMA stream (136, 232)."""
    states, plan, cfg = _hot_setup(12, 2.2, kind=kind, n=n)
    got = ctx.run_batch(states, cfg, plan, "independent")
    want = oracle.run_batch(states, cfg, plan, "independent", 8)
    _parity(got, want)
