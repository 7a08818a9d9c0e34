"""End-to-end parity of the device propagation path (persistent slot kernel)
against the CPU oracle on the same seeded inputs.

Bars (BASELINE.json north_star): final positions/velocities within 1e-10
relative (runner.hpp:139-159 metric over every node sample), Picard iteration
counts within +-1 per (segment, group), identical segment counts.
"""
import subprocess
import os

import numpy as np
import pytest

import paper_2301_03989_b200 as ps

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _parity(got, want, tol=1e-10):
    assert got.iterations.shape == want.iterations.shape
    disc = ps.max_state_discrepancy(got.trajectories, want.trajectories)
    diter = int(np.abs(got.iterations.astype(int) - want.iterations.astype(int)).max())
    assert disc <= tol, disc
    assert diter <= 1, diter
    tdisc = ps.max_state_discrepancy(got.terminal_states[None, :, 1:], want.terminal_states[None, :, 1:])
    assert tdisc <= tol
    assert np.array_equal(got.terminal_states[:, 0], want.terminal_states[:, 0])
    return disc, diter


def _setup(m, n, frac, bodies="reference", spread=1e-5, policy="single", start="warm"):
    base = ps.reference_state()
    states = ps.make_clone_batch(base, m, spread)
    period = ps.osculating_period(base, ps.MU_SUN)
    plan = ps.plan_segments(base, 0.0, frac * period, ps.MU_SUN, policy, n)
    if bodies == "two_body":
        cfg = ps.reference_force_config("two_body", n_nodes=n, start_mode=start)
    else:
        blist = ps.reference_bodies() if bodies == "reference" else ps.planets8()
        cfg = ps.reference_force_config("n_body", bodies=blist, n_nodes=n, start_mode=start)
    return states, plan, cfg


def test_cpp_dropin_api():
    """The C++ drop-in headers (include/pswarm.hpp) on the device library."""
    exe = os.path.join(ROOT, "tests", "cpp", "dropin_test")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.strip().splitlines()[-1].endswith(" 0")


@pytest.mark.parametrize("start", ["cold", "warm"])
def test_c1_two_body_closed_form(ctx, oracle, start):
    """C1: 64 ICs, two-body, one full osculating period, N = 200 (acceptance.cpp:78-124)."""
    el = [1.3e8, 0.2, 0.05, 0.4, 0.9, 0.0, 0.0]
    base = ps.elements_to_state(el, ps.MU_SUN, 0.0)
    states = ps.make_clone_batch(base, 64, 1e-5)
    period = ps.osculating_period(base, ps.MU_SUN)
    plan = ps.plan_segments(base, 0.0, period, ps.MU_SUN, "single", 200)
    cfg = ps.reference_force_config("two_body", start_mode=start)
    got = ctx.run_batch(states, cfg, plan, "independent")
    want = oracle.run_batch(states, cfg, plan, "independent", 8)
    _parity(got, want)
    assert got.converged.all()
    # closed form: every node of every trajectory vs its own conic (1e-10)
    worst = 0.0
    for i in range(0, 64, 7):
        for j in range(0, 200, 9):
            k = oracle.kepler_propagate(states[i], ps.MU_SUN, got.times[j])
            s = got.trajectories[i, j]
            worst = max(worst, np.linalg.norm(s[:3] - k[1:4]) / np.linalg.norm(k[1:4]),
                        np.linalg.norm(s[3:] - k[4:]) / np.linalg.norm(k[4:]))
    assert worst <= 1e-10


@pytest.mark.parametrize("bodies", ["reference", "planets8"])
def test_c2_nbody_independent(ctx, oracle, bodies):
    """C2 (reduced to 64 ICs): Sun + planets, 0.87 period, N = 200, warm start."""
    states, plan, cfg = _setup(64, 200, 0.87, bodies)
    got = ctx.run_batch(states, cfg, plan, "independent")
    want = oracle.run_batch(states, cfg, plan, "independent", 8)
    _parity(got, want)
    # per-iteration error histories agree while the error is above the FP64 noise
    # floor of the iterate differences (~1e-13 relative); below it they are roundoff
    for g in range(0, 64, 9):
        a, b = got.reports[0][g].per_iteration_errors, want.reports[0][g].per_iteration_errors
        k = min(len(a), len(b))
        big = b[:k] > 1e-8
        assert np.allclose(a[:k][big], b[:k][big], rtol=1e-4, atol=0)


@pytest.mark.parametrize("mode,p,m", [("grouped", 8, 64), ("grouped", 16, 64), ("augmented", 1, 8),
                                      ("augmented", 1, 64), ("grouped", 2, 64), ("grouped", 3, 50)])
def test_group_modes_match_oracle(ctx, oracle, mode, p, m):
    """Groups within one CTA (<= 8 members, slot kernel) and wide groups (member-level
    rounds on the slot kernels): a group stops only when its worst member converges."""
    states, plan, cfg = _setup(m, 128, 0.6)
    cfg.p_groups = p
    got = ctx.run_batch(states, cfg, plan, mode)
    want = oracle.run_batch(states, cfg, plan, mode, 4)
    _parity(got, want)
    # mode invariance against independent masking (test_runner.cpp:45-59: < 1e-12)
    ind = ctx.run_batch(states, cfg, plan, "independent")
    assert ps.max_state_discrepancy(got.trajectories, ind.trajectories) < 1e-12


def test_wide_group_multisegment_and_errors(ctx, oracle):
    """Wide groups across segments (exact chaining) and non-convergence reporting."""
    states, plan, cfg = _setup(40, 64, 1.7, policy="per_orbit")
    got = ctx.propagate(states, [17, 23], plan, cfg)
    want = oracle.propagate(states, [17, 23], plan, cfg)
    _parity(got, want)
    cfg.max_iterations = 4
    with pytest.raises(ps.PropagationIncompleteError) as e:
        ctx.propagate(states, [17, 23], plan, cfg)
    with pytest.raises(ps.PropagationIncompleteError) as e_ref:
        oracle.propagate(states, [17, 23], plan, cfg)
    assert (e.value.segment, e.value.group) == (e_ref.value.segment, e_ref.value.group)


def test_wide_group_divergence_coordinates(ctx, oracle):
    states, plan, cfg = _setup(20, 32, 0.5, bodies="two_body", start="cold")
    states[13, 1:4] = [1e-110, 0.0, 0.0]
    with pytest.raises(ps.DivergenceError) as e:
        ctx.propagate(states, [20], plan, cfg)
    with pytest.raises(ps.DivergenceError) as e_ref:
        oracle.propagate(states, [20], plan, cfg)
    assert str(e.value) == str(e_ref.value)


def test_multisegment_per_orbit(ctx, oracle):
    """C3 (reduced): 2.5 periods per-orbit -> segments 1/1/0.5, exact chaining."""
    states, plan, cfg = _setup(32, 96, 2.5, policy="per_orbit")
    assert plan.segments() == 3
    got = ctx.run_batch(states, cfg, plan, "independent")
    want = oracle.run_batch(states, cfg, plan, "independent", 8)
    _parity(got, want)
    n = 96
    for s in range(1, 3):
        assert got.times[s * (n - 1)] == plan.boundaries[s]
    assert np.array_equal(got.terminal_states[:, 1:], got.trajectories[:, -1, :])


def test_backward_round_trip(ctx):
    """test_propagator.cpp:192-212: forward then backward recovers the batch (1e-9)."""
    states, plan, cfg = _setup(16, 64, 0.7, bodies="two_body")
    fwd = ctx.run_batch(states, cfg, plan, "independent")
    t_end = plan.boundaries[-1]
    back_plan = ps.plan_segments(fwd.terminal_states[0], t_end, 0.0, ps.MU_SUN, "single", 64)
    back = ctx.run_batch(fwd.terminal_states, cfg, back_plan, "independent")
    d = ps.max_state_discrepancy(back.terminal_states[None, :, 1:], states[None, :, 1:])
    assert d <= 1e-9


def test_warm_beats_cold(ctx):
    states, plan, cfg = _setup(6, 96, 0.6)
    warm = ctx.run_batch(states, cfg, plan, "independent")
    cfg.start_mode = "cold"
    cold = ctx.run_batch(states, cfg, plan, "independent")
    assert (warm.iterations < cold.iterations).all()


def test_nonconvergence_partial(ctx, oracle):
    states, plan, cfg = _setup(4, 64, 0.8, bodies="two_body", start="cold")
    cfg.max_iterations = 3
    with pytest.raises(ps.PropagationIncompleteError) as e:
        ctx.propagate(states, [2, 2], plan, cfg)
    with pytest.raises(ps.PropagationIncompleteError) as e_ref:
        oracle.propagate(states, [2, 2], plan, cfg)
    assert (e.value.segment, e.value.group) == (0, 0) == (e_ref.value.segment, e_ref.value.group)
    assert not e.value.partial.reports[0][0].converged


def test_timeout(ctx):
    states, plan, cfg = _setup(4, 64, 0.1)
    cfg.timeout_s = 1e-9
    with pytest.raises(ps.TimeoutError):
        ctx.propagate(states, [4], plan, cfg)


@pytest.mark.parametrize("n,kind,mode,opts,kernel", [
    (64, "n_body", "independent", {}, "k_pc_ws_fold.x2"),        # two CTAs per SM
    (200, "n_body", "independent", {}, "k_pc_ws_fold"),
    (200, "n_body", "grouped", {}, "k_pc_ws_fold"),              # in-CTA groups
    (200, "n_body", "augmented", {}, "k_pc_ws_fold"),            # member-level rounds
    (57, "n_body", "independent", {}, "k_pc_ws"),                # dense update
    (33, "n_body", "independent", {}, "k_pc_segment"),
    (200, "n_body", "independent", {"unified": 1}, "k_pc_uni"),
    (128, "n_body_1pn", "independent", {}, "k_pc_uni.x2"),       # relativistic
    (200, "n_body_1pn", "independent", {}, "k_pc_uni"),
])
def test_absolute_error_mode_every_kernel(ctx, oracle, n, kind, mode, opts, kernel):
    """ErrorMode::absolute (augment.hpp:45-47: |dr|, |dv| without the previous iterate's norms)
    through every solve kernel: a km / km/s tolerance, iterations and states against the oracle."""
    base = ps.reference_state()
    states = ps.make_clone_batch(base, 24, 1e-5)
    period = ps.osculating_period(base, ps.MU_SUN)
    plan = ps.plan_segments(base, 0.0, 0.6 * period, ps.MU_SUN, "single", n)
    cfg = ps.reference_force_config(kind, bodies=ps.planets8(), n_nodes=n)
    cfg.error_mode = "absolute"
    # km and km/s.  The absolute change of this orbit's iterate saw-tooths (odd iterations
    # ~1e-3 km, even ones ~1e4 km early on: the position update lags the velocity update), and
    # |r| ~ 1e8 km puts the FP64 noise of the position update near 1e-7 km, so a tolerance
    # around 1e-6 decides on noise; 1e-3 stops at iteration ~9, far from both
    cfg.tolerance = 1e-3
    cfg.p_groups = 6
    for k, v in opts.items():
        ctx.set_option(k, v)
    try:
        got = ctx.run_batch(states, cfg, plan, mode)
        assert ctx.kernel_name() == kernel
    finally:
        for k in opts:
            ctx.set_option(k, 2 if k == "unified" else 1)
    want = oracle.run_batch(states, cfg, plan, mode, 1)
    _parity(got, want)
    assert got.iterations.min() >= 3
    cfg.error_mode = "relative"  # the mode is in effect: a relative 1e-3 stops far earlier
    assert ctx.run_batch(states, cfg, plan, mode).iterations.max() < got.iterations.min()


def test_independent_timeout_is_per_trajectory(ctx, oracle):
    """run_independent gives every trajectory a propagate call -- and a deadline -- of its own
    (runner.hpp:63-80, propagator.hpp:233-236): a budget shorter than the whole batch but longer
    than any one trajectory's solve times nothing out in independent mode, while grouped mode
    (one propagate call for the batch) times out; a budget below one iteration times out
    trajectory 0 with the reference's message in both implementations."""
    states, plan, cfg = _setup(100_000, 64, 0.87, bodies="planets8")
    want = ctx.run_batch(states, cfg, plan, "independent", samples=False)
    cfg.timeout_s = 2e-3  # batch: ~10 ms of device time; one trajectory: ~30 iterations of ~10 us
    got = ctx.run_batch(states, cfg, plan, "independent", samples=False)
    assert np.array_equal(got.terminal_states, want.terminal_states)
    assert np.array_equal(got.iterations, want.iterations)
    with pytest.raises(ps.TimeoutError):
        ctx.run_batch(states, cfg, plan, "grouped", samples=False)
    small, plan_s, cfg_s = _setup(6, 32, 0.3, bodies="planets8")
    cfg_s.timeout_s = 1e-9
    with pytest.raises(ps.TimeoutError) as e:
        ctx.run_batch(small, cfg_s, plan_s, "independent")
    with pytest.raises(ps.TimeoutError) as e_ref:
        oracle.run_batch(small, cfg_s, plan_s, "independent", 1)
    assert str(e.value) == str(e_ref.value)


def test_mixed_epochs_rejected(ctx):
    states, plan, cfg = _setup(3, 16, 0.1, bodies="two_body")
    states[2, 0] = 10.0
    with pytest.raises(ps.AlignmentError, match="state 2"):
        ctx.propagate(states, [3], plan, cfg)


def test_divergence_reports_first_non_finite(ctx, oracle):
    """A state at |r| = 1e-110 passes the zero-radius guard but its 1/|r|^3 overflows,
    so the first update is non-finite; the first (node, column) in row-major order
    is reported with the group prefix (picard.hpp:26-36, augment.hpp:132-135)."""
    states, plan, cfg = _setup(3, 32, 0.5, bodies="two_body", start="cold")
    states[1, 1:4] = [1e-110, 0.0, 0.0]
    with pytest.raises(ps.DivergenceError) as e:
        ctx.propagate(states, [3], plan, cfg)
    with pytest.raises(ps.DivergenceError) as e_ref:
        oracle.propagate(states, [3], plan, cfg)
    assert str(e.value) == str(e_ref.value)
    assert (e.value.node, e.value.column) == (e_ref.value.node, e_ref.value.column)
    assert str(e.value).startswith("group 0: picard iteration produced a non-finite value")


def test_singularity_in_solve_names_body(ctx, oracle):
    """Trajectory 2 starts 0.4 km from venus-like at its epoch: the force guard
    raises SingularityError naming node, trajectory-in-group and body."""
    states, plan, cfg = _setup(4, 16, 0.05, start="cold")
    pos = oracle.body_positions(ps.reference_bodies(), ps.MU_SUN, np.array([0.0]))
    states[2, 1:4] = pos[0, 0] + np.array([0.4, 0.0, 0.0])
    errs = []
    for impl in (ctx, oracle):
        with pytest.raises(ps.SingularityError) as e:
            impl.propagate(states, [4], plan, cfg)
        errs.append(e.value)
    assert str(errs[0]) == str(errs[1]) and errs[0].body == "venus-like"
    assert "trajectory 2" in str(errs[0])


@pytest.mark.parametrize("n", [64, 72, 80, 88, 96, 104, 112, 120, 128, 160, 168, 184, 200, 232, 256])
def test_c5_node_sweep(ctx, oracle, n):
    """C5 node-count sweep (64-256 nodes per segment): every warp plan of the slot
    kernels and every per-N choice (two-CTA variants up to 128, the unified kernel at 80-96 and 112-128,
    single-slot force items up to 80, b0 from the FP group at 168-200) against the oracle,
    Sun + 8 planets, 0.6 period."""
    states, plan, cfg = _setup(24, n, 0.6, "planets8")
    got = ctx.run_batch(states, cfg, plan, "independent")
    want = oracle.run_batch(states, cfg, plan, "independent", 8)
    _parity(got, want)
    assert got.converged.all()


def test_c5_mask_stress_heterogeneous_iterations(ctx, oracle):
    """C5 convergence-mask stress: four quarters with clone spreads 1e-7 .. 1e-2 give
    heterogeneous iteration counts; per-trajectory masking refills freed slots, so
    every trajectory must still match its own oracle solve."""
    base = ps.reference_state()
    quarters = [ps.make_clone_batch(base, 40, sp) for sp in (1e-7, 1e-5, 1e-3, 1e-2)]
    states = np.concatenate(quarters)
    period = ps.osculating_period(base, ps.MU_SUN)
    plan = ps.plan_segments(base, 0.0, 0.87 * period, ps.MU_SUN, "single", 200)
    cfg = ps.reference_force_config("n_body", bodies=ps.planets8(), n_nodes=200)
    ctx.set_option("max_ctas", 3)  # few CTAs: slots are refilled many times
    try:
        got = ctx.run_batch(states, cfg, plan, "independent")
    finally:
        ctx.set_option("max_ctas", 0)
    want = oracle.run_batch(states, cfg, plan, "independent", 8)
    _parity(got, want)
    assert want.iterations.min() < want.iterations.max()  # heterogeneous by construction


def test_pinned_samples_overlapped_copy_identical(ctx):
    """Node samples into a caller-owned pinned buffer are copied per segment while the
    next segment computes; the result must be identical to the end-of-call copy."""
    from paper_2301_03989_b200 import api
    states, plan, cfg = _setup(40, 64, 2.5, policy="per_orbit")
    assert len(plan.boundaries) > 2
    buf = api.pinned_sample_buffer(len(states), plan)
    a = ctx.run_batch(states, cfg, plan, "independent", samples=buf)
    b = ctx.run_batch(states, cfg, plan, "independent")
    assert a.trajectories is buf
    assert np.array_equal(a.trajectories, b.trajectories)
    assert np.array_equal(a.terminal_states, b.terminal_states)


@pytest.mark.parametrize("n", [64, 128, 200, 256])
@pytest.mark.parametrize("fold,unified,kernel", [(1, 1, "k_pc_uni"), (1, 0, "k_pc_ws_fold"), (0, 0, "k_pc_ws")])
def test_mirror_folded_and_dense_updates(ctx, oracle, n, fold, unified, kernel):
    """The Picard update folded over the Chebyshev mirror symmetry (half the DMMAs,
    default where N % 8 == 0) in the unified kernel and in the warp-specialised one, and
    the dense update, all match the oracle; the kernel that ran is the one selected."""
    states, plan, cfg = _setup(24, n, 0.87, "planets8")
    ctx.set_option("fold", fold)
    ctx.set_option("unified", unified)
    try:
        got = ctx.run_batch(states, cfg, plan, "independent")
        name = ctx.kernel_name()
    finally:
        ctx.set_option("fold", 1)
        ctx.set_option("unified", 2)
    assert name.split(".")[0] == kernel
    want = oracle.run_batch(states, cfg, plan, "independent", 8)
    _parity(got, want)
    assert got.converged.all()


def test_unified_kernel_refill_and_multisegment(ctx, oracle):
    """k_pc_uni with few CTAs (slots refilled many times, heterogeneous iteration counts)
    over a multi-segment per-orbit plan: every trajectory matches its own oracle solve."""
    base = ps.reference_state()
    states = np.concatenate([ps.make_clone_batch(base, 30, sp) for sp in (1e-7, 1e-4, 1e-2)])
    period = ps.osculating_period(base, ps.MU_SUN)
    plan = ps.plan_segments(base, 0.0, 2.3 * period, ps.MU_SUN, "per_orbit", 200)
    cfg = ps.reference_force_config("n_body", bodies=ps.planets8(), n_nodes=200)
    ctx.set_option("max_ctas", 2)
    ctx.set_option("unified", 1)
    try:
        got = ctx.run_batch(states, cfg, plan, "independent")
        assert ctx.kernel_name().split(".")[0] == "k_pc_uni"
    finally:
        ctx.set_option("max_ctas", 0)
        ctx.set_option("unified", 2)
    want = oracle.run_batch(states, cfg, plan, "independent", 8)
    _parity(got, want)


@pytest.mark.parametrize("n", [8, 16, 24, 40, 56, 72, 88, 104, 120, 136, 144, 168, 184, 216, 248])
def test_folded_tile_plans(ctx, oracle, n):
    """Every folded tile plan against the oracle: pair-tile counts 1..16, with and without
    leftover tiles as single-n-tile units (staged rows), with and without the anchor row in
    a spare pair row (b0 from the DMMA stream), Sun + 8 planets, 0.5 period."""
    states, plan, cfg = _setup(12, n, 0.5, "planets8")
    ctx.set_option("unified", 0)  # (auto runs k_pc_uni.x2 at N = 80...96)
    try:
        got = ctx.run_batch(states, cfg, plan, "independent")
        assert ctx.kernel_name().split(".")[0] == "k_pc_ws_fold"
    finally:
        ctx.set_option("unified", 2)
    want = oracle.run_batch(states, cfg, plan, "independent", 8)
    _parity(got, want)


@pytest.mark.parametrize("n", [5, 13, 33, 50, 67, 99, 130, 201, 225, 241, 247, 255, 257, 263])
def test_dense_node_counts(ctx, oracle, n):
    """N % 8 != 0 (no mirror fold): the dense warp-specialised or generic slot kernels
    against the oracle, Sun + 8 planets, 0.5 period."""
    states, plan, cfg = _setup(12, n, 0.5, "planets8")
    got = ctx.run_batch(states, cfg, plan, "independent")
    assert ctx.kernel_name().split(".")[0] in ("k_pc_ws", "k_pc_segment")
    want = oracle.run_batch(states, cfg, plan, "independent", 8)
    _parity(got, want)


@pytest.mark.parametrize("n", [8, 24, 56, 104, 136, 184, 216, 248])
@pytest.mark.parametrize("kind", ["n_body", "n_body_1pn"])
def test_unified_tile_plans(ctx, oracle, n, kind):
    """k_pc_uni over its unit plans (2 x pair tiles over 16 warps) for both force models."""
    states, plan, cfg = _setup(12, n, 0.5, "planets8")
    cfg.force_kind = kind
    ctx.set_option("unified", 1)
    try:
        got = ctx.run_batch(states, cfg, plan, "independent")
        assert ctx.kernel_name().split(".")[0] == "k_pc_uni"
    finally:
        ctx.set_option("unified", 2)
    want = oracle.run_batch(states, cfg, plan, "independent", 8)
    _parity(got, want)


@pytest.mark.parametrize("n", [17, 23, 31, 49, 55, 63, 225, 241])
@pytest.mark.parametrize("mode,p", [("independent", 1), ("grouped", 3), ("augmented", 1)])
def test_small_n_staged_rows(ctx, oracle, n, mode, p):
    """The 128-thread small-N plan of the generic slot kernel (also the wide-group rounds) stages up to 31
    rows x 8 slots (more items than threads): every staged row must be finalised."""
    states, plan, cfg = _setup(12, n, 0.4, "planets8")
    cfg.p_groups = p
    ctx.set_option("slot_kernel", 1)  # the generic slot kernel where the mode allows it
    try:
        got = ctx.run_batch(states, cfg, plan, mode)
        assert ctx.kernel_name() == "k_pc_segment"
    finally:
        ctx.set_option("slot_kernel", 0)
    want = oracle.run_batch(states, cfg, plan, mode, 8)
    _parity(got, want)


@pytest.mark.parametrize("n", [64, 136, 200, 216])
@pytest.mark.parametrize("p", [6, 4, 3])  # 12 ICs -> groups of 2, 3, 4 members
def test_grouped_folded_kernels(ctx, oracle, n, p):
    """Grouped mode (group members share one convergence decision) through the folded
    kernels: groups of 2-4 members inside a 4-slot half, every tile plan."""
    states, plan, cfg = _setup(12, n, 0.5, "planets8")
    cfg.p_groups = p
    got = ctx.run_batch(states, cfg, plan, "grouped")
    assert ctx.kernel_name().split(".")[0] == "k_pc_ws_fold"
    want = oracle.run_batch(states, cfg, plan, "grouped", 8)
    _parity(got, want)


def test_non_elliptic_cold_fallback_and_warnings(ctx, oracle):
    """Non-elliptic ICs in a warm-start batch fall back to cold rows with a per-trajectory
    warning (propagator.hpp:94-99); results and warnings match the oracle."""
    base = ps.reference_state()
    states = ps.make_clone_batch(base, 8, 1e-5)
    states[[2, 5], 4:7] *= 1.5  # hyperbolic: beyond escape speed
    period = ps.osculating_period(base, ps.MU_SUN)
    plan = ps.plan_segments(base, 0.0, 0.05 * period, ps.MU_SUN, "single", 200)
    cfg = ps.reference_force_config("n_body", bodies=ps.planets8(), n_nodes=200)
    got = ctx.run_batch(states, cfg, plan, "independent")
    want = oracle.run_batch(states, cfg, plan, "independent", 8)
    _parity(got, want)
    assert got.warnings == want.warnings
    assert len(got.warnings) == 2 and "trajectory 2" in got.warnings[0] and "trajectory 5" in got.warnings[1]


def test_backward_and_single_ic_match_oracle(ctx, oracle):
    """Backward propagation (descending boundaries, omega2 < 0) and a one-IC batch."""
    base = ps.reference_state()
    period = ps.osculating_period(base, ps.MU_SUN)
    cfg = ps.reference_force_config("n_body", bodies=ps.planets8(), n_nodes=200)
    states = ps.make_clone_batch(base, 10, 1e-5)
    plan = ps.plan_segments(base, 0.0, -1.3 * period, ps.MU_SUN, "per_orbit", 200)
    got = ctx.run_batch(states, cfg, plan, "independent")
    want = oracle.run_batch(states, cfg, plan, "independent", 8)
    _parity(got, want)
    one = states[:1]
    plan1 = ps.plan_segments(base, 0.0, 0.7 * period, ps.MU_SUN, "single", 200)
    _parity(ctx.run_batch(one, cfg, plan1, "independent"), oracle.run_batch(one, cfg, plan1, "independent", 8))


def test_run_benchmark_harness(ctx):
    """api.run_benchmark (runner.hpp:186-253) on the device: rows per (mode, workers), the
    independent single-worker baseline, cross-mode discrepancy within the mode-invariance bar."""
    states, plan, cfg = _setup(16, 64, 0.5, "planets8")
    cfg.p_groups = 4
    rep = ps.run_benchmark(ctx, states, cfg, plan, thread_counts=(1, 8),
                           modes=("independent", "augmented_parallel", "grouped"), repeat=2)
    assert len(rep.rows) == 6 and rep.rows[0].speedup == 1.0 and rep.rows[0].groups == 16
    assert [r.groups for r in rep.rows] == [16, 16, 1, 1, 4, 4]
    assert all(r.wall_time_s > 0 and r.max_iterations > 0 for r in rep.rows)
    assert max(r.max_discrepancy for r in rep.rows) <= 1e-9  # test_runner.cpp:45-59


def test_reference_acceptance_program_on_device():
    """The reference's own acceptance program (proj/tests/acceptance.cpp), compiled
    UNCHANGED against include/ and linked with the device library (tests/cpp/Makefile
    ref_acceptance).  Criteria 1-5, 8, 9 are numerical contracts and must pass on the
    device.  Criteria 6 and 7 time CPU properties of the reference's thread pool
    (augmentation beats independent on one core; grouped runtime does not grow with
    workers); on the device `workers` has no meaning, so they are reported, not asserted."""
    exe = os.path.join(ROOT, "tests", "cpp", "ref_acceptance")
    if not os.path.exists(exe):
        pytest.skip("tests/cpp/ref_acceptance not built (needs /root/reference at build time)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=900)
    print(r.stdout)
    lines = [l for l in r.stdout.splitlines() if " criterion " in l]
    assert len(lines) == 9, r.stdout + r.stderr
    numeric = [l for l in lines if not any(f"criterion {k}:" in l for k in (6, 7))]
    assert all(l.startswith("PASS") for l in numeric), numeric


def _raise_info(fn):
    try:
        fn()
    except ps.Error as e:
        return type(e).__name__, str(e), getattr(e, "segment", None)
    return None


def test_independent_error_order_lowest_trajectory(ctx, oracle):
    """run_independent (runner.hpp:63-80) solves trajectory after trajectory: trajectory 0
    running out of iterations is raised before trajectory 5's divergence in the same
    segment (the serial reference never reaches trajectory 5)."""
    states, plan, cfg = _setup(8, 64, 0.5, bodies="two_body", start="cold")
    el = [0.8e8, 0.3, 0.05, 0.4, 0.9, 0.0, 0.0]  # tighter orbit: needs more iterations
    states[0, 1:] = ps.elements_to_state(el, ps.MU_SUN, 0.0)[1:]
    states[5, 1:4] = [1e-110, 0.0, 0.0]
    ok = ctx.run_batch(np.delete(states, 5, axis=0), cfg, plan, "independent")
    it = ok.iterations[0]
    assert it[0] > it[1:].max()  # trajectory 0 is the slow one
    cfg.max_iterations = int(it[1:].max()) + 1
    got = _raise_info(lambda: ctx.run_batch(states, cfg, plan, "independent"))
    want = _raise_info(lambda: oracle.run_batch(states, cfg, plan, "independent", 1))
    assert want[0] == "PropagationIncompleteError"
    assert got == want


def test_independent_error_order_later_segment(ctx, oracle):
    """Trajectory 1 diverges in segment 0, trajectory 0 fails to converge in segment 1:
    the serial reference raises trajectory 0's error (segment 1)."""
    states, plan, cfg = _setup(4, 64, 0.5, bodies="reference", start="cold")
    period = ps.osculating_period(ps.reference_state(), ps.MU_SUN)
    plan = ps.SegmentPlan(np.array([0.0, 0.05 * period, 0.9 * period]), 64)
    ok = ctx.run_batch(states, cfg, plan, "independent")
    k0, k1 = int(ok.iterations[0].max()), int(ok.iterations[1].max())
    assert k1 > k0
    cfg.max_iterations = k0 + 1
    states[1, 1:4] = [1e-110, 0.0, 0.0]
    got = _raise_info(lambda: ctx.run_batch(states, cfg, plan, "independent"))
    want = _raise_info(lambda: oracle.run_batch(states, cfg, plan, "independent", 1))
    assert want[0] == "PropagationIncompleteError" and want[2] == 1
    assert got == want


_FAR = ([0.8e8, 0.3, 0.05, 0.4, 0.9, 0.0, 0.0], [0.9e8, 0.2, 0.1, 0.2, 0.5, 0.3, 0.0])
_NEAR = ([1.15e8, 0.2, 0.05, 0.4, 0.9, 0.0, 0.0], [1.3e8, 0.08, 0.1, 0.2, 0.5, 0.3, 0.0])


def _mixed_states(m, elements=_FAR):
    """Clones of three different orbits interleaved: members of one group converge at
    different iteration counts, so a wide group needs several member-level rounds."""
    base = ps.reference_state()
    other = [ps.elements_to_state(el, ps.MU_SUN, 0.0) for el in elements]
    states = ps.make_clone_batch(base, m, 1e-5)
    for i in range(m):
        if i % 3:
            states[i, 1:] = other[i % 3 - 1][1:] * (1.0 + 1e-6 * i)
    return states


@pytest.mark.parametrize("mode,p", [("augmented", 1), ("grouped", 3), ("grouped", 5)])
@pytest.mark.parametrize("start", ["warm", "cold"])
def test_wide_groups_heterogeneous(ctx, oracle, mode, p, start):
    """Wide groups whose members converge at different counts (several rounds): group
    iterations exact, states within 1e-10, and the group error history equal to the
    oracle's max over members while it is above the noise floor."""
    states, plan, cfg = _setup(60, 64, 0.5, bodies="reference", start=start)
    states = _mixed_states(60)
    cfg.p_groups = p
    got = ctx.run_batch(states, cfg, plan, mode)
    want = oracle.run_batch(states, cfg, plan, mode, 4)
    _parity(got, want)
    assert np.array_equal(got.iterations, want.iterations)
    ind = oracle.run_batch(states, cfg, plan, "independent", 8)
    assert ind.iterations.min() < got.iterations.max()  # members really differ
    for g in range(p):
        a, b = got.reports[0][g].per_iteration_errors, want.reports[0][g].per_iteration_errors
        assert len(a) == len(b)
        big = b > 1e-8
        assert np.allclose(a[big], b[big], rtol=1e-4, atol=0)


def test_wide_groups_multisegment_hot(ctx, oracle):
    """Wide groups across per-orbit segments with hot start (EXTENSION): resumed members
    carry the hot-start correction of the group's final iterate."""
    base = ps.reference_state()
    states = _mixed_states(40, _NEAR)
    period = ps.osculating_period(base, ps.MU_SUN)
    plan = ps.plan_segments(base, 0.0, 2.0 * period, ps.MU_SUN, "per_orbit", 64)
    cfg = ps.reference_force_config("n_body", bodies=ps.reference_bodies(), n_nodes=64, start_mode="hot")
    got = ctx.propagate(states, [13, 27], plan, cfg)
    want = oracle.propagate(states, [13, 27], plan, cfg)
    _parity(got, want)


def test_wide_group_nonconvergence_runs_all_members(ctx, oracle):
    """One slow member out of iterations: the whole wide group runs to max_iterations and
    reports the group error there (propagator.hpp:300-312)."""
    states = _mixed_states(30)
    _, plan, cfg = _setup(30, 64, 0.5, bodies="two_body", start="cold")
    ind = oracle.run_batch(states, cfg, plan, "independent", 8)
    cfg.max_iterations = int(ind.iterations.max()) - 4  # group error ~1e-10, above the noise floor
    errs = []
    for impl in (ctx, oracle):
        with pytest.raises(ps.PropagationIncompleteError) as e:
            impl.propagate(states, [30], plan, cfg)
        errs.append(e.value)
    assert (errs[0].segment, errs[0].group) == (errs[1].segment, errs[1].group)
    a, b = errs[0].partial.reports[0][0], errs[1].partial.reports[0][0]
    assert a.iterations == b.iterations == cfg.max_iterations
    assert abs(a.final_error - b.final_error) <= 1e-3 * b.final_error


def test_pinned_terminal_buffer_direct_copy(ctx):
    """A page-locked caller buffer receives the terminal states by one DMA (device-side
    [M][7] pack): identical to the staged path, and reused across calls."""
    states, plan, cfg = _setup(37, 64, 0.4)
    ref = ctx.run_batch(states, cfg, plan, "independent", samples=False)
    buf = ps.pinned_terminal_buffer(37)
    for _ in range(2):
        got = ctx.run_batch(states, cfg, plan, "independent", samples=False, terminal=buf)
        assert got.terminal_states is buf
        assert np.array_equal(buf, ref.terminal_states)
    with pytest.raises(ps.ShapeError):
        ctx.run_batch(states, cfg, plan, "independent", terminal=np.zeros((36, 7)))


def test_wide_group_singularity_member(ctx, oracle):
    """A wide group (12 members, member-level rounds) with one member 0.4 km from a planet:
    the group's SingularityError carries the reference's node, trajectory-in-group and body
    (force_model.hpp:115-120), formed from the member records."""
    states, plan, cfg = _setup(12, 16, 0.05, start="cold")
    pos = oracle.body_positions(ps.reference_bodies(), ps.MU_SUN, np.array([0.0]))
    states[7, 1:4] = pos[0, 0] + np.array([0.4, 0.0, 0.0])
    errs = []
    for impl in (ctx, oracle):
        with pytest.raises(ps.SingularityError) as e:
            impl.propagate(states, [12], plan, cfg)
        errs.append(e.value)
    assert str(errs[0]) == str(errs[1]) and errs[0].body == errs[1].body


@pytest.mark.parametrize("n", [64, 96, 128])
@pytest.mark.parametrize("kind", ["n_body", "n_body_1pn"])
@pytest.mark.parametrize("mode,p", [("independent", 1), ("grouped", 5), ("augmented", 1)])
def test_two_ctas_per_sm_variants(ctx, oracle, n, kind, mode, p):
    """The 256-thread slot kernels (4 MMA + 4 FP warps, two CTAs per SM, pswarm_dev::small)
    against the oracle and the 512-thread kernels, for both force models and the group paths.
    (Not bit-identical to them: b0 sums one partial per FP warp, 4 instead of 8; the choice
    depends on N and the force model only, so every grouping and shard still runs one of them.)"""
    states = _mixed_states(40, _NEAR)
    _, plan, cfg = _setup(40, n, 0.6, "planets8")
    cfg.force_kind = kind
    cfg.p_groups = p
    out = {}
    for small in (1, 0):
        ctx.set_option("small_ctas", small)
        ctx.set_option("small_max_n", 256 if small else 0)
        try:
            out[small] = ctx.run_batch(states, cfg, plan, mode)
            out[(small, "k")] = ctx.kernel_name()
        finally:
            ctx.set_option("small_ctas", 1)
            ctx.set_option("small_max_n", 0)
    assert out[(1, "k")].endswith(".x2") and not out[(0, "k")].endswith(".x2")
    want = oracle.run_batch(states, cfg, plan, mode, 4)
    _parity(out[1], want)
    _parity(out[1], out[0], tol=1e-12)
