"""Multi-device run_batch (pswarm_run_batch_multi, SURVEY §8a13 `devices` knob / §8e) on one
B200: several contexts on the same GPU ([0, 0], [0, 0, 0]) exercise the whole path — group-
aligned shards, one host thread per context, the terminal-state gather, the report and
sample assembly, the error selection — and must reproduce the single-context run bit for
bit (the gather uses a device copy when a device repeats; distinct devices use NCCL)."""
import numpy as np
import pytest

import paper_2301_03989_b200 as ps

pytestmark = pytest.mark.gpu


def _case(m=61, n=64, span=1.6, policy="per_orbit", spread=1e-4, bodies=None):
    base = ps.reference_state()
    states = ps.make_clone_batch(base, m, spread)
    period = ps.osculating_period(base, ps.MU_SUN)
    plan = ps.plan_segments(base, 0.0, span * period, ps.MU_SUN, policy, n)
    cfg = ps.reference_force_config("n_body", bodies=bodies or ps.planets8(), n_nodes=n)
    cfg.p_groups = 7
    return states, plan, cfg


@pytest.fixture(scope="module")
def multi2():
    return ps.MultiContext([0, 0])


@pytest.fixture(scope="module")
def multi3():
    return ps.MultiContext([0, 0, 0])


@pytest.mark.parametrize("mode", ["independent", "grouped", "augmented_sequential"])
def test_multi_matches_single_bit_for_bit(ctx, multi2, multi3, mode):
    states, plan, cfg = _case()
    one = ctx.run_batch(states, cfg, plan, mode)
    for mc in (multi2, multi3):
        r = mc.run_batch(states, cfg, plan, mode)
        assert np.array_equal(r.terminal_states, one.terminal_states)
        assert np.array_equal(r.trajectories, one.trajectories)
        assert np.array_equal(r.iterations, one.iterations)
        assert np.array_equal(r.converged, one.converged)
        assert len(r.reports) == len(one.reports)
        for s in range(len(one.reports)):
            for g in range(len(one.reports[s])):
                a, b = one.reports[s][g], r.reports[s][g]
                assert a.final_error == b.final_error and np.array_equal(a.per_iteration_errors,
                                                                         b.per_iteration_errors)


def test_multi_backend_and_more_shards_than_trajectories(ctx):
    mc = ps.MultiContext([0, 0, 0, 0])
    assert mc.backend.startswith("peer-copy")
    states, plan, cfg = _case(m=3, n=32, span=0.5, policy="single")
    r = mc.run_batch(states, cfg, plan, "independent")
    assert np.array_equal(r.terminal_states, ctx.run_batch(states, cfg, plan, "independent").terminal_states)


def test_multi_error_is_the_single_device_error(ctx, multi3):
    """A singular trajectory in the last shard: same exception, message and batch index."""
    states, plan, cfg = _case(m=40, n=48, span=0.5, policy="single")
    bad = states.copy()
    bad[33, 1:4] = 0.0  # zero radius: warm start raises (kepler.hpp)
    with pytest.raises(ps.Error) as e1:
        ctx.run_batch(bad, cfg, plan, "independent")
    with pytest.raises(ps.Error) as e2:
        multi3.run_batch(bad, cfg, plan, "independent")
    assert type(e1.value) is type(e2.value) and str(e1.value) == str(e2.value)


def test_multi_independent_lowest_failing_trajectory(ctx, multi3):
    """Independent mode over three shards: a divergence in shard 2 and a non-convergence of a
    LOWER trajectory in shard 1 -> the error of the lower trajectory, as one device (and the
    serial reference, runner.hpp:63-80) raises it."""
    states, plan, cfg = _case(m=40, n=48, span=0.5, policy="single")
    cfg.start_mode = "cold"
    states[20, 1:] = ps.elements_to_state([0.8e8, 0.3, 0.05, 0.4, 0.9, 0.0, 0.0], ps.MU_SUN, 0.0)[1:]
    ok = ctx.run_batch(np.delete(states, 20, axis=0), cfg, plan, "independent")
    cfg.max_iterations = int(ok.iterations.max()) + 1
    states[35, 1:4] = [1e-110, 0.0, 0.0]
    errs = []
    for impl in (ctx, multi3):
        with pytest.raises(ps.Error) as e:
            impl.run_batch(states, cfg, plan, "independent")
        errs.append(e.value)
    assert type(errs[0]) is type(errs[1]) is ps.PropagationIncompleteError
    assert str(errs[0]) == str(errs[1])
