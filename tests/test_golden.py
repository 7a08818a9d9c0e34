"""Golden fixtures (tests/golden/*.npz, written by tests/golden/make_golden.py from the
pinned CPU oracle): the oracle must keep reproducing them bit for bit (CPU), and the
device path must match them within the north-star bars without running the oracle
(GPU: 1e-10 relative on node samples and terminal states, iterations +-1)."""
import os
import sys

import numpy as np
import pytest

import paper_2301_03989_b200 as ps

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
sys.path.insert(0, HERE)
from make_golden import CASES, setup  # noqa: E402


def _load(case):
    return np.load(os.path.join(HERE, f"{case}.npz"))


@pytest.mark.parametrize("case", sorted(CASES))
def test_fixture_inputs_regenerate_bit_exact(case):
    g = _load(case)
    states, plan, _ = setup(case)
    assert np.array_equal(states, g["states"])
    assert np.array_equal(plan.boundaries, g["boundaries"])


@pytest.mark.parametrize("case", sorted(CASES))
def test_oracle_reproduces_fixture(oracle, case):
    g = _load(case)
    states, plan, cfg = setup(case)
    r = oracle.run_batch(states, cfg, plan, "independent", 4)
    assert np.array_equal(r.terminal_states, g["terminal"])
    assert np.array_equal(r.iterations, g["iterations"])


@pytest.mark.gpu
@pytest.mark.parametrize("case", sorted(CASES))
def test_device_matches_fixture(ctx, case):
    g = _load(case)
    states, plan, cfg = setup(case)
    r = ctx.run_batch(states, cfg, plan, "independent")
    rows = g["sample_rows"]
    assert ps.max_state_discrepancy(r.trajectories[:, rows, :], g["samples"]) <= 1e-10
    assert ps.max_state_discrepancy(r.terminal_states[None, :, 1:], g["terminal"][None, :, 1:]) <= 1e-10
    assert np.array_equal(r.terminal_states[:, 0], g["terminal"][:, 0])
    assert int(np.abs(r.iterations.astype(int) - g["iterations"].astype(int)).max()) <= 1
