"""Regenerate the golden fixtures from the CPU oracle (oracle/pswarm_ref.hpp, pinned to the
reference's KATs).  TEST INFRASTRUCTURE: run here, commit the .npz files; the GPU box
only reads them.

    python tests/golden/make_golden.py

Each fixture stores the inputs' recipe (seeded clone cloud, so the ICs are regenerated
bit-exactly by make_clone_batch), the oracle's terminal states [M][7], per-(segment, group)
iteration counts, and a strided subset of node samples."""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import paper_2301_03989_b200 as ps  # noqa: E402
from oracle.oracle_py import Oracle  # noqa: E402

# name: (base, M, spread, span periods, policy, N, force kind, bodies, start)
CASES = {
    "c1_two_body": ("c1", 64, 1e-5, 1.0, "single", 200, "two_body", "none", "cold"),
    "c2_planets8": ("ref", 64, 1e-5, 0.87, "single", 200, "n_body", "planets8", "warm"),
    "c3_multiseg_hot": ("ref", 16, 1e-5, 2.5, "per_orbit", 128, "n_body", "reference", "hot"),
    "c5_1pn_n96": ("ref", 16, 1e-3, 0.87, "single", 96, "n_body_1pn", "planets8", "warm"),
}


def setup(case):
    base_kind, m, spread, span, policy, n, kind, bodies, start = CASES[case]
    if base_kind == "c1":
        base = ps.elements_to_state([1.3e8, 0.2, 0.05, 0.4, 0.9, 0.0, 0.0], ps.MU_SUN, 0.0)
    else:
        base = ps.reference_state()
    states = ps.make_clone_batch(base, m, spread)
    period = ps.osculating_period(base, ps.MU_SUN)
    plan = ps.plan_segments(base, 0.0, span * period, ps.MU_SUN, policy, n)
    blist = {"none": list, "reference": ps.reference_bodies, "planets8": ps.planets8}[bodies]()
    cfg = ps.reference_force_config(kind, bodies=blist, n_nodes=n, start_mode=start)
    return states, plan, cfg


def main():
    orc = Oracle()
    for case in CASES:
        states, plan, cfg = setup(case)
        r = orc.run_batch(states, cfg, plan, "independent", 8)
        rows = np.arange(0, r.trajectories.shape[1], 7)
        np.savez_compressed(os.path.join(HERE, f"{case}.npz"), states=states, boundaries=plan.boundaries,
                            terminal=r.terminal_states, iterations=r.iterations, sample_rows=rows,
                            samples=r.trajectories[:, rows, :])
        print(case, r.terminal_states.shape, int(r.iterations.sum()))


if __name__ == "__main__":
    main()
