"""Small propagations through every solve kernel for compute-sanitizer (diagnostics)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2301_03989_b200 as ps

ctx = ps.Context(0)
base = ps.reference_state()
period = ps.osculating_period(base, ps.MU_SUN)
states = ps.make_clone_batch(base, 24, 1e-5)
other = ps.elements_to_state([1.15e8, 0.2, 0.05, 0.4, 0.9, 0.0, 0.0], ps.MU_SUN, 0.0)
states[1::3, 1:] = other[1:]  # mixed members: wide groups need resume rounds
# (N, mode, p_groups, force kind, start, options)
CASES = [(200, "independent", 1, "n_body", "warm", {}),                      # k_pc_ws_fold, extra units, b0 by the FP group
         (160, "independent", 1, "n_body", "warm", {}),                      # k_pc_ws_fold, 6 extra units
         (256, "independent", 1, "n_body", "warm", {}),                      # k_pc_ws_fold, no extras
         (200, "independent", 1, "n_body", "warm", {"fold": 0}),             # dense k_pc_ws
         (200, "independent", 1, "n_body", "warm", {"unified": 1}),          # k_pc_uni Newtonian
         (96, "independent", 1, "n_body_1pn", "warm", {}),                   # k_pc_uni 1PN (auto)
         (256, "independent", 1, "n_body_1pn", "warm", {"unified": 0}),     # k_pc_ws_fold 1PN
         (64, "grouped", 4, "n_body", "warm", {}),                           # grouped, folded kernels
         (216, "independent", 1, "n_body", "warm", {}),                      # k_pc_ws_fold, no extras, b0 from DMMA
         (55, "independent", 1, "n_body", "warm", {"slot_kernel": 1}),       # generic small-N, 23 staged rows
         (241, "augmented", 1, "n_body", "warm", {}),                        # wide rounds on k_pc_segment (32 m-tiles)
         (72, "grouped", 4, "n_body", "warm", {}),                           # groups of 6 -> wide rounds on k_pc_ws_fold
         (64, "augmented", 1, "n_body", "warm", {}),                         # wide rounds on k_pc_ws_fold (resume)
         (64, "independent", 1, "n_body_1pn", "warm", {}),                   # k_pc_uni, 1PN table bulk-staged
         (64, "independent", 1, "n_body", "hot", {}),                        # hot start, multi-segment
         (96, "grouped", 4, "n_body", "warm", {}),                           # k_pc_uni.x2 Newtonian (two CTAs per SM)
         (104, "independent", 1, "n_body", "warm", {}),                      # k_pc_ws_fold.x2, two-slot items
         (72, "independent", 1, "n_body", "warm", {}),                       # k_pc_ws_fold.x2, single-slot items
         (128, "independent", 1, "n_body", "warm", {}),                      # k_pc_uni.x2 Newtonian
         (160, "independent", 1, "n_body_1pn", "warm", {}),                  # k_pc_uni 1PN, single-slot items
         (128, "augmented", 1, "n_body_1pn", "warm", {})]                    # k_pc_uni.x2, wide rounds
for n, mode, p, kind, start, opts in CASES:
    plan = ps.plan_segments(base, 0.0, (2.2 if start == "hot" else 0.4) * period, ps.MU_SUN,
                            "per_orbit" if start == "hot" else "single", n)
    cfg = ps.reference_force_config(kind, bodies=ps.planets8(), n_nodes=n, start_mode=start)
    cfg.p_groups = p
    for k, v in opts.items():
        ctx.set_option(k, v)
    r = ctx.run_batch(states, cfg, plan, mode)
    print(n, mode, kind, start, opts, ctx.kernel_name(), int(r.iterations.sum()), flush=True)
    ctx.set_option("fold", 1)
    ctx.set_option("unified", 2)
    ctx.set_option("slot_kernel", 0)
