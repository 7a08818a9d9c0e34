#pragma once
// Embedded verification suite (reference: selftest.hpp:13-166), run on the device
// library: the same options, property names, PASS/FAIL/info lines and negative
// control (a perturbed transform must fail every matrix-contract property).

#include <cmath>
#include <functional>
#include <ostream>
#include <string>
#include <vector>

#include "pswarm/runner.hpp"
#include "pswarm/synthetic.hpp"

namespace pswarm {

struct SelftestOptions {  // selftest.hpp:13-21
    Index n_nodes = 200;
    double tolerance = 1e-12;
    Index batch_size = 64;
    bool perturb_matrices = false;  ///< negative-control hook: corrupt xform(1, 1)
};

namespace detail {

/// Operators for the checks; with `perturb` the transform is corrupted by 1e-6 and the
/// derived operators are rebuilt from it (selftest.hpp:24-35).
inline PCMatrices selftest_matrices(Index n, bool perturb) {
    PCMatrices m = build_matrices(n);
    if (!perturb) return m;
    m.xform(1, 1) += 1e-6;
    m.a_op = m.integ * m.xform;
    m.update_op = m.eval * m.a_op;
    RowVec s_full = RowVec::Zero(n);
    s_full.tail(n - 1) = m.s_row;
    m.anchor_op = s_full * m.a_op;
    return m;
}

inline bool selftest_inversion(const SelftestOptions& o) {
    for (Index n : {Index{8}, Index{64}, o.n_nodes}) {
        const PCMatrices m = selftest_matrices(n, o.perturb_matrices);
        const Vec tau = chebyshev_lobatto_nodes(n);
        Mat t(n, n);
        for (Index j = 0; j < n; ++j) chebyshev_values(tau[j], t.row(j).data(), n);
        if ((t * m.xform - Mat::Identity(n, n)).cwiseAbs().maxCoeff() > 1e-12) return false;
    }
    return true;
}

/// One device Picard update integrates t^d exactly for d <= 10 at N = 16.
inline bool selftest_polynomial(const SelftestOptions& o) {
    const Index n = 16;
    const PCMatrices m = selftest_matrices(n, o.perturb_matrices);
    const ChebyshevGrid g = build_grid(n, 0.0, 2.0);
    for (int d = 0; d <= 10; ++d) {
        Mat f(n, 1);
        for (Index j = 0; j < n; ++j) f(j, 0) = g.omega2 * std::pow(g.times[j], d);
        const Mat y = picard_update(m, f, RowVec::Ones(1));
        for (Index j = 0; j < n; ++j) {
            const double want = 1.0 + std::pow(g.times[j], d + 1) / (d + 1);
            if (!(std::abs(y(j, 0) - want) <= 1e-12 * std::abs(want))) return false;
        }
    }
    return true;
}

inline bool selftest_period_recurrence() {
    for (double e : {0.0, 0.2, 0.5, 0.8}) {
        OrbitalElements el;
        el.a = 1.2e8;
        el.e = e;
        el.i = 0.3 * e;
        el.raan = 0.7;
        el.argp = 1.1;
        el.m0 = 0.4;
        const StateVector s = elements_to_state(el, mu_sun_km3s2, 0.0);
        const StateVector b = kepler_propagate(s, mu_sun_km3s2, osculating_period(s, mu_sun_km3s2));
        if ((b.r - s.r).norm() / s.r.norm() > 1e-11 || (b.v - s.v).norm() / s.v.norm() > 1e-11) return false;
    }
    return true;
}

inline bool selftest_energy() {
    const StateVector s = make_reference_state();
    const double e0 = specific_energy(s, mu_sun_km3s2);
    for (int k = 1; k <= 8; ++k)
        if (std::abs(specific_energy(kepler_propagate(s, mu_sun_km3s2, 2.0e6 * k), mu_sun_km3s2) - e0) >
            1e-11 * std::abs(e0))
            return false;
    return true;
}

}  // namespace detail

/// Prints one PASS/FAIL line per property and returns overall success (selftest.hpp:41-164).
inline bool run_selftest(std::ostream& os, const SelftestOptions& opts = {}) {
    bool all = true;
    auto report = [&](const char* name, bool ok) {
        os << (ok ? "PASS " : "FAIL ") << name << "\n";
        all = all && ok;
    };
    report("matrix-inversion-contract", detail::selftest_inversion(opts));
    report("polynomial-exactness", detail::selftest_polynomial(opts));
    report("kepler-period-recurrence", detail::selftest_period_recurrence());
    report("kepler-energy-consistency", detail::selftest_energy());

    // Grouped propagation of the synthetic batch on the device: 1, 4 and singleton groups
    // agree within the tolerance; warm start needs no more iterations than cold.
    PropagationConfig cfg;
    cfg.n_nodes = opts.n_nodes;
    cfg.tolerance = opts.tolerance;
    cfg.force = make_reference_force_model();
    const auto batch = make_clone_batch(make_reference_state(), opts.batch_size, 1e-5);
    const SegmentPlan plan = plan_segments(batch[0], 0.0, 0.87 * osculating_period(batch[0], mu_sun_km3s2),
                                           mu_sun_km3s2, SegmentPolicy::single, cfg.n_nodes);
    auto grouped = [&](Index groups, StartMode start) {
        PropagationConfig c = cfg;
        c.p_groups = groups;
        c.start_mode = start;
        return run_batch(batch, c, plan, RunMode::grouped, 1);
    };
    const RunOutcome one = grouped(1, StartMode::warm), four = grouped(4, StartMode::warm),
                     single = grouped(opts.batch_size, StartMode::warm);
    report("grouping-invariance", max_state_discrepancy(four.result, one.result) <= opts.tolerance &&
                                      max_state_discrepancy(single.result, one.result) <= opts.tolerance);
    int lo = four.result.reports.at(0).at(0).iterations, hi = lo;
    for (const auto& r : four.result.reports.at(0)) {
        lo = std::min(lo, r.iterations);
        hi = std::max(hi, r.iterations);
    }
    os << "info group iteration counts span [" << lo << ", " << hi << "]\n";
    const RunOutcome cold = grouped(4, StartMode::cold);
    const int warm_it = one.result.max_iterations_used(), cold_it = cold.result.max_iterations_used();
    os << "info warm-start iterations " << warm_it << ", cold-start iterations " << cold_it << "\n";
    report("warm-start-benefit", warm_it <= cold_it && one.result.reports.at(0).at(0).converged &&
                                     cold.result.reports.at(0).at(0).converged);
    os << (all ? "selftest: all properties passed" : "selftest: FAILURES detected") << "\n";
    return all;
}

}  // namespace pswarm
