// Pins for the oracle's EXTENSIONS beyond the reference (TEST INFRASTRUCTURE ONLY):
// the relativistic n_body_1pn force model and the hot start (BASELINE configs 3 and 5).
// The reference has neither, so no reference vector exists;
// these cases tie the restatement to closed forms and to an independent integrator:
//   * Sun-only EIH == the Schwarzschild (PPN beta = gamma = 1) test-particle term;
//   * the relativistic perihelion advance 6 pi mu / (c^2 a (1 - e^2)) per orbit;
//   * PC (fixed point) vs RKF7(8) on the same 1PN N-body law <= 1e-9 (acceptance.cpp
//     criterion 3's bar);
//   * Chebyshev derivative (body velocities of tabulated ephemerides) vs the analytic conic;
//   * hot start converges to the same fixed point as the warm start.
// Output format as kat_tests.cpp ("PASS"/"FAIL" lines, "SUMMARY p f").

#include <cstdio>
#include <cstring>
#include <numbers>
#include <string>

#include "pswarm_ref.hpp"

using namespace pswarm_ref;

namespace {

int g_pass = 0, g_fail = 0;
std::string g_detail;

void expect(bool ok, const std::string& what) {
    if (!ok && g_detail.empty()) g_detail = what;
}

template <typename Fn>
void run_case(const char* name, Fn&& fn) {
    g_detail.clear();
    try {
        fn();
    } catch (const std::exception& e) {
        g_detail = std::string("unexpected exception: ") + e.what();
    }
    if (g_detail.empty()) {
        ++g_pass;
        std::printf("PASS %s\n", name);
    } else {
        ++g_fail;
        std::printf("FAIL %s: %s\n", name, g_detail.c_str());
    }
    std::fflush(stdout);
}

std::string fmt(double x) {
    char b[64];
    std::snprintf(b, sizeof b, "%.3e", x);
    return b;
}

Config rel_config(Index n, bool with_bodies) {
    Config c;
    c.n_nodes = n;
    c.force.kind = ForceKind::n_body_1pn;
    c.force.central_mu = mu_sun;
    if (with_bodies) c.force.bodies = reference_bodies();
    return c;
}

V3 ecc_vector(V3 r, V3 v, double mu) {
    const double rn = r.norm();
    return (1.0 / mu) * ((dot(v, v) - mu / rn) * r - dot(r, v) * v);
}

}  // namespace

int main() {
    constexpr double c_light = 299792.458;
    run_case("eih_sun_only_is_schwarzschild", [] {
        const State s = reference_state();
        RelBodies none;
        const V3 got = eih_correction(s.r, s.v, none, mu_sun, c_light);
        const double r = s.r.norm(), c2 = c_light * c_light;
        const V3 want = (mu_sun / (c2 * r * r * r)) *
                        ((4.0 * mu_sun / r - dot(s.v, s.v)) * s.r + 4.0 * dot(s.r, s.v) * s.v);
        expect((got - want).norm() <= 1e-13 * want.norm(), "rel " + fmt((got - want).norm() / want.norm()));
    });
    run_case("chebyshev_velocity_matches_conic", [] {
        const Body earth = reference_bodies()[1];
        const double t0 = 0.0, t1 = 30.0 * 86400.0;
        ChebSeg seg = fit_segment([&](double t) { return elements_to_state(earth.el, mu_sun, t).r; }, t0, t1, 24);
        double worst = 0.0;
        for (int k = 0; k <= 10; ++k) {
            const double t = t0 + (t1 - t0) * k / 10.0;
            const V3 want = elements_to_state(earth.el, mu_sun, t).v;
            worst = std::max(worst, (seg.velocity_at(t) - want).norm() / want.norm());
        }
        expect(worst <= 1e-9, "velocity rel " + fmt(worst));
    });
    run_case("perihelion_advance_per_orbit", [] {
        // 10 osculating periods from perihelion, per-orbit segments, Sun-only 1PN
        const State s = reference_state();
        const double period = osculating_period(s, mu_sun);
        const int orbits = 10;
        const Segments sp = plan_segments(s, 0.0, orbits * period, mu_sun, SegmentPolicy::per_orbit, 200, 1.0);
        const Config cfg = rel_config(200, false);
        const auto out = run_batch({s}, cfg, sp, RunMode::independent, 1);
        const State& e = out.result.terminal_states[0];
        const V3 e0 = ecc_vector(s.r, s.v, mu_sun), e1 = ecc_vector(e.r, e.v, mu_sun);
        const V3 h = cross(s.r, s.v);
        const double ang = std::atan2(dot(cross(e0, e1), h) / h.norm(), dot(e0, e1));
        const double a = 1.25e8, ecc = 0.12;
        const double want = orbits * 6.0 * std::numbers::pi * mu_sun / (c_light * c_light * a * (1.0 - ecc * ecc));
        expect(std::abs(ang - want) <= 0.03 * want, "advance " + fmt(ang) + " want " + fmt(want));
    });
    run_case("pc_vs_rkf78_1pn_nbody", [] {  // acceptance.cpp:148-172 bar on the extension
        const auto st = clone_batch(reference_state(), 8, 1e-5);
        const Config cfg = rel_config(200, true);
        const double period = osculating_period(st[0], mu_sun);
        const Segments sp = plan_segments(st[0], 0.0, 0.87 * period, mu_sun, SegmentPolicy::single, 200);
        const auto out = run_batch(st, cfg, sp, RunMode::independent, 1);
        double worst = 0.0;
        for (std::size_t i = 0; i < st.size(); ++i)
            worst = std::max(worst, compare_trajectories(out.result.trajectories[i],
                                                         rk_sample(st[i], nbody_deriv(cfg.force), out.result.times)));
        expect(worst <= 1e-9, "pc vs rkf78 " + fmt(worst));
    });
    run_case("relativistic_effect_is_resolved", [] {
        const auto st = clone_batch(reference_state(), 4, 1e-5);
        Config rel = rel_config(200, true), newt = rel;
        newt.force.kind = ForceKind::n_body;
        const double period = osculating_period(st[0], mu_sun);
        const Segments sp = plan_segments(st[0], 0.0, 0.87 * period, mu_sun, SegmentPolicy::single, 200);
        const auto a = run_batch(st, rel, sp, RunMode::independent, 1);
        const auto b = run_batch(st, newt, sp, RunMode::independent, 1);
        const double d = max_state_discrepancy(a.result, b.result);
        expect(d > 1e-9 && d < 1e-5, "1PN - Newtonian " + fmt(d));
    });
    run_case("hot_start_same_fixed_point", [] {
        const auto st = clone_batch(reference_state(), 16, 1e-5);
        const double period = osculating_period(st[0], mu_sun);
        const Segments sp = plan_segments(st[0], 0.0, 3.0 * period, mu_sun, SegmentPolicy::per_orbit, 200, 1.0);
        Config warm = rel_config(200, true), hot = warm;
        warm.force.kind = hot.force.kind = ForceKind::n_body;
        hot.start_mode = StartMode::hot;
        const auto w = run_batch(st, warm, sp, RunMode::independent, 1);
        const auto h = run_batch(st, hot, sp, RunMode::independent, 1);
        const double d = max_state_discrepancy(h.result, w.result);
        long iw = 0, ih = 0;
        for (std::size_t seg = 1; seg < w.result.reports.size(); ++seg)
            for (std::size_t g = 0; g < w.result.reports[seg].size(); ++g) {
                iw += w.result.reports[seg][g].iterations;
                ih += h.result.reports[seg][g].iterations;
            }
        std::printf("  hot start: segments>=1 iterations warm %ld hot %ld, discrepancy %s\n", iw, ih, fmt(d).c_str());
        expect(d <= 1e-10, "hot vs warm " + fmt(d));
        expect(h.result.reports[0][0].iterations == w.result.reports[0][0].iterations, "segment 0 must be warm");
    });
    run_case("hot_start_periodic_correction_pays", [] {
        // Sun-only 1PN: the correction is periodic with the orbit, so the previous orbit's
        // (converged - conic) difference is an almost exact guess
        const auto st = clone_batch(reference_state(), 4, 1e-5);
        const double period = osculating_period(st[0], mu_sun);
        const Segments sp = plan_segments(st[0], 0.0, 3.0 * period, mu_sun, SegmentPolicy::per_orbit, 200, 1.0);
        Config warm = rel_config(200, false), hot = warm;
        hot.start_mode = StartMode::hot;
        const auto w = run_batch(st, warm, sp, RunMode::independent, 1);
        const auto h = run_batch(st, hot, sp, RunMode::independent, 1);
        int iw = 0, ih = 0;
        for (std::size_t g = 0; g < st.size(); ++g) {
            iw += w.result.reports[2][g].iterations;
            ih += h.result.reports[2][g].iterations;
        }
        std::printf("  hot start (Sun-only 1PN): segment 2 iterations warm %d hot %d\n", iw, ih);
        expect(10 * ih < 7 * iw, "hot " + std::to_string(ih) + " warm " + std::to_string(iw));
        expect(max_state_discrepancy(h.result, w.result) <= 1e-10, "fixed point");
    });
    std::printf("SUMMARY %d %d\n", g_pass, g_fail);
    return g_fail == 0 ? 0 : 1;
}
