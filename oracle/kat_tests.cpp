// Known-answer and property suite that PINS the CPU oracle (oracle/pswarm_ref.hpp)
// to the reference's own test expectations.  TEST INFRASTRUCTURE ONLY.
//
// Every case restates a check the reference holds in proj/tests/*.cpp or
// proj/tests/acceptance.cpp (cited per case); tolerances are the reference's.
// The reference cannot be compiled here (no Eigen), so these KATs are what
// ties the oracle to the reference's behaviour.
//
// Output: one "PASS <name>" / "FAIL <name>: <detail>" line per case, then
// "SUMMARY <passed> <failed>"; exit status 1 when anything failed.
// Usage: kat_tests [--quick]   (--quick skips the multi-second acceptance runs)

#include <cstdio>
#include <cstring>
#include <random>
#include <sstream>

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

template <typename E, typename Fn>
bool throws(Fn&& fn) {
    try {
        fn();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

bool close_rel(double got, double want, double eps) {  // doctest::Approx semantics
    return std::abs(got - want) <= eps * (1.0 + std::max(std::abs(got), std::abs(want))) ||
           std::abs(got - want) <= eps * std::max(std::abs(got), std::abs(want));
}

std::string fmt(double v) {
    char b[64];
    std::snprintf(b, sizeof b, "%.6e", v);
    return b;
}


double max_abs_diff(const Mat& a, const Mat& b) {
    double w = 0.0;
    for (std::size_t i = 0; i < a.v.size(); ++i) w = std::max(w, std::abs(a.v[i] - b.v[i]));
    return w;
}

double abs_err_fn(const Mat& c, const Mat& p) { return max_abs_diff(c, p); }

State make_state(V3 r, V3 v, double epoch = 0.0) {
    State s;
    s.epoch = epoch;
    s.r = r;
    s.v = v;
    return s;
}

double rel_state(const State& a, const State& b) {
    return std::max((a.r - b.r).norm() / b.r.norm(), (a.v - b.v).norm() / b.v.norm());
}

auto two_body_deriv(double mu) {
    return [mu](double, const S6& y) {
        const V3 r{y[0], y[1], y[2]};
        const double rn = r.norm();
        const V3 a = (-mu / (rn * rn * rn)) * r;
        return S6{y[3], y[4], y[5], a.x, a.y, a.z};
    };
}

Config nbody_config(Index n) {
    Config c;
    c.n_nodes = n;
    c.force = reference_force();
    return c;
}

Config twobody_config(Index n) {
    Config c;
    c.n_nodes = n;
    c.force = reference_force(ForceKind::two_body);
    return c;
}

}  // namespace

// ---------------------------------------------------------------- chebyshev
static void chebyshev_cases() {
    run_case("grid_three_nodes", [] {  // test_chebyshev.cpp:25-35
        const Grid g = build_grid(3, 0.0, 10.0);
        expect(g.tau[0] == -1.0 && g.tau[1] == 0.0 && g.tau[2] == 1.0, "tau");
        expect(g.times[0] == 0.0 && g.times[1] == 5.0 && g.times[2] == 10.0, "times");
        expect(g.omega1 == 5.0 && g.omega2 == 5.0, "omega");
    });
    run_case("grid_interior_closed_form", [] {  // :37-42
        const Grid g = build_grid(5, 0.0, 1.0);
        expect(close_rel(g.tau[1], -std::cos(std::numbers::pi / 4), 1e-15), "tau[1]");
        expect(g.omega1 == 0.5 && g.omega2 == 0.5, "omega");
    });
    run_case("grid_200_reference_segment", [] {  // :44-61
        const double t0 = 6.64e8, span = 0.87 * 2.2e7;
        const Grid g = build_grid(200, t0, t0 + span);
        expect(g.times[0] == t0 && g.times[199] == t0 + span, "pinned endpoints");
        for (Index j = 0; j < 200; ++j) {
            expect(std::abs(g.tau[j] - (-std::cos(static_cast<double>(j) * std::numbers::pi / 199.0))) <= 1e-15,
                   "node closed form");
            if (j > 0) expect(g.tau[j] > g.tau[j - 1], "monotone");
            if (j > 0 && j < 199) expect(g.times[j] == g.omega2 * g.tau[j] + g.omega1, "interior mapping");
        }
    });
    run_case("grid_node_symmetry_exact", [] {  // :63-70
        for (Index n : {3, 4, 16, 17, 200, 300}) {
            const auto tau = lobatto_nodes(n);
            for (Index j = 0; j < n; ++j) expect(tau[j] == -tau[n - 1 - j], "mirror n=" + std::to_string(n));
        }
    });
    run_case("grid_backward_span", [] {  // :72-78
        const Grid g = build_grid(4, 10.0, 2.0);
        expect(g.omega2 == -4.0 && g.times[0] == 10.0 && g.times[3] == 2.0 && g.times[1] > g.times[2], "backward");
    });
    run_case("grid_error_cases", [] {  // :80-84
        expect(throws<InvalidSizeError>([] { build_grid(2, 0.0, 1.0); }), "size");
        expect(throws<InvalidSpanError>([] { build_grid(10, 3.0, 3.0); }), "span");
        expect(throws<InvalidSizeError>([] { build_ops(2); }), "ops size");
    });
    run_case("ops_transform_inverts_interpolation", [] {  // :86-93, acceptance.cpp:37-52
        for (Index n : {3, 8, 16, 64, 200, 300}) {
            const Ops o = build_ops(n);
            const auto tau = lobatto_nodes(n);
            Mat plain(n, n);
            for (Index j = 0; j < n; ++j) cheb_values(tau[j], plain.row(j), n);
            const Mat prod = matmul(plain, o.xform);
            double worst = 0.0;
            for (Index i = 0; i < n; ++i)
                for (Index j = 0; j < n; ++j) worst = std::max(worst, std::abs(prod(i, j) - (i == j ? 1.0 : 0.0)));
            expect(worst <= (n == 3 ? 1e-14 : 1e-12), "residual " + fmt(worst) + " n=" + std::to_string(n));
        }
    });
    run_case("ops_structure", [] {  // :95-113
        const Ops o = build_ops(16);
        expect(o.eval.all_finite() && o.xform.all_finite() && o.integ.all_finite() && o.a_op.all_finite(), "finite");
        for (Index k = 0; k < 16; ++k) expect(o.integ(0, k) == 0.0 && o.a_op(0, k) == 0.0, "row 0 zero");
        for (Index j = 0; j < 16; ++j) expect(o.eval(j, 0) == 0.5, "half column");
        expect(o.s_row[0] == 2.0 && o.s_row[1] == -2.0 && o.s_row[14] == 2.0, "s_row");
    });
    run_case("ops_constant_integrand_ramp", [] {  // :115-137
        const Index n = 6;
        const Ops o = build_ops(n);
        const auto tau = lobatto_nodes(n);
        const double c = 1.75, y0 = -0.4;
        Mat f(n, 1, c);
        std::vector<double> coeffs(n, 0.0);
        for (Index k = 0; k < n; ++k)
            for (Index j = 0; j < n; ++j) coeffs[k] += o.xform(k, j) * c;
        expect(close_rel(coeffs[0], c, 1e-14), "c0");
        for (Index k = 1; k < n; ++k) expect(std::abs(coeffs[k]) <= 1e-14, "tail coeffs");
        double anti1 = 0.0;
        for (Index k = 0; k < n; ++k) anti1 += o.integ(1, k) * coeffs[k];
        expect(close_rel(anti1, c, 1e-14), "anti(1)");
        Mat y;
        picard_update_into(o, f, {y0}, y);
        for (Index j = 0; j < n; ++j) expect(close_rel(y(j, 0), y0 + c * (tau[j] + 1.0), 1e-14), "ramp");
    });
    run_case("ops_cubic_to_quartic", [] {  // :139-152
        const Index n = 8;
        const Ops o = build_ops(n);
        const auto tau = lobatto_nodes(n);
        Mat f(n, 1);
        for (Index j = 0; j < n; ++j) f(j, 0) = tau[j] * tau[j] * tau[j];
        Mat y;
        picard_update_into(o, f, {2.0}, y);
        for (Index j = 0; j < n; ++j)
            expect(close_rel(y(j, 0), 2.0 + (std::pow(tau[j], 4) - 1.0) / 4.0, 1e-13), "quartic");
    });
    run_case("ops_cache_one_instance_per_n", [] {  // :154-160
        expect(cached_ops(21).get() == cached_ops(21).get() && cached_ops(21).get() != cached_ops(22).get(), "cache");
    });
}

// ------------------------------------------------------------------- picard
static void picard_cases() {
    run_case("update_zero_force_keeps_initial_row", [] {  // test_picard.cpp:10-20
        const Index n = 9;
        const Ops o = build_ops(n);
        const std::vector<double> init{1.0, -2.0, 3.0, 0.5, 0.0, -7.25};
        Mat y;
        picard_update_into(o, Mat(n, 6), init, y);
        for (Index j = 0; j < n; ++j)
            for (Index c = 0; c < 6; ++c) expect(close_rel(y(j, c), init[c], 1e-15), "row");
    });
    run_case("update_constant_acceleration", [] {  // :22-54
        const Index n = 12;
        const double t0 = 100.0, dt = 50.0;
        const Grid g = build_grid(n, t0, t0 + dt);
        const Ops o = build_ops(n);
        const double a0[3] = {3e-3, -1e-3, 2e-4}, r0[3] = {10.0, 20.0, 30.0};
        std::vector<double> init{r0[0], r0[1], r0[2], 0.0, 0.0, 0.0};
        Mat f(n, 6);
        for (Index j = 0; j < n; ++j)
            for (int c = 0; c < 3; ++c) {
                f(j, c) = g.omega2 * a0[c] * (g.times[j] - t0);
                f(j, 3 + c) = g.omega2 * a0[c];
            }
        Mat y;
        picard_update_into(o, f, init, y);
        for (Index j = 1; j < n; ++j) {
            const double d = g.times[j] - t0;
            for (int c = 0; c < 3; ++c) {
                expect(close_rel(y(j, 3 + c), a0[c] * d, 1e-12), "velocity");
                expect(close_rel(y(j, c), r0[c] + 0.5 * a0[c] * d * d, 1e-12), "position");
            }
        }
    });
    run_case("update_ramp_integrand", [] {  // :56-70
        const Index n = 10;
        const Grid g = build_grid(n, 0.0, 1.0);
        const Ops o = build_ops(n);
        Mat f(n, 1);
        for (Index j = 0; j < n; ++j) f(j, 0) = g.omega2 * g.times[j];
        Mat y;
        picard_update_into(o, f, {0.0}, y);
        for (Index j = 1; j < n; ++j) expect(close_rel(y(j, 0), 0.5 * g.times[j] * g.times[j], 1e-13), "t^2/2");
    });
    run_case("update_polynomial_exactness_deg0_10", [] {  // :72-89, acceptance.cpp:54-68
        const Index n = 16;
        const Grid g = build_grid(n, 0.0, 2.0);
        const Ops o = build_ops(n);
        double worst = 0.0;
        for (int d = 0; d <= 10; ++d) {
            Mat f(n, 1);
            for (Index j = 0; j < n; ++j) f(j, 0) = g.omega2 * std::pow(g.times[j], d);
            Mat y;
            picard_update_into(o, f, {1.0}, y);
            for (Index j = 0; j < n; ++j) {
                const double e = 1.0 + std::pow(g.times[j], d + 1) / (d + 1);
                worst = std::max(worst, std::abs(y(j, 0) - e) / std::abs(e));
            }
        }
        expect(worst <= 1e-12, "exactness " + fmt(worst));
    });
    run_case("update_anchor_and_literal_chain", [] {  // :91-120
        const Index n = 24;
        const Ops o = build_ops(n);
        std::mt19937 rng(42);
        std::uniform_real_distribution<double> dist(-3.0, 3.0);
        Mat f(n, 6);
        std::vector<double> init(6);
        for (auto& x : f.v) x = dist(rng);
        for (auto& x : init) x = 10.0 * dist(rng);
        Mat y;
        picard_update_into(o, f, init, y);
        for (Index c = 0; c < 6; ++c)
            expect(std::abs(y(0, c) - init[c]) <= 1e-13 * std::max(1.0, std::abs(init[c])), "anchor row");
        Mat b = matmul(o.a_op, f);
        for (Index c = 0; c < 6; ++c) {
            double s = 0.0;
            for (Index k = 1; k < n; ++k) s += o.s_row[k - 1] * b(k, c);
            b(0, c) = s + 2.0 * init[c];
        }
        const Mat yref = matmul(o.eval, b);
        double scale = 0.0;
        for (double x : yref.v) scale = std::max(scale, std::abs(x));
        expect(max_abs_diff(y, yref) / scale <= 1e-13, "literal chain");
    });
    run_case("update_shape_errors", [] {  // :122-126
        const Ops o = build_ops(5);
        Mat out;
        expect(throws<ShapeError>([&] { picard_update_into(o, Mat(4, 6), std::vector<double>(6), out); }), "rows");
        expect(throws<ShapeError>([&] { picard_update_into(o, Mat(5, 6), std::vector<double>(5), out); }), "cols");
    });
    run_case("pc_solve_exponential_decay", [] {  // :137-153
        const Index n = 32;
        const Grid g = build_grid(n, 0.0, 1.0);
        const Ops o = build_ops(n);
        auto dyn = [&](const Mat& y, Mat& f) {
            f = y;
            for (auto& x : f.v) x *= -g.omega2;
        };
        auto [y, rep] = pc_solve(o, dyn, Mat(n, 1, 1.0), {1.0}, 1e-14, 100, abs_err_fn);
        expect(rep.converged && rep.final_error <= 1e-14, "converged");
        expect(rep.iterations == static_cast<int>(rep.history.size()), "history length");
        for (Index j = 0; j < n; ++j) expect(close_rel(y(j, 0), std::exp(-g.times[j]), 1e-13), "exp");
    });
    run_case("pc_solve_nonconvergence_reported", [] {  // :155-165
        const Index n = 16;
        const Grid g = build_grid(n, 0.0, 1.0);
        const Ops o = build_ops(n);
        auto dyn = [&](const Mat& y, Mat& f) {
            f = y;
            for (auto& x : f.v) x *= -g.omega2;
        };
        auto [y, rep] = pc_solve(o, dyn, Mat(n, 1, 1.0), {1.0}, 1e-14, 2, abs_err_fn);
        expect(!rep.converged && rep.iterations == 2, "two iterations, not converged");
    });
    run_case("pc_solve_divergence_coordinates", [] {  // :167-182
        const Ops o = build_ops(8);
        auto dyn = [&](const Mat& y, Mat& f) {
            f = y;
            f(3, 0) = std::numeric_limits<double>::quiet_NaN();
        };
        try {
            pc_solve(o, dyn, Mat(8, 1, 1.0), {1.0}, 1e-12, 10, abs_err_fn);
            expect(false, "no throw");
        } catch (const DivergenceError& e) {
            expect(e.column == 0, "column");
        }
    });
    run_case("pc_solve_bit_identical_reruns", [] {  // :184-196
        const Index n = 20;
        const Grid g = build_grid(n, 0.0, 2.0);
        const Ops o = build_ops(n);
        auto dyn = [&](const Mat& y, Mat& f) {
            f = y;
            for (auto& x : f.v) x = g.omega2 * (x * (1.0 - x));
        };
        auto [y1, r1] = pc_solve(o, dyn, Mat(n, 1, 0.5), {0.5}, 1e-13, 50, abs_err_fn);
        auto [y2, r2] = pc_solve(o, dyn, Mat(n, 1, 0.5), {0.5}, 1e-13, 50, abs_err_fn);
        expect(r1.iterations == r2.iterations && y1.v == y2.v, "bitwise");
    });
}

// ------------------------------------------------------------------- kepler
static void kepler_cases() {
    run_case("solve_kepler_forward_equation", [] {  // test_kepler.cpp:9-19
        for (double e : {0.0, 0.1, 0.5, 0.9, 0.99})
            for (double et : {-2.5, -0.3, 0.0, 0.7, 1.9, 3.0}) {
                const double m = et - e * std::sin(et);
                const double s = solve_kepler(m, e);
                expect(std::abs(s - e * std::sin(s) - m) <= 1e-13, "residual");
                expect(close_rel(s, et, 1e-11), "anomaly");
            }
    });
    run_case("solve_kepler_multi_rev_branch", [] {  // :21-26
        const double e = 0.4, et = 0.9 + 6.0 * std::numbers::pi;
        expect(close_rel(solve_kepler(et - e * std::sin(et), e), et, 1e-12), "branch");
    });
    run_case("kepler_circular_half_full_period", [] {  // :28-40
        const State s = make_state({1, 0, 0}, {0, 1, 0});
        const State h = kepler_propagate(s, 1.0, std::numbers::pi);
        expect((h.r - V3{-1, 0, 0}).norm() <= 1e-12 && (h.v - V3{0, -1, 0}).norm() <= 1e-12, "half");
        const State f = kepler_propagate(s, 1.0, 2.0 * std::numbers::pi);
        expect((f.r - s.r).norm() <= 1e-12 && (f.v - s.v).norm() <= 1e-12, "full");
    });
    run_case("kepler_period_recurrence", [] {  // :42-47
        const State s = reference_state();
        expect(rel_state(kepler_propagate(s, mu_sun, osculating_period(s, mu_sun)), s) <= 1e-11, "recurrence");
    });
    run_case("kepler_matches_rk", [] {  // :49-70
        const State s = make_state({0.5, 0, 0}, {0, std::sqrt(3.0), 0});
        expect(close_rel(specific_energy(s, 1.0), -0.5, 1e-14), "energy");
        RkConfig cfg;
        cfg.rel_tol = 1e-13;
        cfg.abs_tol = 1e-15;
        const State num = rk_propagate(s, two_body_deriv(1.0), 1.0, cfg);
        const State ana = kepler_propagate(s, 1.0, 1.0);
        expect((num.r - ana.r).norm() <= 1e-12 && (num.v - ana.v).norm() <= 1e-12, "rk vs conic");
    });
    run_case("kepler_backward_returns", [] {  // :72-77
        const State s = reference_state();
        const State there = kepler_propagate(s, mu_sun, 3.0e6);
        expect(rel_state(kepler_propagate(there, mu_sun, -3.0e6), s) <= 1e-12, "home");
    });
    run_case("kepler_rejects_unbound", [] {  // :79-92
        const State hyper = make_state({1.0e8, 0, 0}, {0, 60.0, 0});
        expect(specific_energy(hyper, mu_sun) > 0.0, "energy");
        expect(throws<NonEllipticError>([&] { kepler_propagate(hyper, mu_sun, 100.0); }), "hyper");
        expect(throws<NonEllipticError>([&] { osculating_period(hyper, mu_sun); }), "period");
        const State para = make_state({1.0e8, 0, 0}, {0, std::sqrt(2.0 * mu_sun / 1.0e8), 0});
        expect(throws<NonEllipticError>([&] { kepler_propagate(para, mu_sun, 100.0); }), "parabolic");
    });
    run_case("kepler_dt_zero_identity", [] {  // :94-100
        const State s = reference_state();
        const State t = kepler_propagate(s, mu_sun, 0.0);
        expect(t.r.x == s.r.x && t.r.y == s.r.y && t.r.z == s.r.z && t.v.x == s.v.x && t.v.y == s.v.y &&
                   t.v.z == s.v.z && t.epoch == s.epoch,
               "identity");
    });
    run_case("elements_periapsis_and_energy", [] {  // :102-123
        const Elements el{1.3e8, 0.2, 0.1, 0.5, 1.2, 0.0, 0.0};
        const State s = elements_to_state(el, mu_sun, 0.0);
        expect(close_rel(s.r.norm(), el.a * (1.0 - el.e), 1e-13), "periapsis");
        expect(close_rel(specific_energy(s, mu_sun), -mu_sun / (2.0 * el.a), 1e-13), "energy");
        expect(rel_state(elements_to_state(el, mu_sun, 5.0e6), kepler_propagate(s, mu_sun, 5.0e6)) <= 1e-11, "agree");
    });
    run_case("elements_reject_unbound", [] {  // :125-130
        Elements el;
        el.a = 1.0e8;
        el.e = 1.01;
        expect(throws<NonEllipticError>([&] { elements_to_state(el, mu_sun, 0.0); }), "unbound");
    });
}

// ----------------------------------------------------------------- dynamics
static void dynamics_cases() {
    run_case("two_body_closed_form", [] {  // test_dynamics.cpp:10-24
        V3 a = central_acc({1, 0, 0}, 1.0);
        expect(a.x == -1.0 && a.y == 0.0 && a.z == 0.0, "unit");
        a = central_acc({0, 2, 0}, 4.0);
        expect(a.x == 0.0 && a.y == -1.0 && a.z == 0.0, "scaled");
        expect(std::abs(central_acc({6378.137, 0, 0}, 398600.4418).norm() - 9.798e-3) <= 1e-6, "g0");
        expect(throws<SingularityError>([] { central_acc({0, 0, 0}, 1.0); }), "zero radius");
    });
    const Grid g5 = build_grid(5, 0.0, 1.0e6);
    run_case("nbody_without_perturbers_is_two_body", [&] {  // :34-41
        const EphTable t = build_ephemeris({}, g5, mu_sun);
        const State s = reference_state();
        const V3 a = table_acc(s.r, 0, t, ForceKind::n_body, 1.0), b = central_acc(s.r, mu_sun);
        expect(a.x == b.x && a.y == b.y && a.z == b.z, "exact");
    });
    run_case("nbody_vanishing_mass", [&] {  // :43-53
        auto bodies = reference_bodies();
        bodies.resize(1);
        bodies[0].mu = 1e-30;
        const EphTable t = build_ephemeris(bodies, g5, mu_sun);
        const State s = reference_state();
        const V3 a = table_acc(s.r, 2, t, ForceKind::n_body, 1.0), b = central_acc(s.r, mu_sun);
        expect((a - b).norm() / b.norm() <= 1e-15, "recover");
    });
    run_case("nbody_independent_scalar_sum", [] {  // :55-84
        const Grid g = build_grid(7, 0.0, 2.0e6);
        const auto bodies = reference_bodies();
        const EphTable t = build_ephemeris(bodies, g, mu_sun);
        const State s = reference_state();
        const V3 got = table_acc(s.r, 3, t, ForceKind::n_body, 1.0);
        const double rn = s.r.norm();
        double ax = -mu_sun * s.r.x / (rn * rn * rn), ay = -mu_sun * s.r.y / (rn * rn * rn),
               az = -mu_sun * s.r.z / (rn * rn * rn);
        for (const auto& b : bodies) {
            const V3 rb = body_position(b, mu_sun, g.times[3]);
            const double dx = rb.x - s.r.x, dy = rb.y - s.r.y, dz = rb.z - s.r.z;
            const double dn = std::sqrt(dx * dx + dy * dy + dz * dz), bn = rb.norm();
            ax += b.mu * (dx / (dn * dn * dn) - rb.x / (bn * bn * bn));
            ay += b.mu * (dy / (dn * dn * dn) - rb.y / (bn * bn * bn));
            az += b.mu * (dz / (dn * dn * dn) - rb.z / (bn * bn * bn));
        }
        expect(close_rel(got.x, ax, 1e-13) && close_rel(got.y, ay, 1e-13) && close_rel(got.z, az, 1e-13), "sum");
    });
    run_case("nbody_superposition", [] {  // :86-99
        const Grid g = build_grid(4, 0.0, 1.0e6);
        const auto bodies = reference_bodies();
        const EphTable both = build_ephemeris(bodies, g, mu_sun), first = build_ephemeris({bodies[0]}, g, mu_sun),
                       second = build_ephemeris({bodies[1]}, g, mu_sun);
        const State s = reference_state();
        const V3 c = central_acc(s.r, mu_sun);
        const V3 sum = (table_acc(s.r, 1, first, ForceKind::n_body, 1.0) - c) +
                       (table_acc(s.r, 1, second, ForceKind::n_body, 1.0) - c);
        const V3 comb = table_acc(s.r, 1, both, ForceKind::n_body, 1.0) - c;
        expect((comb - sum).norm() <= 1e-15 * sum.norm(), "superposition");
    });
    run_case("nbody_close_approach_named", [] {  // :101-115
        const Grid g = build_grid(3, 0.0, 1.0e5);
        const EphTable t = build_ephemeris(reference_bodies(), g, mu_sun);
        V3 r{t.pos[0](1, 0) + 0.4, t.pos[0](1, 1), t.pos[0](1, 2)};
        try {
            table_acc(r, 1, t, ForceKind::n_body, 1.0);
            expect(false, "no throw");
        } catch (const SingularityError& e) {
            expect(e.body == "venus-like" && std::string(e.what()).find("venus-like") != std::string::npos, "named");
        }
    });
    run_case("force_block_circular_orbit", [] {  // :117-145
        const Index n = 9;
        const double radius = 1.3e8, speed = std::sqrt(mu_sun / radius);
        const double period = 2.0 * std::numbers::pi * radius / speed;
        const Grid g = build_grid(n, 0.0, 0.5 * period);
        const EphTable t = build_ephemeris({}, g, mu_sun);
        const State s = make_state({radius, 0, 0}, {0, speed, 0});
        bool fb = false;
        const Mat guess = warm_guess(s, g, mu_sun, &fb);
        const Block b = assemble_block(&s, 1, g, &guess, 1);
        Mat f;
        eval_force_block(b.data, 1, g, t, reference_force(ForceKind::two_body), f);
        for (Index j = 0; j < n; ++j) {
            const V3 a{f(j, 3) / g.omega2, f(j, 4) / g.omega2, f(j, 5) / g.omega2};
            const V3 r{b.data(j, 0), b.data(j, 1), b.data(j, 2)};
            expect(std::abs(a.norm() * r.sq() - mu_sun) / mu_sun <= 1e-13, "|a||r|^2");
            expect(f(j, 0) == g.omega2 * b.data(j, 3), "velocity row");
        }
    });
    run_case("force_block_replicated_columns", [] {  // :147-162
        const Index n = 6;
        const Grid g = build_grid(n, 0.0, 1.0e6);
        const EphTable t = build_ephemeris(reference_bodies(), g, mu_sun);
        const auto states = clone_batch(reference_state(), 3, 0.0);
        std::vector<Mat> gs;
        for (const auto& s : states) gs.push_back(cold_guess(s, n));
        const Block b = assemble_block(states.data(), 3, g, gs.data(), 3);
        Mat f;
        eval_force_block(b.data, 3, g, t, reference_force(), f);
        for (Index c = 0; c < 6; ++c)
            for (Index k = 1; k < 3; ++k)
                for (Index j = 0; j < n; ++j) expect(f(j, c * 3 + k) == f(j, c * 3), "identical");
    });
    run_case("force_block_equals_per_sample_loop_13509", [] {  // :164-190
        const Index n = 3, m = 13509;
        const Grid g = build_grid(n, 0.0, 2.0e6);
        const EphTable t = build_ephemeris(reference_bodies(), g, mu_sun);
        const auto states = clone_batch(reference_state(), m, 2e-4);
        std::vector<Mat> gs;
        for (const auto& s : states) gs.push_back(cold_guess(s, n));
        const Block b = assemble_block(states.data(), m, g, gs.data(), m);
        Mat f;
        eval_force_block(b.data, m, g, t, reference_force(), f);
        const Index j = 1;
        for (Index k = 0; k < m; ++k) {
            const V3 r{b.data(j, k), b.data(j, m + k), b.data(j, 2 * m + k)};
            const V3 a = table_acc(r, j, t, ForceKind::n_body, 1.0);
            expect(f(j, 3 * m + k) == g.omega2 * a.x && f(j, 4 * m + k) == g.omega2 * a.y &&
                       f(j, 5 * m + k) == g.omega2 * a.z && f(j, k) == g.omega2 * b.data(j, 3 * m + k),
                   "bitwise");
        }
    });
    run_case("force_block_parallel_bit_identical", [] {  // :192-206
        const Index n = 12;
        const Grid g = build_grid(n, 0.0, 3.0e6);
        const EphTable t = build_ephemeris(reference_bodies(), g, mu_sun);
        const auto states = clone_batch(reference_state(), 41, 1e-4);
        std::vector<Mat> gs;
        bool fb;
        for (const auto& s : states) gs.push_back(warm_guess(s, g, mu_sun, &fb));
        const Block b = assemble_block(states.data(), 41, g, gs.data(), 41);
        Mat f1, f2;
        eval_force_block(b.data, 41, g, t, reference_force(), f1);
        Pool pool(2);
        eval_force_block(b.data, 41, g, t, reference_force(), f2, &pool);
        expect(f1.v == f2.v, "bitwise");
    });
    run_case("force_block_singularity_coordinates", [] {  // :208-227
        const Index n = 5;
        const Grid g = build_grid(n, 0.0, 1.0e6);
        const EphTable t = build_ephemeris(reference_bodies(), g, mu_sun);
        auto states = clone_batch(reference_state(), 4, 1e-4);
        states[2].r = {t.pos[0](0, 0), t.pos[0](0, 1), t.pos[0](0, 2)};
        std::vector<Mat> gs;
        for (const auto& s : states) gs.push_back(cold_guess(s, n));
        const Block b = assemble_block(states.data(), 4, g, gs.data(), 4);
        Mat f;
        try {
            eval_force_block(b.data, 4, g, t, reference_force(), f);
            expect(false, "no throw");
        } catch (const SingularityError& e) {
            expect(std::string(e.what()).find("trajectory 2") != std::string::npos && e.body == "venus-like", "tag");
        }
    });
    run_case("ephemeris_zero_bodies", [] {  // :229-235
        const Grid g = build_grid(4, 0.0, 1.0e5);
        const EphTable t = build_ephemeris({}, g, mu_sun);
        expect(t.n_bodies() == 0 && t.central_mu == mu_sun && t.node_times == g.times, "table");
    });
    run_case("ephemeris_circular_body_closes", [] {  // :237-256
        Body b;
        b.name = "circular";
        b.mu = 1e5;
        b.el = {1.1e8, 0.0, 0.2, 0.4, 0.0, 1.0, 0.0};
        const double period = 2.0 * std::numbers::pi * std::sqrt(b.el.a * b.el.a * b.el.a / mu_sun);
        const Grid g = build_grid(33, 0.0, period);
        const EphTable t = build_ephemeris({b}, g, mu_sun);
        const V3 p0{t.pos[0](0, 0), t.pos[0](0, 1), t.pos[0](0, 2)}, p1{t.pos[0](32, 0), t.pos[0](32, 1), t.pos[0](32, 2)};
        expect((p0 - p1).norm() / p0.norm() <= 1e-11, "closure");
    });
    run_case("ephemeris_tabulated_round_trip", [] {  // :258-280
        const auto bodies = reference_bodies();
        const double t1 = 4.0e6;
        Body tab;
        tab.name = bodies[0].name;
        tab.mu = bodies[0].mu;
        tab.tabulated = true;
        tab.segs.push_back(fit_segment([&](double t) { return body_position(bodies[0], mu_sun, t); }, 0.0, t1, 24));
        const Grid g = build_grid(17, 0.0, t1);
        const EphTable ta = build_ephemeris({bodies[0]}, g, mu_sun), tt = build_ephemeris({tab}, g, mu_sun);
        for (Index j = 0; j < 17; ++j) {
            const V3 pa{ta.pos[0](j, 0), ta.pos[0](j, 1), ta.pos[0](j, 2)};
            const V3 pt{tt.pos[0](j, 0), tt.pos[0](j, 1), tt.pos[0](j, 2)};
            expect((pa - pt).norm() / pa.norm() <= 1e-12, "round trip");
        }
    });
    run_case("ephemeris_coverage_error_epoch", [] {  // :282-297
        Body tab;
        tab.name = "short-table";
        tab.mu = 1.0;
        tab.tabulated = true;
        tab.segs.push_back(fit_segment([](double) { return V3{1e8, 0, 0}; }, 0.0, 1.0e5, 8));
        const Grid g = build_grid(5, 0.0, 2.0e5);
        try {
            build_ephemeris({tab}, g, mu_sun);
            expect(false, "no throw");
        } catch (const CoverageError& e) {
            expect(e.epoch > 1.0e5, "epoch");
        }
    });
}

// ------------------------------------------------------------- augmentation
static void augmentation_cases() {
    run_case("split_groups_13509_into_10", [] {  // test_augmentation.cpp:14-32
        const Plan p = split_groups(13509, 10);
        Index sum = 0, hi = 0, lo = 1 << 30;
        for (Index s : p.sizes) {
            sum += s;
            hi = std::max(hi, s);
            lo = std::min(lo, s);
        }
        expect(p.groups() == 10 && sum == 13509 && hi - lo <= 1 && p.sizes[0] >= p.sizes[9], "balance");
        for (Index i = 0; i < 13509; ++i) expect(p.offsets[p.group_of[i]] + p.slot_of[i] == i, "assignment");
    });
    run_case("split_groups_degenerate", [] {  // :34-49
        expect(split_groups(7, 1).sizes[0] == 7, "one");
        const Plan s = split_groups(5, 5);
        for (Index x : s.sizes) expect(x == 1, "singletons");
        expect(throws<InvalidPlanError>([] { split_groups(5, 0); }) && throws<InvalidPlanError>([] { split_groups(5, 6); }) &&
                   throws<InvalidPlanError>([] { split_groups(0, 1); }),
               "errors");
    });
    run_case("plan_from_sizes", [] {  // :51-56
        const Plan p = plan_from_sizes({4, 1, 7});
        expect(p.total == 12 && p.offsets[2] == 5, "offsets");
        expect(throws<InvalidPlanError>([] { plan_from_sizes({3, 0}); }), "zero");
    });
    run_case("assemble_component_order", [] {  // :58-72
        const Grid g = build_grid(4, 0.0, 1.0);
        const State s = make_state({1, 2, 3}, {4, 5, 6});
        const Mat gs = cold_guess(s, 4);
        const Block b = assemble_block(&s, 1, g, &gs, 1);
        for (Index c = 0; c < 6; ++c) expect(b.y0[c] == c + 1.0 && b.data(2, c) == c + 1.0, "order");
    });
    run_case("assemble_round_trip_1501", [] {  // :85-115
        const Index m = 1501, n = 8;
        const Grid g = build_grid(n, 0.0, 1.0);
        std::vector<State> states(m);
        std::vector<Mat> gs(m);
        std::uint64_t rng = 99;
        for (Index t = 0; t < m; ++t) {
            Mat x(n, 6);
            for (auto& v : x.v) v = 1e6 * symmetric_unit(rng);
            states[t] = make_state({x(0, 0), x(0, 1), x(0, 2)}, {x(0, 3), x(0, 4), x(0, 5)});
            gs[t] = std::move(x);
        }
        const Block b = assemble_block(states.data(), m, g, gs.data(), m);
        expect(Block::col(2, 17, m) == 2 * m + 17 && b.data(3, 2 * m + 17) == gs[17](3, 2), "bijection");
        const auto back = disassemble_block(b);
        for (Index t = 0; t < m; ++t) expect(back[t].v == gs[t].v, "round trip");
    });
    run_case("assemble_misaligned_rejected", [] {  // :117-131
        const Grid g = build_grid(4, 0.0, 1.0);
        State s;
        Mat wrong(3, 6), ok(4, 6);
        expect(throws<AlignmentError>([&] { assemble_block(&s, 1, g, &wrong, 1); }), "rows");
        s.epoch = 0.5;
        expect(throws<AlignmentError>([&] { assemble_block(&s, 1, g, &ok, 1); }), "epoch");
        s.epoch = 0.0;
        expect(throws<ShapeError>([&] { assemble_block(&s, 1, g, nullptr, 0); }), "none");
    });
    run_case("block_error_single_perturbation", [] {  // :140-162
        const Index n = 4;
        const Grid g = build_grid(n, 0.0, 1.0);
        std::vector<State> st(2, make_state({1, 0, 0}, {0, 1, 0}));
        std::vector<Mat> gs{cold_guess(st[0], n), cold_guess(st[1], n)};
        const Block prev = assemble_block(st.data(), 2, g, gs.data(), 2);
        Block cur = prev;
        const double delta = 0x1.0p-21;
        cur.data(2, Block::col(0, 1, 2)) += delta;
        double gmax = 0.0;
        const auto per = block_iteration_error(cur.data, prev.data, 2, ErrorMode::relative, &gmax);
        expect(std::abs(gmax - delta) <= 1e-15 && per[0] == 0.0 && std::abs(per[1] - delta) <= 1e-15, "relative");
        block_iteration_error(cur.data, prev.data, 2, ErrorMode::absolute, &gmax);
        expect(std::abs(gmax - delta) <= 1e-15, "absolute");
    });
    run_case("block_error_brute_force_and_parallel", [] {  // :164-210
        const Index n = 6, m = 23;
        const Grid g = build_grid(n, 0.0, 1.0);
        std::vector<State> st(m);
        std::vector<Mat> cg(m), pg(m);
        std::uint64_t rng = 5;
        for (Index t = 0; t < m; ++t) {
            Mat a(n, 6), b(n, 6);
            for (Index j = 0; j < n; ++j)
                for (Index c = 0; c < 6; ++c) {
                    b(j, c) = 10.0 + symmetric_unit(rng);
                    a(j, c) = b(j, c) + 1e-7 * symmetric_unit(rng);
                }
            for (Index c = 0; c < 6; ++c) a(0, c) = b(0, c);
            st[t] = make_state({b(0, 0), b(0, 1), b(0, 2)}, {b(0, 3), b(0, 4), b(0, 5)});
            cg[t] = std::move(a);
            pg[t] = std::move(b);
        }
        const Block cur = assemble_block(st.data(), m, g, cg.data(), m), prev = assemble_block(st.data(), m, g, pg.data(), m);
        double gmax = 0.0;
        block_iteration_error(cur.data, prev.data, m, ErrorMode::relative, &gmax);
        double brute = 0.0;
        for (Index t = 0; t < m; ++t)
            for (Index j = 0; j < n; ++j) {
                const V3 dr{cg[t](j, 0) - pg[t](j, 0), cg[t](j, 1) - pg[t](j, 1), cg[t](j, 2) - pg[t](j, 2)};
                const V3 dv{cg[t](j, 3) - pg[t](j, 3), cg[t](j, 4) - pg[t](j, 4), cg[t](j, 5) - pg[t](j, 5)};
                brute = std::max(brute, dr.norm() / V3{pg[t](j, 0), pg[t](j, 1), pg[t](j, 2)}.norm());
                brute = std::max(brute, dv.norm() / V3{pg[t](j, 3), pg[t](j, 4), pg[t](j, 5)}.norm());
            }
        expect(close_rel(gmax, brute, 1e-14), "brute");
        Pool pool(2);
        expect(block_max_error(cur.data, prev.data, m, ErrorMode::relative, &pool) == gmax, "parallel");
    });
    run_case("reduce_max_levels_and_equivalence", [] {  // :221-250
        expect(reduction_levels(16) == 5 && reduction_levels(1) == 1 && reduction_levels(2) == 2 &&
                   reduction_levels(13509) == 15,
               "levels");
        std::vector<double> v(13509);
        std::uint64_t rng = 31;
        for (auto& x : v) x = 1e3 * symmetric_unit(rng);
        v[5000] = v[123];
        const double e = *std::max_element(v.begin(), v.end());
        Pool pool(2);
        expect(reduce_max(v.data(), v.size()) == e && reduce_max_tree(v.data(), v.size()) == e &&
                   reduce_max_tree(v.data(), v.size(), &pool) == e,
               "equivalence");
        expect(throws<EmptyReductionError>([] { reduce_max(nullptr, 0); }) &&
                   throws<EmptyReductionError>([] { reduce_max_tree(nullptr, 0); }),
               "empty");
    });
    run_case("reduce_max_randomized_1000", [] {  // acceptance.cpp:296-318 (reduction half)
        std::uint64_t rng = 20220411ULL;
        for (int trial = 0; trial < 1000; ++trial) {
            const std::size_t size = 1 + (splitmix64(rng) % 300);
            std::vector<double> v(size);
            for (auto& x : v) x = 1e4 * symmetric_unit(rng);
            if (size > 2 && trial % 4 == 0) v[size - 1] = v[size / 3];
            const double e = *std::max_element(v.begin(), v.end());
            expect(reduce_max_tree(v.data(), size) == e && reduce_max(v.data(), size) == e, "trial");
        }
    });
    auto two_body_case = [](Index n, double frac, Grid& g, EphTable& t) {
        const double period = osculating_period(reference_state(), mu_sun);
        g = build_grid(n, 0.0, frac * period);
        t = build_ephemeris({}, g, mu_sun);
    };
    run_case("solve_group_singleton_equals_standalone", [&] {  // :277-301
        Grid g;
        EphTable t;
        two_body_case(48, 0.4, g, t);
        const auto ops = cached_ops(48);
        const auto st = clone_batch(reference_state(), 1, 0.0);
        bool fb;
        const Mat gs = warm_guess(st[0], g, mu_sun, &fb);
        const Block b = assemble_block(st.data(), 1, g, &gs, 1);
        const ForceConfig cfg = reference_force(ForceKind::two_body);
        auto [solved, rep] = solve_group(b, g, *ops, t, cfg, 1e-12, 100);
        auto dyn = [&](const Mat& y, Mat& f) { eval_force_block(y, 1, g, t, cfg, f); };
        auto err = [&](const Mat& c, const Mat& p) { return block_max_error(c, p, 1, ErrorMode::relative); };
        auto [alone, rep2] = pc_solve(*ops, dyn, b.data, b.y0, 1e-12, 100, err);
        expect(rep.converged && rep2.converged && solved.data.v == alone.v, "bitwise");
    });
    run_case("solve_group_identical_members", [&] {  // :303-317
        Grid g;
        EphTable t;
        two_body_case(40, 0.3, g, t);
        const auto st = clone_batch(reference_state(), 4, 0.0);
        std::vector<Mat> gs;
        bool fb;
        for (const auto& s : st) gs.push_back(warm_guess(s, g, mu_sun, &fb));
        auto [solved, rep] = solve_group(assemble_block(st.data(), 4, g, gs.data(), 4), g, *cached_ops(40), t,
                                         reference_force(ForceKind::two_body), 1e-12, 100);
        expect(rep.converged, "converged");
        const auto tr = disassemble_block(solved);
        double scale = 0.0;
        for (double x : tr[0].v) scale = std::max(scale, std::abs(x));
        for (std::size_t k = 1; k < tr.size(); ++k) expect(max_abs_diff(tr[k], tr[0]) / scale <= 1e-14, "identical");
    });
    run_case("solve_group_warm_two_body_fixed_point", [&] {  // :320-333
        Grid g;
        EphTable t;
        two_body_case(64, 0.6, g, t);
        const auto st = clone_batch(reference_state(), 2, 1e-5);
        std::vector<Mat> gs;
        bool fb;
        for (const auto& s : st) gs.push_back(warm_guess(s, g, mu_sun, &fb));
        auto [solved, rep] = solve_group(assemble_block(st.data(), 2, g, gs.data(), 2), g, *cached_ops(64), t,
                                         reference_force(ForceKind::two_body), 1e-12, 100);
        expect(rep.converged && rep.iterations <= 3, "<= 3 iterations, got " + std::to_string(rep.iterations));
        for (std::size_t i = 2; i < rep.history.size(); ++i) expect(rep.history[i] <= rep.history[i - 1], "monotone");
    });
    run_case("solve_group_perturbed_arc_contracts", [] {  // :335-360
        const auto st = clone_batch(reference_state(), 2, 1e-5);
        const double period = osculating_period(st[0], mu_sun);
        const Grid g = build_grid(128, 0.0, 0.6 * period);
        const EphTable t = build_ephemeris(reference_bodies(), g, mu_sun);
        std::vector<Mat> gs;
        bool fb;
        for (const auto& s : st) gs.push_back(warm_guess(s, g, mu_sun, &fb));
        auto [solved, rep] = solve_group(assemble_block(st.data(), 2, g, gs.data(), 2), g, *cached_ops(128), t,
                                         reference_force(), 1e-12, 100);
        expect(rep.converged, "converged");
        const auto& e = rep.history;
        std::size_t settle = e.size() - 1;
        while (settle > 0 && e[settle] <= e[settle - 1]) --settle;
        expect(settle <= e.size() / 2 && e.back() <= 1e-12 && e.back() < e.front(), "contraction");
    });
    run_case("solve_group_worst_member", [&] {  // :363-374
        Grid g;
        EphTable t;
        two_body_case(40, 0.3, g, t);
        const auto st = clone_batch(reference_state(), 6, 1e-4);
        std::vector<Mat> gs;
        bool fb;
        for (const auto& s : st) gs.push_back(warm_guess(s, g, mu_sun, &fb));
        auto [solved, rep] = solve_group(assemble_block(st.data(), 6, g, gs.data(), 6), g, *cached_ops(40), t,
                                         reference_force(ForceKind::two_body), 1e-12, 100);
        expect(rep.converged && rep.final_error <= 1e-12 && rep.iterations >= 1 &&
                   rep.history.size() == static_cast<std::size_t>(rep.iterations),
               "report");
    });
}

// --------------------------------------------------------------- propagator
static void propagator_cases() {
    run_case("cold_start_replicates", [] {  // test_propagator.cpp:10-25
        const State s = make_state({1, 2, 3}, {-1, 0.5, 0.25});
        const Mat g = cold_guess(s, 3);
        for (Index j = 0; j < 3; ++j) expect(g(j, 0) == 1.0 && g(j, 5) == 0.25, "rows");
    });
    run_case("warm_start_half_period_antipodal", [] {  // :27-44
        const double speed = std::sqrt(mu_sun / 1.3e8);
        const State s = make_state({1.3e8, 0, 0}, {0, speed, 0});
        const Grid g = build_grid(21, 0.0, 0.5 * osculating_period(s, mu_sun));
        bool fb = true;
        const Mat w = warm_guess(s, g, mu_sun, &fb);
        expect(!fb && w(0, 0) == s.r.x && close_rel(w(20, 0), -1.3e8, 1e-10) && close_rel(w(20, 4), -speed, 1e-10),
               "antipode");
    });
    run_case("warm_start_hyperbolic_fallback", [] {  // :46-58
        const State h = make_state({1.0e8, 0, 0}, {0, 60.0, 0});
        const Grid g = build_grid(5, 0.0, 1.0e6);
        bool fb = false;
        const Mat w = warm_guess(h, g, mu_sun, &fb);
        expect(fb, "flag");
        for (Index j = 0; j < 5; ++j) expect(w(j, 0) == 1.0e8 && w(j, 4) == 60.0, "cold rows");
    });
    const State ref = reference_state();
    const double period = osculating_period(ref, mu_sun);
    run_case("plan_segments_single", [&] {  // :60-67
        const Segments p = plan_segments(ref, 0.0, 0.87 * period, mu_sun, SegmentPolicy::per_orbit, 200);
        expect(p.count() == 1 && p.direction == Direction::forward && p.boundaries.back() == 0.87 * period, "single");
    });
    run_case("plan_segments_2p5_periods", [&] {  // :69-77
        const Segments p = plan_segments(ref, 0.0, 2.5 * period, mu_sun, SegmentPolicy::per_orbit, 64);
        expect(p.count() == 3 && close_rel(p.boundaries[1], period, 1e-12) && close_rel(p.boundaries[2], 2 * period, 1e-12) &&
                   close_rel(p.boundaries[3], 2.5 * period, 1e-12),
               "1,1,0.5");
    });
    run_case("plan_segments_backward", [&] {  // :79-88
        const Segments p = plan_segments(ref, 0.0, -1.6 * period, mu_sun, SegmentPolicy::per_orbit, 32);
        expect(p.direction == Direction::backward && p.count() == 2 && p.boundaries[1] < p.boundaries[0] &&
                   build_grid(32, p.boundaries[0], p.boundaries[1]).omega2 < 0.0,
               "backward");
    });
    run_case("plan_segments_guardrails", [&] {  // :90-104
        expect(throws<InvalidSpanError>([&] { plan_segments(ref, 5.0, 5.0, mu_sun, SegmentPolicy::single, 10); }), "degenerate");
        expect(throws<InvalidSpanError>([&] { plan_segments(ref, 0.0, 3.0 * period, mu_sun, SegmentPolicy::single, 10); }),
               "too long");
        const State h = make_state({1.0e8, 0, 0}, {0, 60.0, 0});
        expect(throws<NonEllipticError>([&] { plan_segments(h, 0.0, 1.0e6, mu_sun, SegmentPolicy::per_orbit, 10); }),
               "hyperbolic");
    });
    run_case("propagate_exact_warm_start_fixed_point", [&] {  // :118-139
        const Config cfg = twobody_config(48);
        const auto st = clone_batch(ref, 3, 1e-6);
        const Segments sp = plan_segments(st[0], 0.0, 0.5 * period, mu_sun, SegmentPolicy::single, 48);
        const Result r = propagate(st, split_groups(3, 1), sp, cfg);
        expect(r.reports.size() == 1 && r.reports[0][0].converged && r.reports[0][0].iterations <= 3, "iterations");
        for (Index j = 0; j < 48; ++j) {
            const State e = kepler_propagate(st[1], mu_sun, r.times[j]);
            const V3 got{r.trajectories[1](j, 0), r.trajectories[1](j, 1), r.trajectories[1](j, 2)};
            expect((got - e.r).norm() / e.r.norm() <= 1e-12, "conic");
        }
    });
    run_case("propagate_segments_chain_exactly", [&] {  // :141-166
        Config cfg = twobody_config(32);
        cfg.segment_policy = SegmentPolicy::per_orbit;
        const auto st = clone_batch(ref, 2, 1e-5);
        const Segments sp = plan_segments(st[0], 0.0, 1.7 * period, mu_sun, SegmentPolicy::per_orbit, 32);
        expect(sp.count() == 2, "two segments");
        const Result r = propagate(st, split_groups(2, 2), sp, cfg);
        expect(static_cast<Index>(r.times.size()) == 1 + 2 * 31 && r.times[31] == sp.boundaries[1], "times");
        for (std::size_t i = 0; i < 2; ++i) {
            const Mat& tr = r.trajectories[i];
            const Index last = tr.r - 1;
            expect(r.terminal_states[i].r.x == tr(last, 0) && r.terminal_states[i].v.z == tr(last, 5) &&
                       r.terminal_states[i].epoch == sp.boundaries[2],
                   "terminal");
        }
        for (const auto& s : r.reports)
            for (const auto& q : s) expect(q.converged, "converged");
    });
    run_case("propagate_warm_beats_cold", [&] {  // :168-190
        Config cfg = nbody_config(96);
        const auto st = clone_batch(ref, 6, 1e-5);
        const Segments sp = plan_segments(st[0], 0.0, 0.6 * period, mu_sun, SegmentPolicy::single, 96);
        const Plan pl = split_groups(6, 2);
        const Result w = propagate(st, pl, sp, cfg);
        cfg.start_mode = StartMode::cold;
        const Result c = propagate(st, pl, sp, cfg);
        for (Index g = 0; g < 2; ++g)
            expect(w.reports[0][g].iterations < c.reports[0][g].iterations && w.reports[0][g].converged &&
                       c.reports[0][g].converged,
                   "warm < cold");
    });
    run_case("propagate_forward_backward_round_trip", [&] {  // :192-212
        const Config cfg = twobody_config(64);
        const auto st = clone_batch(ref, 4, 1e-5);
        const double t_end = 0.7 * period;
        const Result f = propagate(st, split_groups(4, 1),
                                   plan_segments(st[0], 0.0, t_end, mu_sun, SegmentPolicy::single, 64), cfg);
        const Result b = propagate(f.terminal_states, split_groups(4, 1),
                                   plan_segments(f.terminal_states[0], t_end, 0.0, mu_sun, SegmentPolicy::single, 64), cfg);
        for (std::size_t i = 0; i < 4; ++i) expect(rel_state(b.terminal_states[i], st[i]) <= 1e-9, "round trip");
    });
    run_case("propagate_mixed_epochs_rejected", [&] {  // :214-227
        const Config cfg = twobody_config(16);
        auto st = clone_batch(ref, 3, 1e-5);
        st[2].epoch = 10.0;
        const Segments sp = plan_segments(st[0], 0.0, 1.0e6, mu_sun, SegmentPolicy::single, 16);
        try {
            propagate(st, split_groups(3, 1), sp, cfg);
            expect(false, "no throw");
        } catch (const AlignmentError& e) {
            expect(std::string(e.what()).find("state 2") != std::string::npos, "index");
        }
    });
    run_case("propagate_nonconvergence_partial", [&] {  // :229-249
        Config cfg = twobody_config(64);
        cfg.start_mode = StartMode::cold;
        cfg.max_iterations = 3;
        const auto st = clone_batch(ref, 4, 1e-5);
        const Segments sp = plan_segments(st[0], 0.0, 0.8 * period, mu_sun, SegmentPolicy::single, 64);
        try {
            propagate(st, split_groups(4, 2), sp, cfg);
            expect(false, "no throw");
        } catch (const IncompleteError& e) {
            expect(e.segment == 0 && e.group == 0 && e.partial && !e.partial->reports.at(0).at(0).converged, "partial");
        }
    });
    run_case("propagate_timeout", [&] {  // :251-261
        Config cfg = nbody_config(64);
        cfg.timeout_s = 1e-9;
        const auto st = clone_batch(ref, 4, 1e-5);
        const Segments sp = plan_segments(st[0], 0.0, 1.0e6, mu_sun, SegmentPolicy::single, 64);
        expect(throws<TimeoutError>([&] { propagate(st, split_groups(4, 1), sp, cfg); }), "timeout");
    });
}

// ------------------------------------------------------------------- runner
static void runner_cases() {
    auto make = [](Index m, Index n, double frac, Config& cfg, std::vector<State>& st, Segments& sp) {
        cfg = nbody_config(n);
        st = clone_batch(reference_state(), m, 1e-5);
        sp = plan_segments(st[0], 0.0, frac * osculating_period(st[0], mu_sun), mu_sun, SegmentPolicy::single, n);
    };
    run_case("run_batch_singleton_grouped_equals_independent", [&] {  // test_runner.cpp:31-43
        Config cfg;
        std::vector<State> st;
        Segments sp;
        make(6, 64, 0.4, cfg, st, sp);
        cfg.p_groups = 6;
        const auto g = run_batch(st, cfg, sp, RunMode::grouped, 1);
        const auto i = run_batch(st, cfg, sp, RunMode::independent, 1);
        expect(g.result.plan.groups() == 6 && i.result.plan.groups() == 6, "groups");
        for (std::size_t k = 0; k < 6; ++k) expect(g.result.trajectories[k].v == i.result.trajectories[k].v, "bitwise");
    });
    run_case("run_batch_four_modes_agree", [&] {  // :45-59
        Config cfg;
        std::vector<State> st;
        Segments sp;
        make(12, 80, 0.5, cfg, st, sp);
        cfg.p_groups = 3;
        const auto ind = run_batch(st, cfg, sp, RunMode::independent, 2);
        const auto seq = run_batch(st, cfg, sp, RunMode::augmented_sequential, 1);
        const auto par = run_batch(st, cfg, sp, RunMode::augmented_parallel, 2);
        const auto grp = run_batch(st, cfg, sp, RunMode::grouped, 2);
        expect(max_state_discrepancy(seq.result, ind.result) < 1e-12 &&
                   max_state_discrepancy(par.result, ind.result) < 1e-12 &&
                   max_state_discrepancy(grp.result, ind.result) < 1e-12 &&
                   max_state_discrepancy(par.result, seq.result) < 1e-12,
               "agreement");
    });
    run_case("run_batch_reproducible", [&] {  // :61-70
        Config cfg;
        std::vector<State> st;
        Segments sp;
        make(5, 48, 0.3, cfg, st, sp);
        const auto a = run_batch(st, cfg, sp, RunMode::augmented_sequential, 1);
        const auto b = run_batch(st, cfg, sp, RunMode::augmented_sequential, 1);
        for (std::size_t k = 0; k < 5; ++k) expect(a.result.trajectories[k].v == b.result.trajectories[k].v, "bitwise");
        expect(a.result.max_iterations_used() == b.result.max_iterations_used(), "iterations");
    });
    run_case("run_batch_zero_workers", [&] {  // :72-76
        Config cfg;
        std::vector<State> st;
        Segments sp;
        make(3, 16, 0.1, cfg, st, sp);
        expect(throws<InvalidPlanError>([&] { run_batch(st, cfg, sp, RunMode::grouped, 0); }), "rejected");
    });
}

// ------------------------------------------------------------------- oracle
static void rk_cases() {
    run_case("rkf78_tableau_row_sums", [] {  // test_oracle.cpp:28-42
        for (std::size_t i = 0; i < 13; ++i) {
            double s = 0.0;
            for (std::size_t l = 0; l < i; ++l) s += rkf78::a[i][l];
            expect(close_rel(s, rkf78::c[i], 1e-14), "row sum");
        }
        double b = 0.0;
        for (double x : rkf78::b8) b += x;
        expect(close_rel(b, 1.0, 1e-15), "weights");
    });
    run_case("rk_full_period_returns", [] {  // :44-50
        const State s = reference_state();
        const State o = rk_propagate(s, two_body_deriv(mu_sun), osculating_period(s, mu_sun));
        expect((o.r - s.r).norm() / s.r.norm() <= 1e-11 && (o.v - s.v).norm() / s.v.norm() <= 1e-11, "return");
    });
    run_case("rk_agrees_with_conic_varied_arcs", [] {  // :52-70
        std::uint64_t seed = 7;
        for (int trial = 0; trial < 6; ++trial) {
            Elements el;
            el.a = 1.0e8 * (1.0 + 0.08 * trial);
            el.e = 0.1 * trial + 0.05;
            el.i = 0.2 * symmetric_unit(seed);
            el.raan = std::numbers::pi * symmetric_unit(seed);
            el.argp = std::numbers::pi * symmetric_unit(seed);
            el.m0 = std::numbers::pi * symmetric_unit(seed);
            const State s = elements_to_state(el, mu_sun, 0.0);
            const double dt = (0.1 + 0.15 * trial) * osculating_period(s, mu_sun);
            const State num = rk_propagate(s, two_body_deriv(mu_sun), dt), ana = kepler_propagate(s, mu_sun, dt);
            expect((num.r - ana.r).norm() / ana.r.norm() <= 1e-11 && (num.v - ana.v).norm() / ana.v.norm() <= 1e-11,
                   "trial " + std::to_string(trial));
        }
    });
    run_case("rk_backward", [] {  // :72-78
        const State s = reference_state();
        const State f = kepler_propagate(s, mu_sun, 2.0e6);
        expect((rk_propagate(f, two_body_deriv(mu_sun), s.epoch).r - s.r).norm() / s.r.norm() <= 1e-11, "backward");
    });
    run_case("rk_tolerance_monotonicity", [] {  // :80-92
        const State s = reference_state();
        RkConfig loose, tight;
        loose.rel_tol = 1e-10;
        tight.rel_tol = 1e-11;
        const State a = rk_propagate(s, two_body_deriv(mu_sun), 4.0e6, loose);
        const State b = rk_propagate(s, two_body_deriv(mu_sun), 4.0e6, tight);
        expect((a.r - b.r).norm() / b.r.norm() < 1e-10 && (a.v - b.v).norm() / b.v.norm() < 1e-10, "monotone");
    });
    run_case("rk_step_exhaustion", [] {  // :94-100
        const State s = reference_state();
        RkConfig cfg;
        cfg.max_steps = 3;
        expect(throws<OracleError>([&] { rk_propagate(s, two_body_deriv(mu_sun), osculating_period(s, mu_sun), cfg); }),
               "exhaustion");
    });
    run_case("pc_two_body_tracks_rk_over_period", [] {  // :102-117
        Config cfg = twobody_config(200);
        cfg.start_mode = StartMode::cold;
        const auto st = clone_batch(reference_state(), 1, 0.0);
        const Segments sp =
            plan_segments(st[0], 0.0, osculating_period(st[0], mu_sun), mu_sun, SegmentPolicy::single, 200);
        const Result r = propagate(st, split_groups(1, 1), sp, cfg);
        expect(r.reports[0][0].converged, "converged");
        const Mat ref = rk_sample(st[0], two_body_deriv(mu_sun), r.times);
        expect(compare_trajectories(r.trajectories[0], ref) <= 1e-10, "tracks rk");
    });
    run_case("rk_sample_and_compare", [] {  // :119-147
        const State s = reference_state();
        const std::vector<double> times{0.0, 1.0e5, 5.0e5, 1.2e6};
        const Mat smp = rk_sample(s, two_body_deriv(mu_sun), times);
        expect(compare_trajectories(smp, smp) == 0.0, "self");
        Mat conic(4, 6);
        for (Index j = 0; j < 4; ++j) {
            const State sj = kepler_propagate(s, mu_sun, times[j]);
            conic(j, 0) = sj.r.x; conic(j, 1) = sj.r.y; conic(j, 2) = sj.r.z;
            conic(j, 3) = sj.v.x; conic(j, 4) = sj.v.y; conic(j, 5) = sj.v.z;
        }
        expect(compare_trajectories(smp, conic) <= 1e-11, "conic");
        expect(throws<OracleError>([&] { rk_sample(s, two_body_deriv(mu_sun), {5.0, 10.0}); }), "epoch");
    });
}

// --------------------------------------------------------------- acceptance
static void acceptance_cases() {
    run_case("acceptance_2_two_body_full_period", [] {  // acceptance.cpp:78-124
        const State s = elements_to_state({1.3e8, 0.2, 0.05, 0.4, 0.9, 0.0, 0.0}, mu_sun, 0.0);
        const double period = osculating_period(s, mu_sun);
        Config cfg = twobody_config(200);
        cfg.start_mode = StartMode::cold;
        const Result r = propagate({s}, split_groups(1, 1),
                                   plan_segments(s, 0.0, period, mu_sun, SegmentPolicy::single, 200), cfg);
        double ws = 0, we = 0, wm = 0;
        const double e0 = specific_energy(s, mu_sun);
        const V3 h0 = angular_momentum(s);
        for (std::size_t j = 0; j < r.times.size(); ++j) {
            const State want = kepler_propagate(s, mu_sun, r.times[j]);
            const State got = make_state({r.trajectories[0](j, 0), r.trajectories[0](j, 1), r.trajectories[0](j, 2)},
                                         {r.trajectories[0](j, 3), r.trajectories[0](j, 4), r.trajectories[0](j, 5)});
            ws = std::max({ws, (got.r - want.r).norm() / want.r.norm(), (got.v - want.v).norm() / want.v.norm()});
            we = std::max(we, std::abs(specific_energy(got, mu_sun) - e0) / std::abs(e0));
            wm = std::max(wm, (angular_momentum(got) - h0).norm() / h0.norm());
        }
        expect(r.reports[0][0].converged && ws <= 1e-10 && we <= 1e-11 && wm <= 1e-11,
               "state " + fmt(ws) + " energy " + fmt(we) + " momentum " + fmt(wm));
    });
    run_case("acceptance_3_4_5_9_reference_batch", [] {  // acceptance.cpp:135-234
        const auto st = clone_batch(reference_state(), 64, 1e-5);
        Config cfg = nbody_config(200);
        const double period = osculating_period(st[0], mu_sun), t_end = 0.87 * period;
        const Segments sp = plan_segments(st[0], 0.0, t_end, mu_sun, SegmentPolicy::single, 200);
        cfg.p_groups = 4;
        const auto grouped = run_batch(st, cfg, sp, RunMode::grouped, 1);
        double worst = 0.0;
        for (std::size_t i = 0; i < st.size(); ++i)
            worst = std::max(worst, compare_trajectories(grouped.result.trajectories[i],
                                                         rk_sample(st[i], nbody_deriv(cfg.force), grouped.result.times)));
        expect(worst <= 1e-9, "criterion 3 oracle " + fmt(worst));
        const auto ind = run_batch(st, cfg, sp, RunMode::independent, 1);
        cfg.p_groups = 1;
        const auto one = run_batch(st, cfg, sp, RunMode::grouped, 1);
        cfg.p_groups = 64;
        const auto many = run_batch(st, cfg, sp, RunMode::grouped, 1);
        const Result* runs[4] = {&ind.result, &one.result, &grouped.result, &many.result};
        double pair = 0.0;
        for (int a = 0; a < 4; ++a)
            for (int b = a + 1; b < 4; ++b) pair = std::max(pair, max_state_discrepancy(*runs[a], *runs[b]));
        expect(pair <= 1e-12, "criterion 4 invariance " + fmt(pair));
        Config cold = nbody_config(200);
        cold.start_mode = StartMode::cold;
        const auto c = run_batch(st, cold, sp, RunMode::grouped, 1);
        const int wi = one.result.max_iterations_used(), ci = c.result.max_iterations_used();
        expect(c.result.reports[0][0].converged && wi < ci && ci <= 100,
               "criterion 5 warm " + std::to_string(wi) + " cold " + std::to_string(ci));
        const Segments back = plan_segments(one.result.terminal_states[0], t_end, 0.0, mu_sun, SegmentPolicy::single, 200);
        Config bc = nbody_config(200);
        const auto bk = run_batch(one.result.terminal_states, bc, back, RunMode::grouped, 1);
        double ret = 0.0;
        for (std::size_t i = 0; i < st.size(); ++i) ret = std::max(ret, rel_state(bk.result.terminal_states[i], st[i]));
        expect(ret <= 1e-9, "criterion 9 symmetry " + fmt(ret));
    });
}

int main(int argc, char** argv) {
    const bool quick = argc > 1 && std::strcmp(argv[1], "--quick") == 0;
    chebyshev_cases();
    picard_cases();
    kepler_cases();
    dynamics_cases();
    augmentation_cases();
    propagator_cases();
    runner_cases();
    rk_cases();
    if (!quick) acceptance_cases();
    std::printf("SUMMARY %d %d\n", g_pass, g_fail);
    return g_fail == 0 ? 0 : 1;
}
