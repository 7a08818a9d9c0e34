// Drop-in check of the C++ API (include/pswarm.hpp -> libpswarm_b200.so, sm_100a)
// against the CPU oracle (oracle/pswarm_ref.hpp, test infrastructure).  Each case
// re-runs a property the reference's own suites hold (proj/tests/*.cpp) through the
// B200 path, written against the same API names the reference callers use.
// Output: "PASS name" / "FAIL name: detail" lines and "SUMMARY pass fail".
#include <cstdio>
#include <random>
#include <string>

#include "pswarm.hpp"
#include "pswarm_ref.hpp"

namespace ps = pswarm;
namespace rf = pswarm_ref;

namespace {
int n_pass = 0, n_fail = 0;
std::string detail;

void expect(bool ok, const std::string& what) {
    if (!ok && detail.empty()) detail = what;
}

template <typename Fn>
void run(const char* name, Fn&& fn) {
    detail.clear();
    try {
        fn();
    } catch (const std::exception& e) {
        detail = std::string("unexpected exception: ") + e.what();
    }
    if (detail.empty()) {
        ++n_pass;
        std::printf("PASS %s\n", name);
    } else {
        ++n_fail;
        std::printf("FAIL %s: %s\n", name, detail.c_str());
    }
    std::fflush(stdout);
}

std::string sci(double v) {
    char b[32];
    std::snprintf(b, sizeof b, "%.3e", v);
    return b;
}

std::vector<rf::State> to_ref(const std::vector<ps::StateVector>& v) {
    std::vector<rf::State> o;
    for (const auto& s : v) {
        rf::State x;
        x.epoch = s.epoch;
        x.r = {s.r.x(), s.r.y(), s.r.z()};
        x.v = {s.v.x(), s.v.y(), s.v.z()};
        o.push_back(x);
    }
    return o;
}

rf::Config ref_config(const ps::PropagationConfig& c) {
    rf::Config o;
    o.n_nodes = c.n_nodes;
    o.tolerance = c.tolerance;
    o.max_iterations = c.max_iterations;
    o.start_mode = c.start_mode == ps::StartMode::cold  ? rf::StartMode::cold
                   : c.start_mode == ps::StartMode::hot ? rf::StartMode::hot
                                                        : rf::StartMode::warm;
    o.force = c.force.kind == ps::ForceKind::two_body ? rf::reference_force(rf::ForceKind::two_body)
                                                      : rf::reference_force();
    if (c.force.kind == ps::ForceKind::n_body_1pn) o.force.kind = rf::ForceKind::n_body_1pn;
    o.p_groups = c.p_groups;
    return o;
}

/// max relative discrepancy of device vs oracle samples (runner.hpp:139-159 metric)
double discrepancy(const ps::PropagationResult& a, const rf::Result& b) {
    double w = 0.0;
    for (std::size_t i = 0; i < a.trajectories.size(); ++i)
        for (ps::Index j = 0; j < a.trajectories[i].rows(); ++j) {
            const auto& ta = a.trajectories[i];
            const auto& tb = b.trajectories[i];
            double dr = 0, dv = 0, rn = 0, vn = 0;
            for (int c = 0; c < 3; ++c) {
                dr += (ta(j, c) - tb(j, c)) * (ta(j, c) - tb(j, c));
                dv += (ta(j, c + 3) - tb(j, c + 3)) * (ta(j, c + 3) - tb(j, c + 3));
                rn += tb(j, c) * tb(j, c);
                vn += tb(j, c + 3) * tb(j, c + 3);
            }
            w = std::max({w, std::sqrt(dr / rn), std::sqrt(dv / vn)});
        }
    return w;
}

int max_iter_diff(const ps::PropagationResult& a, const rf::Result& b) {
    int w = 0;
    for (std::size_t s = 0; s < a.reports.size(); ++s)
        for (std::size_t g = 0; g < a.reports[s].size(); ++g)
            w = std::max(w, std::abs(a.reports[s][g].iterations - b.reports[s][g].iterations));
    return w;
}
}  // namespace

int main() {
    run("picard_update_polynomial_exactness", [] {  // test_picard.cpp:72-89
        const ps::Index n = 16;
        const auto grid = ps::build_grid(n, 0.0, 2.0);
        const auto mats = ps::build_matrices(n);
        double worst = 0.0;
        for (int d = 0; d <= 10; ++d) {
            ps::Mat f(n, 1);
            for (ps::Index j = 0; j < n; ++j) f(j, 0) = grid.omega2 * std::pow(grid.times[j], d);
            const ps::RowVec y0 = ps::RowVec::Ones(1);
            const ps::Mat y = ps::picard_update(mats, f, y0);
            for (ps::Index j = 0; j < n; ++j) {
                const double e = 1.0 + std::pow(grid.times[j], d + 1) / (d + 1);
                worst = std::max(worst, std::abs(y(j, 0) - e) / std::abs(e));
            }
        }
        expect(worst <= 1e-12, "exactness " + sci(worst));
    });
    run("picard_update_matches_oracle_n200", [] {
        const ps::Index n = 200, cols = 6 * 37;
        const auto mats = ps::cached_matrices(n);
        std::mt19937 rng(7);
        std::uniform_real_distribution<double> dist(-3.0, 3.0);
        ps::Mat f(n, cols);
        ps::RowVec y0(cols);
        for (ps::Index i = 0; i < f.size(); ++i) f.data()[i] = dist(rng);
        for (ps::Index c = 0; c < cols; ++c) y0[c] = 10.0 * dist(rng);
        const ps::Mat y = ps::picard_update(*mats, f, y0);
        rf::Mat rfm(n, cols), ry;
        std::copy(f.data(), f.data() + f.size(), rfm.v.begin());
        rf::picard_update_into(*rf::cached_ops(n), rfm, std::vector<double>(y0.data(), y0.data() + cols), ry);
        double scale = 0.0, diff = 0.0;
        for (ps::Index i = 0; i < y.size(); ++i) {
            scale = std::max(scale, std::abs(ry.v[i]));
            diff = std::max(diff, std::abs(y.data()[i] - ry.v[i]));
        }
        expect(diff / scale <= 1e-13, "relative " + sci(diff / scale));
    });
    run("force_block_singularity_coordinates", [] {  // test_dynamics.cpp:208-227
        const ps::Index n = 5;
        const auto grid = ps::build_grid(n, 0.0, 1.0e6);
        const auto table = ps::build_ephemeris_cache(ps::make_reference_bodies(), grid, ps::mu_sun_km3s2);
        auto states = ps::make_clone_batch(ps::make_reference_state(), 4, 1e-4);
        states[2].r = ps::Vec3(table.body_positions[0](0, 0), table.body_positions[0](0, 1), table.body_positions[0](0, 2));
        const auto guesses = ps::cold_start(states, n);
        const auto block = ps::assemble_block(states, grid, guesses);
        try {
            ps::eval_force_block(block, grid, table, ps::make_reference_force_model());
            expect(false, "no throw");
        } catch (const ps::SingularityError& e) {
            expect(std::string(e.what()).find("trajectory 2") != std::string::npos && e.body() == "venus-like",
                   std::string("tag: ") + e.what());
        }
    });
    run("block_iteration_error_single_perturbation", [] {  // test_augmentation.cpp:140-162
        const ps::Index n = 4;
        const auto grid = ps::build_grid(n, 0.0, 1.0);
        std::vector<ps::StateVector> st(2);
        for (auto& s : st) {
            s.r = ps::Vec3(1.0, 0.0, 0.0);
            s.v = ps::Vec3(0.0, 1.0, 0.0);
        }
        const auto guesses = ps::cold_start(st, n);
        const auto prev = ps::assemble_block(st, grid, guesses);
        auto cur = prev;
        const double delta = 0x1.0p-21;
        cur.data(2, ps::TrajectoryBlock::col_index(0, 1, 2)) += delta;
        const auto s = ps::block_iteration_error(cur, prev, ps::ErrorMode::relative);
        expect(std::abs(s.group_max - delta) <= 1e-15 && s.per_state_errors[0] == 0.0 &&
                   std::abs(s.per_state_errors[1] - delta) <= 1e-15,
               "errors");
    });
    run("warm_start_half_period_antipode", [] {  // test_propagator.cpp:27-44
        ps::StateVector s;
        s.r = ps::Vec3(1.3e8, 0.0, 0.0);
        const double speed = std::sqrt(ps::mu_sun_km3s2 / 1.3e8);
        s.v = ps::Vec3(0.0, speed, 0.0);
        const auto grid = ps::build_grid(21, 0.0, 0.5 * ps::osculating_period(s, ps::mu_sun_km3s2));
        const std::vector<ps::StateVector> states{s};
        const auto w = ps::warm_start(states, grid, ps::mu_sun_km3s2);
        const ps::Mat& g = w.guesses[0];
        expect(!w.cold_fallback[0] && g(0, 0) == s.r.x() && std::abs(g(20, 0) + 1.3e8) <= 1e-10 * 1.3e8 &&
                   std::abs(g(20, 4) + speed) <= 1e-10 * speed,
               "antipode");
    });
    run("propagate_exact_warm_start_fixed_point", [] {  // test_propagator.cpp:118-139
        ps::PropagationConfig cfg;
        cfg.n_nodes = 48;
        cfg.force = ps::make_reference_force_model(ps::ForceKind::two_body);
        const auto st = ps::make_clone_batch(ps::make_reference_state(), 3, 1e-6);
        const double period = ps::osculating_period(st[0], ps::mu_sun_km3s2);
        const auto sp = ps::plan_segments(st[0], 0.0, 0.5 * period, ps::mu_sun_km3s2, ps::SegmentPolicy::single, 48);
        const auto r = ps::propagate(st, ps::split_groups(3, 1), sp, cfg);
        expect(r.reports[0][0].converged && r.reports[0][0].iterations <= 3,
               "iterations " + std::to_string(r.reports[0][0].iterations));
        for (ps::Index j = 0; j < 48; ++j) {
            const auto e = ps::kepler_propagate(st[1], ps::mu_sun_km3s2, r.times[j]);
            const ps::Vec3 got(r.trajectories[1](j, 0), r.trajectories[1](j, 1), r.trajectories[1](j, 2));
            expect((got - e.r).norm() / e.r.norm() <= 1e-12, "conic");
        }
    });
    run("acceptance_2_two_body_full_period", [] {  // acceptance.cpp:78-124
        const auto s = ps::elements_to_state(ps::OrbitalElements{1.3e8, 0.2, 0.05, 0.4, 0.9, 0.0, 0.0},
                                             ps::mu_sun_km3s2, 0.0);
        const double period = ps::osculating_period(s, ps::mu_sun_km3s2);
        ps::PropagationConfig cfg;
        cfg.start_mode = ps::StartMode::cold;
        cfg.force = ps::make_reference_force_model(ps::ForceKind::two_body);
        const std::vector<ps::StateVector> batch{s};
        const auto r = ps::propagate(batch, ps::split_groups(1, 1),
                                     ps::plan_segments(s, 0.0, period, ps::mu_sun_km3s2, ps::SegmentPolicy::single, 200),
                                     cfg);
        double ws = 0, we = 0;
        const double e0 = ps::specific_energy(s, ps::mu_sun_km3s2);
        for (ps::Index j = 0; j < r.times.size(); ++j) {
            const auto want = ps::kepler_propagate(s, ps::mu_sun_km3s2, r.times[j]);
            ps::StateVector got;
            got.r = ps::Vec3(r.trajectories[0](j, 0), r.trajectories[0](j, 1), r.trajectories[0](j, 2));
            got.v = ps::Vec3(r.trajectories[0](j, 3), r.trajectories[0](j, 4), r.trajectories[0](j, 5));
            ws = std::max({ws, (got.r - want.r).norm() / want.r.norm(), (got.v - want.v).norm() / want.v.norm()});
            we = std::max(we, std::abs(ps::specific_energy(got, ps::mu_sun_km3s2) - e0) / std::abs(e0));
        }
        expect(r.reports[0][0].converged && ws <= 1e-10 && we <= 1e-11, "state " + sci(ws) + " energy " + sci(we));
    });
    run("run_batch_modes_match_oracle_nbody_n200", [] {  // test_runner.cpp:45-59 + parity
        ps::PropagationConfig cfg;
        cfg.force = ps::make_reference_force_model();
        cfg.p_groups = 8;
        const auto st = ps::make_clone_batch(ps::make_reference_state(), 64, 1e-5);
        const double period = ps::osculating_period(st[0], ps::mu_sun_km3s2);
        const auto sp = ps::plan_segments(st[0], 0.0, 0.87 * period, ps::mu_sun_km3s2, ps::SegmentPolicy::single, 200);
        const auto ind = ps::run_batch(st, cfg, sp, ps::RunMode::independent);
        const auto grp = ps::run_batch(st, cfg, sp, ps::RunMode::grouped);
        const auto rst = to_ref(st);
        rf::Segments rsp;
        rsp.boundaries = sp.boundaries;
        rsp.n_nodes = 200;
        const auto rind = rf::run_batch(rst, ref_config(cfg), rsp, rf::RunMode::independent, 4);
        const auto rgrp = rf::run_batch(rst, ref_config(cfg), rsp, rf::RunMode::grouped, 4);
        const double d1 = discrepancy(ind.result, rind.result), d2 = discrepancy(grp.result, rgrp.result);
        const int i1 = max_iter_diff(ind.result, rind.result), i2 = max_iter_diff(grp.result, rgrp.result);
        expect(d1 <= 1e-10 && d2 <= 1e-10 && i1 <= 1 && i2 <= 1,
               "independent " + sci(d1) + "/" + std::to_string(i1) + " grouped " + sci(d2) + "/" + std::to_string(i2));
        expect(ps::max_state_discrepancy(grp.result, ind.result) < 1e-12,
               "mode invariance " + sci(ps::max_state_discrepancy(grp.result, ind.result)));
    });
    run("extensions_1pn_hot_start_match_oracle", [] {  // BASELINE configs 3 and 5 through the C++ API
        const auto st = ps::make_clone_batch(ps::make_reference_state(), 16, 1e-5);
        const double period = ps::osculating_period(st[0], ps::mu_sun_km3s2);
        const auto sp = ps::plan_segments(st[0], 0.0, 2.5 * period, ps::mu_sun_km3s2, ps::SegmentPolicy::per_orbit, 128);
        rf::Segments rsp;
        rsp.boundaries = sp.boundaries;
        rsp.n_nodes = 128;
        const auto rst = to_ref(st);
        for (int variant = 0; variant < 2; ++variant) {
            ps::PropagationConfig cfg;
            cfg.n_nodes = 128;
            cfg.force = ps::make_reference_force_model();
            if (variant == 0) cfg.force.kind = ps::ForceKind::n_body_1pn;
            else cfg.start_mode = ps::StartMode::hot;
            const auto got = ps::run_batch(st, cfg, sp, ps::RunMode::independent);
            const auto want = rf::run_batch(rst, ref_config(cfg), rsp, rf::RunMode::independent, 4);
            const double d = discrepancy(got.result, want.result);
            const int di = max_iter_diff(got.result, want.result);
            expect(d <= 1e-10 && di <= 1, (variant ? "hot " : "1pn ") + sci(d) + "/" + std::to_string(di));
        }
    });
    run("propagate_nonconvergence_partial", [] {  // test_propagator.cpp:229-249
        ps::PropagationConfig cfg;
        cfg.n_nodes = 64;
        cfg.force = ps::make_reference_force_model(ps::ForceKind::two_body);
        cfg.start_mode = ps::StartMode::cold;
        cfg.max_iterations = 3;
        const auto st = ps::make_clone_batch(ps::make_reference_state(), 4, 1e-5);
        const double period = ps::osculating_period(st[0], ps::mu_sun_km3s2);
        const auto sp = ps::plan_segments(st[0], 0.0, 0.8 * period, ps::mu_sun_km3s2, ps::SegmentPolicy::single, 64);
        try {
            ps::propagate(st, ps::split_groups(4, 2), sp, cfg);
            expect(false, "no throw");
        } catch (const ps::PropagationIncompleteError& e) {
            expect(e.segment() == 0 && e.group() == 0 && e.partial() && !e.partial()->reports.at(0).at(0).converged,
                   "partial");
        }
    });
    run("propagate_timeout", [] {  // test_propagator.cpp:251-261
        ps::PropagationConfig cfg;
        cfg.n_nodes = 64;
        cfg.force = ps::make_reference_force_model();
        cfg.timeout_s = 1e-9;
        const auto st = ps::make_clone_batch(ps::make_reference_state(), 4, 1e-5);
        const auto sp = ps::plan_segments(st[0], 0.0, 1.0e6, ps::mu_sun_km3s2, ps::SegmentPolicy::single, 64);
        try {
            ps::propagate(st, ps::split_groups(4, 1), sp, cfg);
            expect(false, "no throw");
        } catch (const ps::TimeoutError&) {
        }
    });
    run("oracle_check_batch_acceptance_bar", [] {  // cli.hpp:238-261 + acceptance.cpp:148-172
        ps::PropagationConfig cfg;
        cfg.force = ps::make_reference_force_model();
        const auto st = ps::make_clone_batch(ps::make_reference_state(), 16, 1e-5);
        const double period = ps::osculating_period(st[0], ps::mu_sun_km3s2);
        const auto sp = ps::plan_segments(st[0], 0.0, 0.87 * period, ps::mu_sun_km3s2, ps::SegmentPolicy::single, 200);
        const auto out = ps::run_batch(st, cfg, sp, ps::RunMode::independent);
        ps::Mat per_node;
        const auto mx = ps::oracle_check_batch(st, out.result, cfg, {}, &per_node);
        double worst = 0.0;
        for (double x : mx) worst = std::max(worst, x);
        expect(mx.size() == 16 && worst <= 1e-9, "pc vs rkf78 " + std::to_string(worst));
        expect(per_node.rows() == static_cast<ps::Index>(out.result.times.size()) && per_node.cols() == 16,
               "per-node shape");
    });
    run("run_benchmark_rows", [] {  // runner.hpp:186-253: rows, baseline, cross-mode discrepancy
        ps::PropagationConfig cfg;
        cfg.force = ps::make_reference_force_model();
        cfg.p_groups = 4;
        const auto st = ps::make_clone_batch(ps::make_reference_state(), 16, 1e-5);
        const double period = ps::osculating_period(st[0], ps::mu_sun_km3s2);
        const auto sp = ps::plan_segments(st[0], 0.0, 0.5 * period, ps::mu_sun_km3s2, ps::SegmentPolicy::single, 64);
        const auto rep = ps::run_benchmark(st, cfg, sp, {1, 4},
                                           {ps::RunMode::independent, ps::RunMode::augmented_parallel,
                                            ps::RunMode::grouped},
                                           2);
        expect(rep.repeat == 2 && rep.rows.size() == 6, "rows " + std::to_string(rep.rows.size()));
        expect(rep.rows[0].speedup == 1.0 && rep.rows[0].max_discrepancy == 0.0 && rep.rows[0].groups == 16,
               "baseline row");
        double worst = 0.0;
        for (const auto& r : rep.rows) {
            expect(r.wall_time_s > 0.0 && r.max_iterations > 0, "row timing");
            worst = std::max(worst, r.max_discrepancy);
        }
        expect(rep.rows[2].groups == 1 && rep.rows[4].groups == 4, "group counts");
        expect(worst <= 1e-9, "cross-mode discrepancy " + sci(worst));  // test_runner.cpp:45-59 (mode invariance)
        bool threw = false;
        try {
            ps::run_benchmark(st, cfg, sp, {1}, {ps::RunMode::independent}, 0);
        } catch (const ps::InvalidPlanError&) {
            threw = true;
        }
        expect(threw, "repeat 0 must throw");
    });
    run("run_batch_devices_knob_matches_one_device", [] {  // SURVEY §8a13 devices knob, runner.hpp:111-135
        ps::PropagationConfig cfg;
        cfg.force = ps::make_reference_force_model();
        cfg.p_groups = 7;
        const auto st = ps::make_clone_batch(ps::make_reference_state(), 61, 1e-4);
        const double period = ps::osculating_period(st[0], ps::mu_sun_km3s2);
        const auto sp = ps::plan_segments(st[0], 0.0, 1.6 * period, ps::mu_sun_km3s2, ps::SegmentPolicy::per_orbit, 64);
        int dev = 0;
        if (const char* d = std::getenv("PSWARM_DEVICE")) dev = std::atoi(d);
        const std::vector<int> two{dev, dev}, three{dev, dev, dev};  // several contexts on one GPU
        for (auto mode : {ps::RunMode::independent, ps::RunMode::grouped, ps::RunMode::augmented_parallel}) {
            const auto one = ps::run_batch(st, cfg, sp, mode, 1);
            for (const auto* devs : {&two, &three}) {
                const auto many = ps::run_batch(st, cfg, sp, mode, 1, *devs);
                bool same = one.result.terminal_states.size() == many.result.terminal_states.size();
                for (std::size_t i = 0; same && i < st.size(); ++i)
                    same = one.result.terminal_states[i].r == many.result.terminal_states[i].r &&
                           one.result.terminal_states[i].v == many.result.terminal_states[i].v &&
                           one.result.trajectories[i] == many.result.trajectories[i];
                for (std::size_t sg = 0; same && sg < one.result.reports.size(); ++sg)
                    for (std::size_t g = 0; same && g < one.result.reports[sg].size(); ++g)
                        same = one.result.reports[sg][g].iterations == many.result.reports[sg][g].iterations &&
                               one.result.reports[sg][g].per_iteration_errors ==
                                   many.result.reports[sg][g].per_iteration_errors;
                expect(same, "multi-device result differs from one device (mode " + ps::to_string(mode) + ", " +
                                 std::to_string(devs->size()) + " shards)");
            }
        }
    });
    std::printf("SUMMARY %d %d\n", n_pass, n_fail);
    return n_fail == 0 ? 0 : 1;
}
