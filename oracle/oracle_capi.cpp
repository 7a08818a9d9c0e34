// C API over the CPU oracle (oracle/pswarm_ref.hpp) for the Python test suite
// and bench.py's CPU baseline.  TEST INFRASTRUCTURE ONLY — never linked by the
// product.  Entry points mirror include/pswarm_gpu.h one for one with a `ref_`
// prefix and take the same plain-C descriptors, so a parity test calls both
// sides with identical arguments.
#include <cstring>

#include "pswarm_gpu.h"
#include "pswarm_ref.hpp"

using namespace pswarm_ref;

namespace {

void set_err(pswarm_error* err, int32_t status, const std::string& msg) {
    if (!err) return;
    std::memset(err, 0, sizeof(*err));
    err->status = status;
    err->body = -1;
    err->segment = err->group = err->node = err->column = err->trajectory = -1;
    std::snprintf(err->message, sizeof(err->message), "%s", msg.c_str());
}

template <typename Fn>
int32_t guarded(pswarm_error* err, Fn&& fn) {
    if (err) set_err(err, PSWARM_OK, "");
    try {
        fn();
        return PSWARM_OK;
    } catch (const IncompleteError& e) {
        set_err(err, PSWARM_ERR_INCOMPLETE, e.what());
        if (err) {
            err->segment = e.segment;
            err->group = e.group;
        }
        return PSWARM_ERR_INCOMPLETE;
    } catch (const DivergenceError& e) {
        set_err(err, PSWARM_ERR_DIVERGENCE, e.what());
        if (err) {
            err->node = e.node;
            err->column = e.column;
        }
        return PSWARM_ERR_DIVERGENCE;
    } catch (const SingularityError& e) {
        set_err(err, PSWARM_ERR_SINGULARITY, e.what());
        if (err) std::snprintf(err->body_name, sizeof(err->body_name), "%s", e.body.c_str());
        return PSWARM_ERR_SINGULARITY;
    } catch (const CoverageError& e) {
        set_err(err, PSWARM_ERR_COVERAGE, e.what());
        if (err) err->value = e.epoch;
        return PSWARM_ERR_COVERAGE;
    } catch (const InvalidSpanError& e) {
        set_err(err, PSWARM_ERR_INVALID_SPAN, e.what());
        return PSWARM_ERR_INVALID_SPAN;
    } catch (const InvalidSizeError& e) {
        set_err(err, PSWARM_ERR_INVALID_SIZE, e.what());
        return PSWARM_ERR_INVALID_SIZE;
    } catch (const ShapeError& e) {
        set_err(err, PSWARM_ERR_SHAPE, e.what());
        return PSWARM_ERR_SHAPE;
    } catch (const AlignmentError& e) {
        set_err(err, PSWARM_ERR_ALIGNMENT, e.what());
        return PSWARM_ERR_ALIGNMENT;
    } catch (const NonEllipticError& e) {
        set_err(err, PSWARM_ERR_NON_ELLIPTIC, e.what());
        return PSWARM_ERR_NON_ELLIPTIC;
    } catch (const SolverError& e) {
        set_err(err, PSWARM_ERR_SOLVER, e.what());
        return PSWARM_ERR_SOLVER;
    } catch (const InvalidPlanError& e) {
        set_err(err, PSWARM_ERR_INVALID_PLAN, e.what());
        return PSWARM_ERR_INVALID_PLAN;
    } catch (const TimeoutError& e) {
        set_err(err, PSWARM_ERR_TIMEOUT, e.what());
        return PSWARM_ERR_TIMEOUT;
    } catch (const std::exception& e) {
        set_err(err, PSWARM_ERR_GENERIC, e.what());
        return PSWARM_ERR_GENERIC;
    }
}

State state_from(const double* s) {
    State x;
    x.epoch = s[0];
    x.r = {s[1], s[2], s[3]};
    x.v = {s[4], s[5], s[6]};
    return x;
}

void state_to(const State& s, double* out) {
    out[0] = s.epoch;
    out[1] = s.r.x; out[2] = s.r.y; out[3] = s.r.z;
    out[4] = s.v.x; out[5] = s.v.y; out[6] = s.v.z;
}

std::vector<State> states_from(int64_t n, const double* s) {
    std::vector<State> v(static_cast<std::size_t>(n));
    for (int64_t i = 0; i < n; ++i) v[i] = state_from(s + 7 * i);
    return v;
}

Body body_from(const pswarm_body& b) {
    Body o;
    o.name = b.name ? b.name : "";
    o.mu = b.mu;
    if (b.kind == 0) {
        o.el = {b.elements[0], b.elements[1], b.elements[2], b.elements[3], b.elements[4], b.elements[5], b.elements[6]};
    } else {
        o.tabulated = true;
        for (int32_t s = 0; s < b.n_segments; ++s) {
            ChebSeg seg;
            seg.t_start = b.seg_bounds[2 * s];
            seg.t_end = b.seg_bounds[2 * s + 1];
            const double* c = b.coeffs + static_cast<std::size_t>(s) * 3 * b.n_coeffs;
            seg.cx.assign(c, c + b.n_coeffs);
            seg.cy.assign(c + b.n_coeffs, c + 2 * b.n_coeffs);
            seg.cz.assign(c + 2 * b.n_coeffs, c + 3 * b.n_coeffs);
            o.segs.push_back(std::move(seg));
        }
    }
    return o;
}

Config config_from(const pswarm_config& c) {
    Config o;
    o.n_nodes = c.n_nodes;
    o.tolerance = c.tolerance;
    o.error_mode = c.error_mode == 1 ? ErrorMode::absolute : ErrorMode::relative;
    o.max_iterations = c.max_iterations;
    o.start_mode = c.start_mode == 1 ? StartMode::cold : c.start_mode == 2 ? StartMode::hot : StartMode::warm;
    o.segment_policy = c.segment_policy == 1 ? SegmentPolicy::per_orbit : SegmentPolicy::single;
    o.max_segment_periods = c.max_segment_periods;
    o.force.kind = c.force_kind == 1   ? ForceKind::n_body
                   : c.force_kind == 2 ? ForceKind::n_body_1pn
                                       : ForceKind::two_body;
    o.force.c_light = c.c_light > 0.0 ? c.c_light : 299792.458;
    o.force.central_mu = c.central_mu;
    for (int32_t b = 0; b < c.n_bodies; ++b) o.force.bodies.push_back(body_from(c.bodies[b]));
    o.force.proximity_floor_km = c.proximity_floor_km;
    o.p_groups = c.p_groups;
    o.timeout_s = c.timeout_s;
    return o;
}

Segments segments_from(int64_t nb, const double* b, int64_t n) {
    Segments s;
    s.boundaries.assign(b, b + nb);
    s.n_nodes = n;
    s.direction = (nb >= 2 && b[nb - 1] < b[0]) ? Direction::backward : Direction::forward;
    return s;
}

void export_result(const Result& r, int64_t max_it, pswarm_outputs* out, bool complete) {
    if (!out) return;
    const int64_t M = static_cast<int64_t>(r.trajectories.size());
    const int64_t P = r.plan.groups();
    const int64_t R = static_cast<int64_t>(r.times.size());
    out->segments_reported = static_cast<int64_t>(r.reports.size());
    out->segments_completed = complete ? static_cast<int64_t>(r.reports.size())
                                       : std::max<int64_t>(0, static_cast<int64_t>(r.reports.size()) - 1);
    if (out->times)
        for (int64_t j = 0; j < R; ++j) out->times[j] = r.times[j];
    if (out->samples)
        for (int64_t i = 0; i < M; ++i)
            std::memcpy(out->samples + i * R * 6, r.trajectories[i].v.data(), sizeof(double) * R * 6);
    if (out->terminal_states && complete)
        for (int64_t i = 0; i < M; ++i) state_to(r.terminal_states[i], out->terminal_states + 7 * i);
    for (std::size_t s = 0; s < r.reports.size(); ++s) {
        for (int64_t g = 0; g < P; ++g) {
            const Report& q = r.reports[s][g];
            const int64_t k = static_cast<int64_t>(s) * P + g;
            if (out->iterations) out->iterations[k] = q.iterations;
            if (out->final_error) out->final_error[k] = q.final_error;
            if (out->converged) out->converged[k] = q.converged ? 1 : 0;
            if (out->error_history)
                for (int64_t it = 0; it < max_it; ++it)
                    out->error_history[k * max_it + it] =
                        it < static_cast<int64_t>(q.history.size()) ? q.history[it] : std::nan("");
        }
    }
    if (out->cold_fallback) {
        // warnings carry "segment s, trajectory i" (propagator.hpp:262-269); in
        // independent mode they are prefixed "trajectory i: " (runner.hpp:101).
        for (const auto& w : r.warnings) {
            long long a = -1, b = -1, c = -1;
            if (std::sscanf(w.c_str(), "trajectory %lld: segment %lld, trajectory %lld", &a, &b, &c) == 3)
                out->cold_fallback[b * M + a] = 1;
            else if (std::sscanf(w.c_str(), "segment %lld, trajectory %lld", &b, &c) == 2)
                out->cold_fallback[b * M + c] = 1;
        }
    }
}

}  // namespace

extern "C" {

int32_t ref_propagate(int64_t n_states, const double* states, int64_t n_groups, const int64_t* group_sizes,
                      int64_t n_boundaries, const double* boundaries, int64_t n_nodes, const pswarm_config* config,
                      int32_t group_workers, int32_t inner_workers, pswarm_outputs* out, pswarm_error* err) {
    return guarded(err, [&] {
        const auto st = states_from(n_states, states);
        const Plan plan = plan_from_sizes(std::vector<Index>(group_sizes, group_sizes + n_groups));
        const Segments sp = segments_from(n_boundaries, boundaries, n_nodes);
        const Config cfg = config_from(*config);
        Exec ex;
        ex.group_workers = static_cast<unsigned>(std::max(1, group_workers));
        ex.inner_workers = static_cast<unsigned>(std::max(1, inner_workers));
        const auto t0 = Clock::now();
        try {
            const Result r = propagate(st, plan, sp, cfg, ex);
            if (out) out->wall_s = std::chrono::duration<double>(Clock::now() - t0).count();
            export_result(r, cfg.max_iterations, out, true);
        } catch (const IncompleteError& e) {
            if (out) out->wall_s = std::chrono::duration<double>(Clock::now() - t0).count();
            export_result(*e.partial, cfg.max_iterations, out, false);
            throw;
        }
    });
}

int32_t ref_run_batch(int64_t n_states, const double* states, int64_t n_boundaries, const double* boundaries,
                      int64_t n_nodes, const pswarm_config* config, int32_t mode, int32_t workers,
                      pswarm_outputs* out, pswarm_error* err) {
    return guarded(err, [&] {
        const auto st = states_from(n_states, states);
        const Segments sp = segments_from(n_boundaries, boundaries, n_nodes);
        const Config cfg = config_from(*config);
        const RunMode rm = mode == 0 ? RunMode::independent
                           : mode == 1 ? RunMode::augmented_sequential
                           : mode == 2 ? RunMode::augmented_parallel
                                       : RunMode::grouped;
        try {
            const Outcome o = run_batch(st, cfg, sp, rm, static_cast<unsigned>(workers < 0 ? 0 : workers));
            if (out) out->wall_s = o.wall_time_s;
            export_result(o.result, cfg.max_iterations, out, true);
        } catch (const IncompleteError& e) {
            export_result(*e.partial, cfg.max_iterations, out, false);
            throw;
        }
    });
}

int32_t ref_picard_update(int64_t n_nodes, int64_t n_cols, const double* force, const double* initial_row,
                          double* out, pswarm_error* err) {
    return guarded(err, [&] {
        const auto ops = cached_ops(n_nodes);
        Mat f(n_nodes, n_cols);
        std::memcpy(f.v.data(), force, sizeof(double) * n_nodes * n_cols);
        Mat y;
        picard_update_into(*ops, f, std::vector<double>(initial_row, initial_row + n_cols), y);
        std::memcpy(out, y.v.data(), sizeof(double) * n_nodes * n_cols);
    });
}

/// update_op [N][N] and anchor_op [N] exactly as the oracle builds them.
int32_t ref_build_operators(int64_t n_nodes, double* update_op, double* anchor_op, pswarm_error* err) {
    return guarded(err, [&] {
        const auto ops = cached_ops(n_nodes);
        if (update_op) std::memcpy(update_op, ops->update_op.v.data(), sizeof(double) * n_nodes * n_nodes);
        if (anchor_op) std::memcpy(anchor_op, ops->anchor_op.data(), sizeof(double) * n_nodes);
    });
}

int32_t ref_eval_force_block(int64_t n_nodes, int64_t group_size, const double* y, double omega2, int32_t force_kind,
                             double central_mu, int32_t n_bodies, const double* body_positions, const double* body_mus,
                             const char* const* body_names, double floor_km, double* force, pswarm_error* err) {
    return guarded(err, [&] {
        Grid g;
        g.n = n_nodes;
        g.omega2 = omega2;
        g.times.assign(static_cast<std::size_t>(n_nodes), 0.0);
        EphTable t;
        t.node_times = g.times;
        t.central_mu = central_mu;
        for (int32_t b = 0; b < n_bodies; ++b) {
            Mat p(n_nodes, 3);
            std::memcpy(p.v.data(), body_positions + static_cast<std::size_t>(b) * n_nodes * 3,
                        sizeof(double) * n_nodes * 3);
            t.pos.push_back(std::move(p));
            t.mus.push_back(body_mus[b]);
            t.names.push_back(body_names && body_names[b] ? body_names[b] : "");
        }
        ForceConfig cfg;
        cfg.kind = force_kind == 1 ? ForceKind::n_body : ForceKind::two_body;
        cfg.central_mu = central_mu;
        cfg.proximity_floor_km = floor_km;
        Mat ym(n_nodes, 6 * group_size), f;
        std::memcpy(ym.v.data(), y, sizeof(double) * ym.v.size());
        eval_force_block(ym, group_size, g, t, cfg, f);
        std::memcpy(force, f.v.data(), sizeof(double) * f.v.size());
    });
}

int32_t ref_block_iteration_error(int64_t n_nodes, int64_t group_size, const double* cur, const double* prev,
                                  int32_t error_mode, double* per_state, double* group_max, pswarm_error* err) {
    return guarded(err, [&] {
        Mat c(n_nodes, 6 * group_size), p(n_nodes, 6 * group_size);
        std::memcpy(c.v.data(), cur, sizeof(double) * c.v.size());
        std::memcpy(p.v.data(), prev, sizeof(double) * p.v.size());
        double gm = 0.0;
        const auto per =
            block_iteration_error(c, p, group_size, error_mode == 1 ? ErrorMode::absolute : ErrorMode::relative, &gm);
        if (per_state) std::memcpy(per_state, per.data(), sizeof(double) * per.size());
        if (group_max) *group_max = gm;
    });
}

int32_t ref_warm_start(int64_t n_states, const double* states, int64_t n_nodes, const double* times,
                       double central_mu, double* guesses, uint8_t* cold_fallback, pswarm_error* err) {
    return guarded(err, [&] {
        Grid g;
        g.n = n_nodes;
        g.times.assign(times, times + n_nodes);
        for (int64_t i = 0; i < n_states; ++i) {
            bool fb = false;
            const Mat w = warm_guess(state_from(states + 7 * i), g, central_mu, &fb);
            std::memcpy(guesses + i * n_nodes * 6, w.v.data(), sizeof(double) * n_nodes * 6);
            if (cold_fallback) cold_fallback[i] = fb ? 1 : 0;
        }
    });
}

int32_t ref_kepler_propagate(const double* state, double mu, double dt, double* out, pswarm_error* err) {
    return guarded(err, [&] { state_to(kepler_propagate(state_from(state), mu, dt), out); });
}

int32_t ref_elements_to_state(const double* elements, double mu, double t, double* out, pswarm_error* err) {
    return guarded(err, [&] {
        const Elements el{elements[0], elements[1], elements[2], elements[3], elements[4], elements[5], elements[6]};
        state_to(elements_to_state(el, mu, t), out);
    });
}

int32_t ref_osculating_period(const double* state, double mu, double* period, pswarm_error* err) {
    return guarded(err, [&] { *period = osculating_period(state_from(state), mu); });
}

/// plan_segments; boundaries must hold room for max_boundaries values.
int32_t ref_plan_segments(const double* representative, double t_start, double t_end, double mu, int32_t policy,
                          int64_t n_nodes, double max_periods, int64_t max_boundaries, double* boundaries,
                          int64_t* n_boundaries, pswarm_error* err) {
    return guarded(err, [&] {
        const Segments s = plan_segments(state_from(representative), t_start, t_end, mu,
                                         policy == 1 ? SegmentPolicy::per_orbit : SegmentPolicy::single, n_nodes,
                                         max_periods);
        if (static_cast<int64_t>(s.boundaries.size()) > max_boundaries) throw Error("ref_plan_segments: buffer too small");
        std::memcpy(boundaries, s.boundaries.data(), sizeof(double) * s.boundaries.size());
        *n_boundaries = static_cast<int64_t>(s.boundaries.size());
    });
}

int32_t ref_build_grid(int64_t n_nodes, double t0, double t1, double* times, double* omega2, pswarm_error* err) {
    return guarded(err, [&] {
        const Grid g = build_grid(n_nodes, t0, t1);
        std::memcpy(times, g.times.data(), sizeof(double) * n_nodes);
        if (omega2) *omega2 = g.omega2;
    });
}

/// Ephemeris table [B][N][3] for the analytic / tabulated bodies at `times`.
int32_t ref_body_positions(int32_t n_bodies, const pswarm_body* bodies, double central_mu, int64_t n_times,
                           const double* times, double* out, pswarm_error* err) {
    return guarded(err, [&] {
        for (int32_t b = 0; b < n_bodies; ++b) {
            const Body bd = body_from(bodies[b]);
            for (int64_t j = 0; j < n_times; ++j) {
                const V3 p = body_position(bd, central_mu, times[j]);
                double* o = out + (static_cast<std::size_t>(b) * n_times + j) * 3;
                o[0] = p.x;
                o[1] = p.y;
                o[2] = p.z;
            }
        }
    });
}

void ref_make_clone_batch(const double* base, int64_t count, double spread, uint64_t seed, double* out) {
    const auto v = clone_batch(state_from(base), count, spread, seed);
    for (int64_t i = 0; i < count; ++i) state_to(v[i], out + 7 * i);
}

void ref_reference_state(double* out) { state_to(reference_state(), out); }

/// Independent RKF7(8) samples of one trajectory at `times` (oracle.hpp:136-150).
int32_t ref_rk_sample(const double* state, const pswarm_config* config, int64_t n_times, const double* times,
                      double* out, pswarm_error* err) {
    return guarded(err, [&] {
        const Config cfg = config_from(*config);
        const Mat m = rk_sample(state_from(state), nbody_deriv(cfg.force), std::vector<double>(times, times + n_times));
        std::memcpy(out, m.v.data(), sizeof(double) * m.v.size());
    });
}

unsigned ref_hardware_threads(void) { return std::max(1u, std::thread::hardware_concurrency()); }

}  // extern "C"
