// C API over the REFERENCE ITSELF (/root/reference/proj/include/pswarm, compiled
// unchanged against oracle/eigen_shim) — TEST INFRASTRUCTURE ONLY, built into
// oracle/_ref/libpswarm_refsrc.so by oracle/Makefile.ref.  It exports the same
// `ref_*` entry points as oracle/oracle_capi.cpp (the restatement), with the same
// plain-C descriptors (include/pswarm_gpu.h), so oracle/oracle_py.Oracle can load
// either library:
//   * tests pin the restatement (pswarm_ref.hpp) to the reference's own code;
//   * bench.py times the reference's own run_batch as the CPU baseline
//     (cpu_baseline.kind = "reference").
// The reference has neither the EIH 1PN force nor hot start:
// those configurations are rejected with PSWARM_ERR_GENERIC.
#include <chrono>
#include <cstdio>
#include <cstring>
#include <thread>

#include "pswarm/oracle.hpp"
#include "pswarm/runner.hpp"
#include "pswarm/synthetic.hpp"
#include "pswarm_gpu.h"

using namespace pswarm;

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
    } catch (const PropagationIncompleteError& e) {
        set_err(err, PSWARM_ERR_INCOMPLETE, e.what());
        if (err) {
            err->segment = e.segment();
            err->group = e.group();
        }
        return PSWARM_ERR_INCOMPLETE;
    } catch (const DivergenceError& e) {
        set_err(err, PSWARM_ERR_DIVERGENCE, e.what());
        if (err) {
            err->node = e.node();
            err->column = e.column();
        }
        return PSWARM_ERR_DIVERGENCE;
    } catch (const SingularityError& e) {
        set_err(err, PSWARM_ERR_SINGULARITY, e.what());
        if (err) std::snprintf(err->body_name, sizeof(err->body_name), "%s", e.body().c_str());
        return PSWARM_ERR_SINGULARITY;
    } catch (const CoverageError& e) {
        set_err(err, PSWARM_ERR_COVERAGE, e.what());
        if (err) err->value = e.epoch();
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
    } catch (const OracleError& e) {
        set_err(err, PSWARM_ERR_ORACLE, e.what());
        return PSWARM_ERR_ORACLE;
    } catch (const std::exception& e) {
        set_err(err, PSWARM_ERR_GENERIC, e.what());
        return PSWARM_ERR_GENERIC;
    }
}

StateVector state_from(const double* s) {
    StateVector x;
    x.epoch = s[0];
    x.r = Vec3(s[1], s[2], s[3]);
    x.v = Vec3(s[4], s[5], s[6]);
    return x;
}

void state_to(const StateVector& s, double* out) {
    out[0] = s.epoch;
    for (int c = 0; c < 3; ++c) {
        out[1 + c] = s.r[c];
        out[4 + c] = s.v[c];
    }
}

std::vector<StateVector> states_from(int64_t n, const double* s) {
    std::vector<StateVector> v(static_cast<std::size_t>(n));
    for (int64_t i = 0; i < n; ++i) v[static_cast<std::size_t>(i)] = state_from(s + 7 * i);
    return v;
}

BodySpec body_from(const pswarm_body& b) {
    BodySpec o;
    o.name = b.name ? b.name : "";
    o.mu = b.mu;
    if (b.kind == 0) {
        OrbitalElements el;
        el.a = b.elements[0];
        el.e = b.elements[1];
        el.i = b.elements[2];
        el.raan = b.elements[3];
        el.argp = b.elements[4];
        el.m0 = b.elements[5];
        el.epoch = b.elements[6];
        o.ephemeris = el;
    } else {
        ChebyshevEphemeris eph;
        for (int32_t s = 0; s < b.n_segments; ++s) {
            ChebyshevSegment seg;
            seg.t_start = b.seg_bounds[2 * s];
            seg.t_end = b.seg_bounds[2 * s + 1];
            const double* c = b.coeffs + static_cast<std::size_t>(s) * 3 * b.n_coeffs;
            seg.coeffs_x = Eigen::Map<const Vec>(c, b.n_coeffs);
            seg.coeffs_y = Eigen::Map<const Vec>(c + b.n_coeffs, b.n_coeffs);
            seg.coeffs_z = Eigen::Map<const Vec>(c + 2 * b.n_coeffs, b.n_coeffs);
            eph.segments.push_back(std::move(seg));
        }
        o.ephemeris = std::move(eph);
    }
    return o;
}

PropagationConfig config_from(const pswarm_config& c) {
    if (c.force_kind == 2) throw Error("reference: the EIH 1PN force model is an extension (SPEC.md:17)");
    if (c.start_mode == 2) throw Error("reference: hot start is an extension (SPEC.md:350)");
    PropagationConfig o;
    o.n_nodes = c.n_nodes;
    o.tolerance = c.tolerance;
    o.error_mode = c.error_mode == 1 ? ErrorMode::absolute : ErrorMode::relative;
    o.max_iterations = c.max_iterations;
    o.start_mode = c.start_mode == 1 ? StartMode::cold : StartMode::warm;
    o.segment_policy = c.segment_policy == 1 ? SegmentPolicy::per_orbit : SegmentPolicy::single;
    o.max_segment_periods = c.max_segment_periods;
    o.force.kind = c.force_kind == 1 ? ForceKind::n_body : ForceKind::two_body;
    o.force.central_mu = c.central_mu;
    for (int32_t b = 0; b < c.n_bodies; ++b) o.force.bodies.push_back(body_from(c.bodies[b]));
    o.force.proximity_floor_km = c.proximity_floor_km;
    o.p_groups = c.p_groups;
    o.timeout_s = c.timeout_s;
    return o;
}

SegmentPlan segments_from(int64_t nb, const double* b, int64_t n) {
    SegmentPlan s;
    s.boundaries.assign(b, b + nb);
    s.n_nodes = n;
    s.direction = (nb >= 2 && b[nb - 1] < b[0]) ? Direction::backward : Direction::forward;
    return s;
}

void export_result(const PropagationResult& r, int64_t max_it, pswarm_outputs* out, bool complete) {
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
            std::memcpy(out->samples + i * R * 6, r.trajectories[static_cast<std::size_t>(i)].data(),
                        sizeof(double) * static_cast<std::size_t>(R * 6));
    if (out->terminal_states && complete)
        for (int64_t i = 0; i < M; ++i) state_to(r.terminal_states[static_cast<std::size_t>(i)], out->terminal_states + 7 * i);
    for (std::size_t s = 0; s < r.reports.size(); ++s) {
        for (int64_t g = 0; g < P; ++g) {
            const IterationReport& q = r.reports[s][static_cast<std::size_t>(g)];
            const int64_t k = static_cast<int64_t>(s) * P + g;
            if (out->iterations) out->iterations[k] = q.iterations;
            if (out->final_error) out->final_error[k] = q.final_error;
            if (out->converged) out->converged[k] = q.converged ? 1 : 0;
            if (out->error_history)
                for (int64_t it = 0; it < max_it; ++it)
                    out->error_history[k * max_it + it] =
                        it < static_cast<int64_t>(q.per_iteration_errors.size())
                            ? q.per_iteration_errors[static_cast<std::size_t>(it)]
                            : std::nan("");
        }
    }
    if (out->cold_fallback) {
        for (const auto& w : r.warnings) {  // propagator.hpp:262-269, runner.hpp:101
            long long a = -1, b = -1, c = -1;
            if (std::sscanf(w.c_str(), "trajectory %lld: segment %lld, trajectory %lld", &a, &b, &c) == 3)
                out->cold_fallback[b * M + a] = 1;
            else if (std::sscanf(w.c_str(), "segment %lld, trajectory %lld", &b, &c) == 2)
                out->cold_fallback[b * M + c] = 1;
        }
    }
}

using Clock = std::chrono::steady_clock;

}  // namespace

extern "C" {

int32_t ref_propagate(int64_t n_states, const double* states, int64_t n_groups, const int64_t* group_sizes,
                      int64_t n_boundaries, const double* boundaries, int64_t n_nodes, const pswarm_config* config,
                      int32_t group_workers, int32_t inner_workers, pswarm_outputs* out, pswarm_error* err) {
    return guarded(err, [&] {
        const auto st = states_from(n_states, states);
        const GroupingPlan plan = plan_from_sizes(std::vector<Index>(group_sizes, group_sizes + n_groups));
        const SegmentPlan sp = segments_from(n_boundaries, boundaries, n_nodes);
        const PropagationConfig cfg = config_from(*config);
        ExecutionPolicy ex;
        ex.group_workers = static_cast<unsigned>(std::max(1, group_workers));
        ex.inner_workers = static_cast<unsigned>(std::max(1, inner_workers));
        const auto t0 = Clock::now();
        try {
            const PropagationResult r = propagate(st, plan, sp, cfg, ex);
            if (out) out->wall_s = std::chrono::duration<double>(Clock::now() - t0).count();
            export_result(r, cfg.max_iterations, out, true);
        } catch (const PropagationIncompleteError& e) {
            if (out) out->wall_s = std::chrono::duration<double>(Clock::now() - t0).count();
            export_result(*e.partial(), cfg.max_iterations, out, false);
            throw;
        }
    });
}

int32_t ref_run_batch(int64_t n_states, const double* states, int64_t n_boundaries, const double* boundaries,
                      int64_t n_nodes, const pswarm_config* config, int32_t mode, int32_t workers,
                      pswarm_outputs* out, pswarm_error* err) {
    return guarded(err, [&] {
        const auto st = states_from(n_states, states);
        const SegmentPlan sp = segments_from(n_boundaries, boundaries, n_nodes);
        const PropagationConfig cfg = config_from(*config);
        const RunMode rm = mode == 0   ? RunMode::independent
                           : mode == 1 ? RunMode::augmented_sequential
                           : mode == 2 ? RunMode::augmented_parallel
                                       : RunMode::grouped;
        try {
            const RunOutcome o = run_batch(st, cfg, sp, rm, static_cast<unsigned>(workers < 0 ? 0 : workers));
            if (out) out->wall_s = o.wall_time_s;
            export_result(o.result, cfg.max_iterations, out, true);
        } catch (const PropagationIncompleteError& e) {
            export_result(*e.partial(), cfg.max_iterations, out, false);
            throw;
        }
    });
}

int32_t ref_picard_update(int64_t n_nodes, int64_t n_cols, const double* force, const double* initial_row,
                          double* out, pswarm_error* err) {
    return guarded(err, [&] {
        const auto mats = cached_matrices(n_nodes);
        const Mat f = Eigen::Map<const Mat>(force, n_nodes, n_cols);
        const RowVec y0 = Eigen::Map<const RowVec>(initial_row, n_cols);
        Mat y;
        picard_update_into(*mats, f, y0, y, nullptr);
        std::memcpy(out, y.data(), sizeof(double) * static_cast<std::size_t>(n_nodes * n_cols));
    });
}

int32_t ref_build_operators(int64_t n_nodes, double* update_op, double* anchor_op, pswarm_error* err) {
    return guarded(err, [&] {
        const auto m = build_matrices(n_nodes);
        std::memcpy(update_op, m.update_op.data(), sizeof(double) * static_cast<std::size_t>(n_nodes * n_nodes));
        std::memcpy(anchor_op, m.anchor_op.data(), sizeof(double) * static_cast<std::size_t>(n_nodes));
    });
}

void ref_make_clone_batch(const double* base, int64_t count, double spread, uint64_t seed, double* out) {
    const auto v = make_clone_batch(state_from(base), count, spread, seed);
    for (std::size_t i = 0; i < v.size(); ++i) state_to(v[i], out + 7 * i);
}

void ref_reference_state(double* out) { state_to(make_reference_state(), out); }

unsigned ref_hardware_threads(void) { return std::max(1u, std::thread::hardware_concurrency()); }

/// 1 = this library runs the reference's own sources (0 in liboracle.so's restatement)
int32_t ref_is_reference_source(void) { return 1; }

}  // extern "C"
