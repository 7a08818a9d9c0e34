#pragma once
// Batch propagation — the drop-in boundary (reference: propagator.hpp:24-347).
// propagate() validates on the host, then hands the whole multi-segment solve to
// the device through the C-ABI (pswarm_propagate): warm start, every Picard
// iteration, per-group convergence masking and segment chaining stay on the GPU;
// the host receives terminal states, node samples and per-(segment, group) reports.

#include <chrono>
#include <condition_variable>
#include <cstdint>
#include <functional>
#include <mutex>
#include <cmath>
#include <memory>
#include <optional>
#include <span>
#include <string>
#include <thread>
#include <utility>
#include <vector>

#include "pswarm/augment.hpp"
#include "pswarm/block.hpp"
#include "pswarm/chebyshev.hpp"
#include "pswarm/device.hpp"
#include "pswarm/ephemeris.hpp"
#include "pswarm/errors.hpp"
#include "pswarm/force_model.hpp"
#include "pswarm/kepler.hpp"
#include "pswarm/pc_matrices.hpp"
#include "pswarm/reduction.hpp"
#include "pswarm/types.hpp"

namespace pswarm {

enum class StartMode { warm, cold, hot };  // hot: EXTENSION (Macomber hot start)
enum class SegmentPolicy { single, per_orbit };
enum class Direction { forward, backward };

struct SegmentPlan {  // propagator.hpp:28-34
    std::vector<double> boundaries;
    Index n_nodes = 200;
    Direction direction = Direction::forward;
    Index segments() const { return static_cast<Index>(boundaries.size()) - 1; }
};

struct PropagationConfig {  // propagator.hpp:38-49
    Index n_nodes = 200;
    double tolerance = 1e-12;
    ErrorMode error_mode = ErrorMode::relative;
    int max_iterations = 100;
    StartMode start_mode = StartMode::warm;
    SegmentPolicy segment_policy = SegmentPolicy::single;
    double max_segment_periods = 1.0;
    ForceModelConfig force;
    Index p_groups = 1;
    double timeout_s = 0.0;
};

/// Host worker split of the reference (propagator.hpp:54-57).  The device path
/// ignores it (all groups run concurrently on the GPU); kept for source compatibility.
struct ExecutionPolicy {
    unsigned group_workers = 1;
    unsigned inner_workers = 1;
};

struct IterationReport {  // picard.hpp:17-22
    int iterations = 0;
    double final_error = std::numeric_limits<double>::infinity();
    bool converged = false;
    std::vector<double> per_iteration_errors;
};

struct WarmStartResult {  // propagator.hpp:59-62
    std::vector<Mat> guesses;
    std::vector<char> cold_fallback;
};

inline std::vector<Mat> cold_start(std::span<const StateVector> states, Index n_nodes) {  // propagator.hpp:65-77
    std::vector<Mat> out;
    out.reserve(states.size());
    for (const auto& s : states) {
        Mat g(n_nodes, state_dim);
        for (Index j = 0; j < n_nodes; ++j) {
            g(j, 0) = s.r.x(); g(j, 1) = s.r.y(); g(j, 2) = s.r.z();
            g(j, 3) = s.v.x(); g(j, 4) = s.v.y(); g(j, 5) = s.v.z();
        }
        out.push_back(std::move(g));
    }
    return out;
}

namespace detail {
inline std::vector<double> pack_states(std::span<const StateVector> states) {
    std::vector<double> v(states.size() * 7);
    for (std::size_t i = 0; i < states.size(); ++i) {
        const auto& s = states[i];
        double* o = v.data() + 7 * i;
        o[0] = s.epoch;
        o[1] = s.r.x(); o[2] = s.r.y(); o[3] = s.r.z();
        o[4] = s.v.x(); o[5] = s.v.y(); o[6] = s.v.z();
    }
    return v;
}
inline StateVector unpack_state(const double* o) {
    StateVector s;
    s.epoch = o[0];
    s.r = Vec3(o[1], o[2], o[3]);
    s.v = Vec3(o[4], o[5], o[6]);
    return s;
}
}  // namespace detail

/// Conic warm start per (node, trajectory) on the device (propagator.hpp:81-103).
inline WarmStartResult warm_start(std::span<const StateVector> states, const ChebyshevGrid& grid, double central_mu) {
    const Index m = static_cast<Index>(states.size()), n = grid.n_nodes;
    const auto packed = detail::pack_states(states);
    std::vector<double> g(static_cast<std::size_t>(m * n * 6));
    std::vector<uint8_t> fb(static_cast<std::size_t>(m));
    if (m > 0)
        check_call([&](pswarm_error* e) {
            return pswarm_warm_start(default_context(), m, packed.data(), n, grid.times.data(), central_mu, g.data(),
                                     fb.data(), e);
        });
    WarmStartResult out;
    out.cold_fallback.assign(fb.begin(), fb.end());
    for (Index i = 0; i < m; ++i) {
        Mat x(n, state_dim);
        std::copy(g.begin() + i * n * 6, g.begin() + (i + 1) * n * 6, x.data());
        out.guesses.push_back(std::move(x));
    }
    return out;
}

/// Single / per-orbit segmentation of [t_start, t_end] (propagator.hpp:109-148).
inline SegmentPlan plan_segments(const StateVector& representative, double t_start, double t_end, double central_mu,
                                 SegmentPolicy policy, Index n_nodes, double max_periods = 1.0) {
    if (t_start == t_end) throw InvalidSpanError("plan_segments: degenerate span at t = " + std::to_string(t_start));
    SegmentPlan plan;
    plan.n_nodes = n_nodes;
    plan.direction = t_end > t_start ? Direction::forward : Direction::backward;
    const double span = t_end - t_start;
    if (policy == SegmentPolicy::single) {
        std::optional<double> period;
        try {
            period = osculating_period(representative, central_mu);
        } catch (const NonEllipticError&) {
        }
        if (period && std::abs(span) > max_periods * (*period) * (1.0 + 1e-12))
            throw InvalidSpanError("plan_segments: span of " + std::to_string(std::abs(span)) + " s exceeds " +
                                   std::to_string(max_periods) + " nominal periods; use the per-orbit policy");
        plan.boundaries = {t_start, t_end};
        return plan;
    }
    const double period = osculating_period(representative, central_mu);
    const double step = std::copysign(max_periods * period, span);
    plan.boundaries.push_back(t_start);
    double at = t_start;
    while ((t_end - at - step) * (span > 0 ? 1.0 : -1.0) > 1e-9 * period) {
        at += step;
        plan.boundaries.push_back(at);
    }
    plan.boundaries.push_back(t_end);
    return plan;
}

struct PropagationResult {  // propagator.hpp:151-169
    Vec times;
    std::vector<Mat> trajectories;
    std::vector<StateVector> terminal_states;
    std::vector<std::vector<IterationReport>> reports;  // [segment][group]
    GroupingPlan plan;
    SegmentPlan segments;
    std::vector<std::string> warnings;
    int max_iterations_used() const {
        int worst = 0;
        for (const auto& seg : reports)
            for (const auto& r : seg) worst = std::max(worst, r.iterations);
        return worst;
    }
};

class PropagationIncompleteError : public Error {  // propagator.hpp:173-186
public:
    PropagationIncompleteError(const std::string& what, Index segment, Index group,
                               std::shared_ptr<const PropagationResult> partial)
        : Error(what), segment_(segment), group_(group), partial_(std::move(partial)) {}
    Index segment() const noexcept { return segment_; }
    Index group() const noexcept { return group_; }
    const std::shared_ptr<const PropagationResult>& partial() const noexcept { return partial_; }

private:
    Index segment_;
    Index group_;
    std::shared_ptr<const PropagationResult> partial_;
};

namespace detail {

/// Plain-C view of a PropagationConfig (bodies flattened for the C-ABI).
struct ConfigMarshal {
    pswarm_config cfg{};
    std::vector<pswarm_body> bodies;
    std::vector<std::vector<double>> bounds, coeffs;

    explicit ConfigMarshal(const PropagationConfig& c) {
        for (const auto& b : c.force.bodies) {
            pswarm_body pb{};
            pb.name = b.name.c_str();
            pb.mu = b.mu;
            if (const auto* el = std::get_if<OrbitalElements>(&b.ephemeris)) {
                pb.kind = 0;
                const double e[7] = {el->a, el->e, el->i, el->raan, el->argp, el->m0, el->epoch};
                for (int k = 0; k < 7; ++k) pb.elements[k] = e[k];
            } else {
                const auto& eph = std::get<ChebyshevEphemeris>(b.ephemeris);
                pb.kind = 1;
                pb.n_segments = static_cast<int32_t>(eph.segments.size());
                Index nc = 0;
                for (const auto& s : eph.segments) nc = std::max(nc, s.coeffs_x.size());
                pb.n_coeffs = static_cast<int32_t>(nc);
                std::vector<double> bd, cf;
                for (const auto& s : eph.segments) {
                    bd.push_back(s.t_start);
                    bd.push_back(s.t_end);
                    for (const Vec* v : {&s.coeffs_x, &s.coeffs_y, &s.coeffs_z})
                        for (Index k = 0; k < nc; ++k) cf.push_back(k < v->size() ? (*v)[k] : 0.0);
                }
                bounds.push_back(std::move(bd));
                coeffs.push_back(std::move(cf));
                pb.seg_bounds = bounds.back().data();
                pb.coeffs = coeffs.back().data();
            }
            bodies.push_back(pb);
        }
        cfg.n_nodes = c.n_nodes;
        cfg.tolerance = c.tolerance;
        cfg.error_mode = c.error_mode == ErrorMode::absolute ? 1 : 0;
        cfg.max_iterations = c.max_iterations;
        cfg.start_mode = c.start_mode == StartMode::cold ? 1 : c.start_mode == StartMode::hot ? 2 : 0;
        cfg.segment_policy = c.segment_policy == SegmentPolicy::per_orbit ? 1 : 0;
        cfg.max_segment_periods = c.max_segment_periods;
        cfg.force_kind = c.force.kind == ForceKind::n_body ? 1 : c.force.kind == ForceKind::n_body_1pn ? 2 : 0;
        cfg.n_bodies = static_cast<int32_t>(bodies.size());
        cfg.central_mu = c.force.central_mu;
        cfg.bodies = bodies.empty() ? nullptr : bodies.data();
        cfg.proximity_floor_km = c.force.proximity_floor_km;
        cfg.p_groups = c.p_groups;
        cfg.timeout_s = c.timeout_s;
        cfg.c_light = c.force.c_light;
    }
    ConfigMarshal(const ConfigMarshal&) = delete;
};

/// Host buffers of one device call and their conversion into a PropagationResult.
/// Persistent host helper threads for the result assembly (created on first use, kept for
/// the process): a call with W workers costs no thread creation, and each helper keeps its
/// malloc arena warm across calls.  run(n, fn) executes fn(0..n-1), the caller taking 0.
class HostPool {
public:
    static HostPool& instance() {
        static HostPool pool;
        return pool;
    }
    void run(unsigned n, const std::function<void(unsigned)>& fn) {
        if (n <= 1) {
            if (n == 1) fn(0);
            return;
        }
        std::lock_guard call(call_mu_);  // one assembly at a time
        {
            std::unique_lock lk(mu_);
            while (threads_.size() < n - 1) {
                const unsigned id = static_cast<unsigned>(threads_.size()) + 1;
                threads_.emplace_back([this, id] { loop(id); });
            }
            job_ = &fn;
            active_ = n;
            pending_ = n - 1;
            ++generation_;
        }
        cv_start_.notify_all();
        fn(0);
        std::unique_lock lk(mu_);
        cv_done_.wait(lk, [&] { return pending_ == 0; });
        job_ = nullptr;
    }
    ~HostPool() {
        {
            std::lock_guard lk(mu_);
            stop_ = true;
        }
        cv_start_.notify_all();
        for (auto& t : threads_) t.join();
    }

private:
    void loop(unsigned id) {
        std::uint64_t seen = 0;
        for (;;) {
            const std::function<void(unsigned)>* job;
            {
                std::unique_lock lk(mu_);
                cv_start_.wait(lk, [&] { return stop_ || generation_ != seen; });
                if (stop_) return;
                seen = generation_;
                if (id >= active_) continue;
                job = job_;
            }
            (*job)(id);
            std::lock_guard lk(mu_);
            if (--pending_ == 0) cv_done_.notify_all();
        }
    }
    std::mutex call_mu_, mu_;
    std::condition_variable cv_start_, cv_done_;
    std::vector<std::thread> threads_;
    const std::function<void(unsigned)>* job_ = nullptr;
    unsigned active_ = 0, pending_ = 0;
    std::uint64_t generation_ = 0;
    bool stop_ = false;
};

/// Per-thread, grow-only page-locked staging for the large per-call outputs (node samples,
/// error histories, terminal states): the device writes them at DMA speed and no call pays
/// fresh-page faults for megabytes of result buffers.  to_result copies out of it, so it is
/// free again when a propagate / run_batch call returns.
struct PinnedScratch {
    void* p = nullptr;
    std::size_t cap = 0;
    template <typename T>
    T* get(std::size_t count) {
        const std::size_t bytes = std::max<std::size_t>(count * sizeof(T), 64);
        if (bytes > cap) {
            pswarm_pinned_free(p);
            p = pswarm_pinned_alloc(bytes);
            cap = p ? bytes : 0;
            if (!p) throw Error("pswarm_pinned_alloc: cannot allocate " + std::to_string(bytes) + " bytes");
        }
        return static_cast<T*>(p);
    }
    PinnedScratch() = default;
    PinnedScratch(const PinnedScratch&) = delete;
    PinnedScratch& operator=(const PinnedScratch&) = delete;
    ~PinnedScratch() { pswarm_pinned_free(p); }
};
inline PinnedScratch& scratch(int which) {
    thread_local PinnedScratch s[3];
    return s[which];
}

struct OutputBuffers {
    Index M, P, S, R, max_it;
    double *terminal, *samples, *history;  // pinned scratch (see PinnedScratch)
    std::vector<double> times, final_err;
    std::vector<int32_t> iters;
    std::vector<uint8_t> conv, fallback;
    pswarm_outputs out{};

    OutputBuffers(Index m, Index p, Index s, Index n, int max_iterations)
        : M(m), P(p), S(s), R(1 + s * (n - 1)), max_it(std::max(max_iterations, 0)) {
        terminal = scratch(0).get<double>(static_cast<std::size_t>(M * 7));
        samples = scratch(1).get<double>(static_cast<std::size_t>(M * R * 6));
        history = scratch(2).get<double>(static_cast<std::size_t>(S * P * std::max<Index>(max_it, 1)));
        times.assign(static_cast<std::size_t>(R), 0.0);
        iters.assign(static_cast<std::size_t>(S * P), 0);
        final_err.assign(static_cast<std::size_t>(S * P), 0.0);
        conv.assign(static_cast<std::size_t>(S * P), 0);
        fallback.assign(static_cast<std::size_t>(S * M), 0);
        out.terminal_states = terminal;
        out.samples = samples;
        out.times = times.data();
        out.iterations = iters.data();
        out.final_error = final_err.data();
        out.converged = conv.data();
        out.error_history = history;
        out.cold_fallback = fallback.data();
    }

    /// `workers` host threads assemble the per-trajectory sample matrices (the reference's
    /// worker count is a host thread count; on the device path the host work left is this
    /// copy of M x R x 6 doubles out of the pinned staging).
    PropagationResult to_result(const GroupingPlan& plan, const SegmentPlan& sp, bool complete,
                                bool independent_warnings, unsigned workers = 1) const {
        PropagationResult r;
        r.plan = plan;
        r.segments = sp;
        r.times.resize(R);
        for (Index j = 0; j < R; ++j) r.times[j] = times[j];
        r.trajectories.reserve(static_cast<std::size_t>(M));
        // rows of completed segments only: a failed segment's rows stay zero, as the
        // reference appends a segment's samples after it converged (propagator.hpp:314-330)
        const Index done = out.segments_completed;
        const Index rows = complete ? R : (done > 0 && S > 0 ? 1 + done * ((R - 1) / S) : 0);
        r.trajectories.resize(static_cast<std::size_t>(M));
        auto fill = [&](Index lo, Index hi) {
            for (Index i = lo; i < hi; ++i) {
                Mat t(R, state_dim);
                std::copy(samples + i * R * 6, samples + (i * R + rows) * 6, t.data());
                r.trajectories[static_cast<std::size_t>(i)] = std::move(t);
            }
        };
        const Index W = std::clamp<Index>(static_cast<Index>(workers), 1, std::max<Index>(M, 1));
        if (W == 1 || M * R * 6 < (Index{1} << 16)) {
            fill(0, M);
        } else {  // contiguous chunks, as the reference pool's parallel_chunks (thread_pool.hpp:44-62)
            HostPool::instance().run(static_cast<unsigned>(W),
                                     [&](unsigned w) { fill(M * w / W, M * (w + 1) / W); });
        }
        if (complete)
            for (Index i = 0; i < M; ++i) r.terminal_states.push_back(unpack_state(terminal + 7 * i));
        for (Index s = 0; s < out.segments_reported; ++s) {
            std::vector<IterationReport> seg(static_cast<std::size_t>(P));
            for (Index g = 0; g < P; ++g) {
                const Index k = s * P + g;
                auto& q = seg[static_cast<std::size_t>(g)];
                q.iterations = iters[k];
                q.final_error = final_err[k];
                q.converged = conv[k] != 0;
                for (Index it = 0; it < std::min<Index>(q.iterations, max_it); ++it)
                    q.per_iteration_errors.push_back(history[k * max_it + it]);
            }
            r.reports.push_back(std::move(seg));
        }
        for (Index s = 0; s < out.segments_reported; ++s)
            for (Index i = 0; i < M; ++i)
                if (fallback[s * M + i]) {
                    std::string w = "segment " + std::to_string(s) + ", trajectory " +
                                    std::to_string(independent_warnings ? 0 : i) + ": non-elliptic state, cold start used";
                    if (independent_warnings) w = "trajectory " + std::to_string(i) + ": " + w;
                    r.warnings.push_back(std::move(w));
                }
        return r;
    }
};

}  // namespace detail

/// propagate (propagator.hpp:192-347) on the device.
inline PropagationResult propagate(std::span<const StateVector> states, const GroupingPlan& plan,
                                   const SegmentPlan& segment_plan, const PropagationConfig& config,
                                   const ExecutionPolicy& exec = {}) {
    // the pool size of the reference (propagator.hpp:228-236) sizes the host-side assembly
    const unsigned workers = std::max({exec.group_workers, exec.inner_workers, 1u});
    detail::ConfigMarshal cm(config);
    const auto packed = detail::pack_states(states);
    const Index S = std::max<Index>(segment_plan.segments(), 0);
    detail::OutputBuffers ob(static_cast<Index>(states.size()), plan.groups(), S, segment_plan.n_nodes,
                             config.max_iterations);
    pswarm_error e{};
    const pswarm_status st =
        pswarm_propagate(default_context(), static_cast<int64_t>(states.size()), packed.data(), plan.groups(),
                         plan.group_sizes.data(), static_cast<int64_t>(segment_plan.boundaries.size()),
                         segment_plan.boundaries.data(), segment_plan.n_nodes, &cm.cfg, &ob.out, &e);
    if (st == PSWARM_ERR_INCOMPLETE) {
        auto partial = std::make_shared<PropagationResult>(ob.to_result(plan, segment_plan, false, false, workers));
        throw PropagationIncompleteError(e.message, e.segment, e.group, std::move(partial));
    }
    if (st != PSWARM_OK) throw_from_status(e);
    return ob.to_result(plan, segment_plan, true, false, workers);
}

}  // namespace pswarm
