// ============================================================================
// pswarm_ref — CPU ORACLE for the augmented Picard–Chebyshev hot path.
//
// TEST INFRASTRUCTURE ONLY.  This header is an Eigen-free C++ restatement of
// the reference library `pswarm` (/root/reference/proj/include/pswarm, a
// header-only C++20 library that needs Eigen, which is absent from this image,
// so the reference itself cannot be compiled here — see DESIGN.md §Oracle).
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
// `--impl reference` leg may link or execute it, and only as the checker or
// the CPU baseline.  The product (paper_2301_03989_b200/, include/) never
// includes or links anything under oracle/.
//
// Parity pinning: the reference ships no golden vectors; this restatement is
// pinned by re-running every known-answer test and property the reference's
// own suites hold (proj/tests/*.cpp, proj/tests/acceptance.cpp) — see
// oracle/kat_tests.cpp — and by its independent RKF7(8) integrator.
//
// Arithmetic follows the reference operation order where practical and is
// compiled with -O3 -ffp-contract=off and no -march (the reference builds
// plain CMake Release on x86-64, proj/CMakeLists.txt:8-10, i.e. no FMA).
// Each function cites the reference file:line it restates.
// ============================================================================
#pragma once

#include <algorithm>
#include <array>
#include <atomic>
#include <bit>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <cstdint>
#include <exception>
#include <functional>
#include <limits>
#include <memory>
#include <mutex>
#include <numbers>
#include <optional>
#include <stdexcept>
#include <string>
#include <thread>
#include <unordered_map>
#include <utility>
#include <vector>

namespace pswarm_ref {

using Index = std::int64_t;
inline constexpr Index state_dim = 6;  // types.hpp:18

// ---------------------------------------------------------------------------
// Minimal dense containers (stand-ins for the Eigen aliases of types.hpp:11-15)
// ---------------------------------------------------------------------------
struct V3 {
    double x = 0.0, y = 0.0, z = 0.0;
    double operator[](int i) const { return i == 0 ? x : (i == 1 ? y : z); }
    double& operator[](int i) { return i == 0 ? x : (i == 1 ? y : z); }
    double sq() const { return x * x + y * y + z * z; }
    double norm() const { return std::sqrt(sq()); }  // Eigen: sqrt(squaredNorm())
};
inline V3 operator+(V3 a, V3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
inline V3 operator-(V3 a, V3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
inline V3 operator*(double s, V3 a) { return {s * a.x, s * a.y, s * a.z}; }
inline V3 operator/(V3 a, double s) { return {a.x / s, a.y / s, a.z / s}; }
inline double dot(V3 a, V3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
inline V3 cross(V3 a, V3 b) {
    return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}

/// Row-major dense matrix (types.hpp:11).
struct Mat {
    Index r = 0, c = 0;
    std::vector<double> v;
    Mat() = default;
    Mat(Index rows, Index cols, double fill = 0.0)
        : r(rows), c(cols), v(static_cast<std::size_t>(rows * cols), fill) {}
    double& operator()(Index i, Index j) { return v[static_cast<std::size_t>(i * c + j)]; }
    double operator()(Index i, Index j) const { return v[static_cast<std::size_t>(i * c + j)]; }
    double* row(Index i) { return v.data() + i * c; }
    const double* row(Index i) const { return v.data() + i * c; }
    Index rows() const { return r; }
    Index cols() const { return c; }
    void resize(Index rows, Index cols) {
        r = rows;
        c = cols;
        v.assign(static_cast<std::size_t>(rows * cols), 0.0);
    }
    bool all_finite() const {
        for (double x : v) {
            if (!std::isfinite(x)) return false;
        }
        return true;
    }
};

inline Mat matmul(const Mat& a, const Mat& b) {
    Mat out(a.r, b.c);
    for (Index i = 0; i < a.r; ++i) {
        double* o = out.row(i);
        for (Index k = 0; k < a.c; ++k) {
            const double aik = a(i, k);
            const double* bk = b.row(k);
            for (Index j = 0; j < b.c; ++j) o[j] += aik * bk[j];
        }
    }
    return out;
}

// ---------------------------------------------------------------------------
// Errors (errors.hpp:10-113)
// ---------------------------------------------------------------------------
struct Error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct InvalidSpanError : Error { using Error::Error; };
struct InvalidSizeError : Error { using Error::Error; };
struct ShapeError : Error { using Error::Error; };
struct AlignmentError : Error { using Error::Error; };
struct DivergenceError : Error {
    DivergenceError(const std::string& w, Index n, Index col) : Error(w), node(n), column(col) {}
    Index node, column;
};
struct SingularityError : Error {
    explicit SingularityError(const std::string& w, std::string b = {}) : Error(w), body(std::move(b)) {}
    std::string body;
};
struct CoverageError : Error {
    CoverageError(const std::string& w, double e) : Error(w), epoch(e) {}
    double epoch;
};
struct NonEllipticError : Error { using Error::Error; };
struct SolverError : Error { using Error::Error; };
struct InvalidPlanError : Error { using Error::Error; };
struct EmptyReductionError : Error { using Error::Error; };
struct OracleError : Error { using Error::Error; };
struct TimeoutError : Error { using Error::Error; };

// ---------------------------------------------------------------------------
// Worker pool (thread_pool.hpp:13-154): caller participates, static chunks
// for intra-block work, dynamic task queue for group solves.
// ---------------------------------------------------------------------------
class Pool {
public:
    explicit Pool(unsigned workers) : n_(workers == 0 ? 1 : workers) {
        for (unsigned i = 0; i + 1 < n_; ++i) threads_.emplace_back([this, i] { loop(i); });
    }
    Pool(const Pool&) = delete;
    ~Pool() {
        {
            std::lock_guard g(mu_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto& t : threads_) t.join();
    }
    unsigned size() const { return n_; }

    void chunks(Index total, const std::function<void(Index, Index)>& fn) {  // :46-63
        if (total <= 0) return;
        if (n_ == 1 || total == 1) {
            fn(0, total);
            return;
        }
        const Index w = n_;
        run([&](unsigned k) {
            const Index b = total * k / w, e = total * (k + 1) / w;
            if (b < e) fn(b, e);
        });
    }
    void tasks(Index n_tasks, const std::function<void(Index)>& fn) {  // :67-87
        if (n_tasks <= 0) return;
        if (n_ == 1) {
            for (Index i = 0; i < n_tasks; ++i) fn(i);
            return;
        }
        std::atomic<Index> next{0};
        run([&](unsigned) {
            for (;;) {
                const Index i = next.fetch_add(1);
                if (i >= n_tasks) return;
                fn(i);
            }
        });
    }

private:
    void loop(unsigned idx) {
        std::uint64_t seen = 0;
        for (;;) {
            const std::function<void(unsigned)>* job;
            {
                std::unique_lock l(mu_);
                cv_.wait(l, [&] { return stop_ || gen_ != seen; });
                if (stop_) return;
                seen = gen_;
                job = job_;
            }
            call(*job, idx);
            std::lock_guard g(mu_);
            if (--pending_ == 0) done_.notify_all();
        }
    }
    void call(const std::function<void(unsigned)>& job, unsigned idx) {
        try {
            job(idx);
        } catch (...) {
            std::lock_guard g(mu_);
            if (!err_) err_ = std::current_exception();
        }
    }
    void run(const std::function<void(unsigned)>& job) {
        {
            std::lock_guard g(mu_);
            job_ = &job;
            pending_ = static_cast<unsigned>(threads_.size());
            err_ = nullptr;
            ++gen_;
        }
        cv_.notify_all();
        call(job, n_ - 1);
        std::unique_lock l(mu_);
        done_.wait(l, [&] { return pending_ == 0; });
        if (err_) {
            auto e = err_;
            err_ = nullptr;
            l.unlock();
            std::rethrow_exception(e);
        }
    }
    unsigned n_;
    std::vector<std::thread> threads_;
    std::mutex mu_;
    std::condition_variable cv_, done_;
    const std::function<void(unsigned)>* job_ = nullptr;
    std::uint64_t gen_ = 0;
    unsigned pending_ = 0;
    bool stop_ = false;
    std::exception_ptr err_;
};

// ---------------------------------------------------------------------------
// State (state.hpp:11-29) and error metric (error_metric.hpp:12-23)
// ---------------------------------------------------------------------------
struct State {
    double epoch = 0.0;
    V3 r, v;
};
inline double specific_energy(const State& s, double mu) { return 0.5 * s.v.sq() - mu / s.r.norm(); }
inline V3 angular_momentum(const State& s) { return cross(s.r, s.v); }

enum class ErrorMode { relative, absolute };
inline constexpr double error_norm_floor = 1e-30;
inline double component_error(double delta, double norm, ErrorMode mode) {
    if (mode == ErrorMode::absolute) return delta;
    return delta / std::max(norm, error_norm_floor);
}

// ---------------------------------------------------------------------------
// Chebyshev grid (chebyshev.hpp:16-84)
// ---------------------------------------------------------------------------
inline std::vector<double> lobatto_nodes(Index n) {  // :26-45
    if (n < 3) throw InvalidSizeError("chebyshev_lobatto_nodes: need at least 3 nodes, got " + std::to_string(n));
    const Index m = n - 1;
    std::vector<double> tau(static_cast<std::size_t>(n));
    for (Index j = 0; 2 * j < m; ++j) {
        const double c = std::cos(static_cast<double>(j) * std::numbers::pi / static_cast<double>(m));
        tau[j] = -c;
        tau[m - j] = c;
    }
    if (m % 2 == 0) tau[m / 2] = 0.0;
    tau[0] = -1.0;
    tau[m] = 1.0;
    return tau;
}

inline void cheb_values(double x, double* t, Index count) {  // :48-59
    if (count <= 0) return;
    t[0] = 1.0;
    if (count > 1) t[1] = x;
    for (Index k = 2; k < count; ++k) t[k] = 2.0 * x * t[k - 1] - t[k - 2];
}

struct Grid {
    Index n = 0;
    std::vector<double> tau, times;
    double omega1 = 0.0, omega2 = 0.0;
};

inline Grid build_grid(Index n, double t0, double t1) {  // :61-84
    if (n < 3) throw InvalidSizeError("build_grid: need at least 3 nodes, got " + std::to_string(n));
    if (t0 == t1) throw InvalidSpanError("build_grid: degenerate span at t = " + std::to_string(t0));
    Grid g;
    g.n = n;
    g.tau = lobatto_nodes(n);
    g.omega1 = 0.5 * (t1 + t0);
    g.omega2 = 0.5 * (t1 - t0);
    g.times.resize(static_cast<std::size_t>(n));
    for (Index j = 0; j < n; ++j) g.times[j] = g.omega2 * g.tau[j] + g.omega1;
    g.times[0] = t0;
    g.times[n - 1] = t1;
    return g;
}

// ---------------------------------------------------------------------------
// PC operators (pc_matrices.hpp:33-116) and the linear update (:123-151)
// ---------------------------------------------------------------------------
struct Ops {
    Index n = 0;
    Mat eval, xform, integ, a_op, update_op;
    std::vector<double> s_row, anchor_op;
};

inline Ops build_ops(Index n) {  // :44-103
    if (n < 3) throw InvalidSizeError("build_matrices: need at least 3 nodes, got " + std::to_string(n));
    const Index m = n - 1;
    const auto tau = lobatto_nodes(n);
    Mat tval(n, n);
    for (Index j = 0; j < n; ++j) cheb_values(tau[j], tval.row(j), n);
    Ops o;
    o.n = n;
    o.eval = tval;
    for (Index j = 0; j < n; ++j) o.eval(j, 0) *= 0.5;
    o.xform.resize(n, n);
    for (Index k = 0; k < n; ++k) {
        const double nu = (k == 0 || k == m) ? 2.0 : 1.0;
        for (Index j = 0; j < n; ++j) {
            const double half = (j == 0 || j == m) ? 0.5 : 1.0;
            o.xform(k, j) = 2.0 / (static_cast<double>(m) * nu) * half * tval(j, k);
        }
    }
    o.integ.resize(n, n);
    o.integ(1, 0) = 1.0;
    if (n > 2) o.integ(1, 2) = -0.5;
    for (Index k = 2; k <= m; ++k) {
        const double inv2k = 1.0 / (2.0 * static_cast<double>(k));
        o.integ(k, k - 1) = inv2k;
        if (k + 1 <= m) o.integ(k, k + 1) = -inv2k;
    }
    o.a_op = matmul(o.integ, o.xform);
    o.s_row.resize(static_cast<std::size_t>(m));
    for (Index k = 1; k <= m; ++k) o.s_row[k - 1] = (k % 2 == 0) ? -2.0 : 2.0;
    o.update_op = matmul(o.eval, o.a_op);
    o.anchor_op.assign(static_cast<std::size_t>(n), 0.0);
    for (Index i = 0; i < n; ++i) {
        double acc = 0.0;
        for (Index k = 1; k < n; ++k) acc += o.s_row[k - 1] * o.a_op(k, i);
        o.anchor_op[i] = acc;
    }
    return o;
}

inline std::shared_ptr<const Ops> cached_ops(Index n) {  // :106-116
    static std::mutex mu;
    static std::unordered_map<Index, std::shared_ptr<const Ops>> cache;
    std::lock_guard g(mu);
    auto it = cache.find(n);
    if (it == cache.end()) it = cache.emplace(n, std::make_shared<const Ops>(build_ops(n))).first;
    return it->second;
}

/// Y = update_op*F + 1/2*(anchor_op*F + 2*y0) broadcast over rows (:123-151).
/// Row bands over the pool do not change any value (each output element is
/// the same dot product either way).
inline void picard_update_into(const Ops& o, const Mat& f, const std::vector<double>& y0, Mat& out,
                               Pool* pool = nullptr) {
    const Index n = o.n;
    if (f.r != n)
        throw ShapeError("picard_update: force block has " + std::to_string(f.r) + " rows, expected " +
                         std::to_string(n));
    if (static_cast<Index>(y0.size()) != f.c)
        throw ShapeError("picard_update: initial row has " + std::to_string(y0.size()) +
                         " columns, force block has " + std::to_string(f.c));
    const Index cols = f.c;
    out.resize(n, cols);
    std::vector<double> b0(static_cast<std::size_t>(cols), 0.0);
    for (Index k = 0; k < n; ++k) {
        const double a = o.anchor_op[k];
        const double* fk = f.row(k);
        for (Index c = 0; c < cols; ++c) b0[c] += a * fk[c];
    }
    for (Index c = 0; c < cols; ++c) b0[c] = 0.5 * (b0[c] + 2.0 * y0[c]);
    auto band = [&](Index r0, Index r1) {
        for (Index j = r0; j < r1; ++j) {
            double* oj = out.row(j);
            for (Index k = 0; k < n; ++k) {
                const double u = o.update_op(j, k);
                const double* fk = f.row(k);
                for (Index c = 0; c < cols; ++c) oj[c] += u * fk[c];
            }
            for (Index c = 0; c < cols; ++c) oj[c] += b0[c];
        }
    };
    if (pool && pool->size() > 1 && n >= 2 * static_cast<Index>(pool->size()))
        pool->chunks(n, band);
    else
        band(0, n);
}

// ---------------------------------------------------------------------------
// Conics (kepler.hpp:14-131)
// ---------------------------------------------------------------------------
struct Elements {
    double a = 0, e = 0, i = 0, raan = 0, argp = 0, m0 = 0, epoch = 0;
};

inline double solve_kepler(double mean_anomaly, double ecc) {  // :26-42
    constexpr double two_pi = 2.0 * std::numbers::pi;
    const double mw = std::remainder(mean_anomaly, two_pi);
    double e = (ecc < 0.8) ? mw : std::copysign(std::numbers::pi, mw);
    for (int it = 0; it < 50; ++it) {
        const double f = e - ecc * std::sin(e) - mw;
        const double fp = 1.0 - ecc * std::cos(e);
        const double step = f / fp;
        e -= step;
        if (std::abs(step) <= 1e-14) return e + (mean_anomaly - mw);
    }
    throw SolverError("solve_kepler: Newton iteration did not converge for M = " + std::to_string(mean_anomaly) +
                      ", e = " + std::to_string(ecc));
}

inline double osculating_period(const State& s, double mu) {  // :45-53
    const double energy = specific_energy(s, mu);
    if (!(energy < 0.0))
        throw NonEllipticError("osculating_period: state is not bound (specific energy " + std::to_string(energy) +
                               " km^2/s^2)");
    const double a = -mu / (2.0 * energy);
    return 2.0 * std::numbers::pi * std::sqrt(a * a * a / mu);
}

inline State kepler_propagate(const State& s, double mu, double dt) {  // :59-98
    const double r0n = s.r.norm();
    if (!(r0n > 0.0)) throw SingularityError("kepler_propagate: zero-radius state");
    const double energy = 0.5 * s.v.sq() - mu / r0n;
    if (!(energy < 0.0))
        throw NonEllipticError("kepler_propagate: specific energy " + std::to_string(energy) +
                               " km^2/s^2 is not negative");
    if (dt == 0.0) return s;
    const double a = -mu / (2.0 * energy);
    const double n = std::sqrt(mu / (a * a * a));
    const double esin = dot(s.r, s.v) / std::sqrt(mu * a);
    const double ecos = 1.0 - r0n / a;
    const double ecc = std::hypot(esin, ecos);
    if (ecc >= 1.0 - 1e-8)
        throw NonEllipticError("kepler_propagate: eccentricity " + std::to_string(ecc) + " too close to parabolic");
    const double e0 = std::atan2(esin, ecos);
    const double m0 = e0 - esin;
    const double e1 = solve_kepler(m0 + n * dt, ecc);
    const double de = e1 - e0;
    const double cde = std::cos(de), sde = std::sin(de);
    const double f = 1.0 - (a / r0n) * (1.0 - cde);
    const double g = dt + (sde - de) / n;
    State out;
    out.epoch = s.epoch + dt;
    out.r = f * s.r + g * s.v;
    const double r1n = a * (1.0 - ecc * std::cos(e1));
    const double fdot = -std::sqrt(mu * a) * sde / (r1n * r0n);
    const double gdot = 1.0 - (a / r1n) * (1.0 - cde);
    out.v = fdot * s.r + gdot * s.v;
    return out;
}

inline State elements_to_state(const Elements& el, double mu, double t) {  // :102-131
    if (!(el.a > 0.0) || el.e < 0.0 || el.e >= 1.0 - 1e-8)
        throw NonEllipticError("elements_to_state: elements do not define a bound conic (a = " +
                               std::to_string(el.a) + ", e = " + std::to_string(el.e) + ")");
    const double n = std::sqrt(mu / (el.a * el.a * el.a));
    const double E = solve_kepler(el.m0 + n * (t - el.epoch), el.e);
    const double ce = std::cos(E), se = std::sin(E);
    const double beta = std::sqrt(1.0 - el.e * el.e);
    const double rn = el.a * (1.0 - el.e * ce);
    const double xp = el.a * (ce - el.e), yp = el.a * beta * se;
    const double vs = std::sqrt(mu * el.a) / rn;
    const double vxp = -vs * se, vyp = vs * beta * ce;
    const double co = std::cos(el.raan), so = std::sin(el.raan);
    const double ci = std::cos(el.i), si = std::sin(el.i);
    const double cw = std::cos(el.argp), sw = std::sin(el.argp);
    const V3 p{co * cw - so * sw * ci, so * cw + co * sw * ci, sw * si};
    const V3 q{-co * sw - so * cw * ci, -so * sw + co * cw * ci, cw * si};
    State out;
    out.epoch = t;
    out.r = xp * p + yp * q;
    out.v = vxp * p + vyp * q;
    return out;
}

// ---------------------------------------------------------------------------
// Ephemerides (ephemeris.hpp:17-152)
// ---------------------------------------------------------------------------
struct ChebSeg {
    double t_start = 0, t_end = 0;
    std::vector<double> cx, cy, cz;
    static double clenshaw(const std::vector<double>& c, double x) {  // :29-38
        double b1 = 0.0, b2 = 0.0;
        for (Index k = static_cast<Index>(c.size()) - 1; k >= 1; --k) {
            const double b0 = c[k] + 2.0 * x * b1 - b2;
            b2 = b1;
            b1 = b0;
        }
        return c[0] + x * b1 - b2;
    }
    V3 position_at(double t) const {  // :24-27
        const double tau = (2.0 * t - (t_start + t_end)) / (t_end - t_start);
        return {clenshaw(cx, tau), clenshaw(cy, tau), clenshaw(cz, tau)};
    }
    // EXTENSION (relativistic model, not in the reference): d/dt of the series via the
    // derivative-coefficient recurrence c'_{k-1} = c'_{k+1} + 2k c_k, c'_0 halved.
    static std::vector<double> derivative(const std::vector<double>& c) {
        const Index n = static_cast<Index>(c.size());
        std::vector<double> d(static_cast<std::size_t>(std::max<Index>(n, 1)), 0.0);
        for (Index k = n - 1; k >= 1; --k) d[k - 1] = (k + 1 < n ? d[k + 1] : 0.0) + 2.0 * k * c[k];
        d[0] *= 0.5;
        return d;
    }
    V3 velocity_at(double t) const {
        const double tau = (2.0 * t - (t_start + t_end)) / (t_end - t_start);
        const double s = 2.0 / (t_end - t_start);
        return {s * clenshaw(derivative(cx), tau), s * clenshaw(derivative(cy), tau), s * clenshaw(derivative(cz), tau)};
    }
};

struct Body {
    std::string name;
    double mu = 0.0;
    bool tabulated = false;
    Elements el;
    std::vector<ChebSeg> segs;
};

inline V3 body_position(const Body& b, double central_mu, double t) {  // :58-73
    if (!b.tabulated) return elements_to_state(b.el, central_mu, t).r;
    for (const auto& s : b.segs) {
        const bool fwd = s.t_start <= s.t_end;
        if ((fwd && t >= s.t_start && t <= s.t_end) || (!fwd && t <= s.t_start && t >= s.t_end))
            return s.position_at(t);
    }
    throw CoverageError("ephemeris for body '" + b.name + "' does not cover epoch " + std::to_string(t), t);
}

/// EXTENSION (relativistic model): heliocentric position and velocity of a body.
inline std::pair<V3, V3> body_state(const Body& b, double central_mu, double t) {
    if (!b.tabulated) {
        const State s = elements_to_state(b.el, central_mu, t);
        return {s.r, s.v};
    }
    for (const auto& s : b.segs) {
        const bool fwd = s.t_start <= s.t_end;
        if ((fwd && t >= s.t_start && t <= s.t_end) || (!fwd && t <= s.t_start && t >= s.t_end))
            return {s.position_at(t), s.velocity_at(t)};
    }
    throw CoverageError("ephemeris for body '" + b.name + "' does not cover epoch " + std::to_string(t), t);
}

struct EphTable {  // :77-86
    std::vector<double> node_times;
    double central_mu = 0.0;
    std::vector<std::string> names;
    std::vector<double> mus;
    std::vector<Mat> pos;  // per body N x 3
    Index n_bodies() const { return static_cast<Index>(mus.size()); }
    // EXTENSION (relativistic model): body velocities, Newtonian heliocentric
    // accelerations and the potentials of the other massive bodies at each body, frozen per
    // node like the positions.
    bool rel = false;
    double c_light = 0.0;
    std::vector<Mat> vel, acc;           // per body N x 3
    std::vector<std::vector<double>> phi;  // per body [N]: mu_sun/|r_b| + sum_{k!=b} mu_k/|r_k - r_b|
    std::vector<double> phi_sun;         // [N]: sum_k mu_k/|r_k|
};

/// Massive-body quantities of the EIH test-particle equation at one epoch: positions,
/// velocities, Newtonian heliocentric accelerations and external potentials (EXTENSION).
struct RelBodies {
    std::vector<V3> r, v, a;
    std::vector<double> mu, phi;
    double phi_sun = 0.0;
};

inline void rel_derive(RelBodies& q, double central_mu) {
    const std::size_t B = q.r.size();
    q.a.assign(B, V3{});
    q.phi.assign(B, 0.0);
    q.phi_sun = 0.0;
    for (std::size_t b = 0; b < B; ++b) {
        const double rb = q.r[b].norm();
        q.phi_sun += q.mu[b] / rb;
        V3 a = (-(central_mu + q.mu[b]) / (rb * rb * rb)) * q.r[b];
        double phi = central_mu / rb;
        for (std::size_t k = 0; k < B; ++k) {
            if (k == b) continue;
            const V3 d = q.r[k] - q.r[b];
            const double dn = d.norm(), rk = q.r[k].norm();
            a = a + q.mu[k] * (d / (dn * dn * dn) - q.r[k] / (rk * rk * rk));
            phi += q.mu[k] / dn;
        }
        q.a[b] = a;
        q.phi[b] = phi;
    }
}

/// EXTENSION: first post-Newtonian (EIH, beta = gamma = 1) correction for a massless
/// particle at r, v among the Sun (at the origin, at rest) and the bodies in q
/// (Explanatory Supplement to the Astronomical Almanac 1992, eq. 8.1),
/// textbook two-pass form.  The Newtonian part is added separately (table_acc).
inline V3 eih_correction(V3 r, V3 v, const RelBodies& q, double central_mu, double c_light) {
    const double c2 = c_light * c_light;
    const std::size_t B = q.r.size();
    auto at = [&](std::size_t A, V3& rA, V3& vA, V3& aA, double& muA, double& phiA) {
        if (A == 0) {
            rA = V3{};
            vA = V3{};
            aA = V3{};
            muA = central_mu;
            phiA = q.phi_sun;
        } else {
            rA = q.r[A - 1];
            vA = q.v[A - 1];
            aA = q.a[A - 1];
            muA = q.mu[A - 1];
            phiA = q.phi[A - 1];
        }
    };
    double U = 0.0;  // potential of all massive bodies at the particle
    for (std::size_t A = 0; A <= B; ++A) {
        V3 rA, vA, aA;
        double muA, phiA;
        at(A, rA, vA, aA, muA, phiA);
        U += muA / (r - rA).norm();
    }
    const double v2 = dot(v, v);
    V3 out{};
    for (std::size_t A = 0; A <= B; ++A) {
        V3 rA, vA, aA;
        double muA, phiA;
        at(A, rA, vA, aA, muA, phiA);
        const V3 d = rA - r;  // r_A - r
        const double rho = d.norm();
        const double rho3 = rho * rho * rho;
        const double proj = dot(r - rA, vA) / rho;
        const double bracket = -4.0 * U / c2 - phiA / c2 + v2 / c2 + 2.0 * dot(vA, vA) / c2 -
                               4.0 * dot(v, vA) / c2 - 1.5 * proj * proj / c2 + 0.5 * dot(d, aA) / c2;
        out = out + (muA / rho3 * bracket) * d;
        out = out + (muA / rho3 * dot(r - rA, 4.0 * v - 3.0 * vA) / c2) * (v - vA);
        out = out + (3.5 * muA / rho / c2) * aA;
    }
    return out;
}

/// Massive-body quantities of node j of a table (derived on first use from positions and
/// velocities).
inline RelBodies rel_at_node(const EphTable& t, Index j) {
    RelBodies q;
    for (Index b = 0; b < t.n_bodies(); ++b) {
        q.r.push_back({t.pos[b](j, 0), t.pos[b](j, 1), t.pos[b](j, 2)});
        q.v.push_back({t.vel[b](j, 0), t.vel[b](j, 1), t.vel[b](j, 2)});
        q.mu.push_back(t.mus[b]);
    }
    rel_derive(q, t.central_mu);
    return q;
}

inline EphTable build_ephemeris(const std::vector<Body>& bodies, const Grid& g, double central_mu) {  // :89-107
    EphTable t;
    t.node_times = g.times;
    t.central_mu = central_mu;
    for (const auto& b : bodies) {
        Mat p(g.n, 3);
        for (Index j = 0; j < g.n; ++j) {
            const V3 r = body_position(b, central_mu, g.times[j]);
            p(j, 0) = r.x;
            p(j, 1) = r.y;
            p(j, 2) = r.z;
        }
        t.names.push_back(b.name);
        t.mus.push_back(b.mu);
        t.pos.push_back(std::move(p));
    }
    return t;
}

/// Massive-body quantities of node j read from a finished relativistic table.
inline RelBodies rel_cached(const EphTable& t, Index j) {
    RelBodies q;
    for (Index b = 0; b < t.n_bodies(); ++b) {
        q.r.push_back({t.pos[b](j, 0), t.pos[b](j, 1), t.pos[b](j, 2)});
        q.v.push_back({t.vel[b](j, 0), t.vel[b](j, 1), t.vel[b](j, 2)});
        q.a.push_back({t.acc[b](j, 0), t.acc[b](j, 1), t.acc[b](j, 2)});
        q.mu.push_back(t.mus[b]);
        q.phi.push_back(t.phi[b][j]);
    }
    q.phi_sun = t.phi_sun[j];
    return q;
}

/// EXTENSION: the per-node table of the relativistic model (positions as above, plus
/// velocities, accelerations and potentials).
inline EphTable build_ephemeris_rel(const std::vector<Body>& bodies, const Grid& g, double central_mu,
                                    double c_light) {
    EphTable t = build_ephemeris(bodies, g, central_mu);
    t.rel = true;
    t.c_light = c_light;
    const std::size_t B = bodies.size();
    for (std::size_t b = 0; b < B; ++b) {
        Mat v(g.n, 3);
        for (Index j = 0; j < g.n; ++j) {
            const V3 vb = body_state(bodies[b], central_mu, g.times[j]).second;
            v(j, 0) = vb.x;
            v(j, 1) = vb.y;
            v(j, 2) = vb.z;
        }
        t.vel.push_back(std::move(v));
        t.acc.emplace_back(g.n, 3);
        t.phi.emplace_back(static_cast<std::size_t>(g.n), 0.0);
    }
    t.phi_sun.assign(static_cast<std::size_t>(g.n), 0.0);
    for (Index j = 0; j < g.n; ++j) {
        RelBodies q = rel_at_node(t, j);
        for (std::size_t b = 0; b < B; ++b) {
            t.acc[b](j, 0) = q.a[b].x;
            t.acc[b](j, 1) = q.a[b].y;
            t.acc[b](j, 2) = q.a[b].z;
            t.phi[b][j] = q.phi[b];
        }
        t.phi_sun[j] = q.phi_sun;
    }
    return t;
}

template <typename PosFn>
ChebSeg fit_segment(PosFn&& position, double t0, double t1, Index n) {  // :112-152
    if (n < 3) throw InvalidSizeError("fit_chebyshev_segment: need at least 3 coefficients");
    if (t0 == t1) throw InvalidSpanError("fit_chebyshev_segment: degenerate span");
    const Index m = n - 1;
    const auto tau = lobatto_nodes(n);
    Mat samples(n, 3), tval(n, n);
    for (Index j = 0; j < n; ++j) {
        const double t = 0.5 * (t1 - t0) * tau[j] + 0.5 * (t1 + t0);
        const V3 p = position(t);
        samples(j, 0) = p.x;
        samples(j, 1) = p.y;
        samples(j, 2) = p.z;
        cheb_values(tau[j], tval.row(j), n);
    }
    ChebSeg s;
    s.t_start = t0;
    s.t_end = t1;
    s.cx.resize(n);
    s.cy.resize(n);
    s.cz.resize(n);
    for (Index k = 0; k < n; ++k) {
        const double nu = (k == 0 || k == m) ? 2.0 : 1.0;
        double ax = 0, ay = 0, az = 0;
        for (Index j = 0; j < n; ++j) {
            const double w = ((j == 0 || j == m) ? 0.5 : 1.0) * tval(j, k);
            ax += w * samples(j, 0);
            ay += w * samples(j, 1);
            az += w * samples(j, 2);
        }
        const double sc = 2.0 / (static_cast<double>(m) * nu);
        s.cx[k] = sc * ax;
        s.cy[k] = sc * ay;
        s.cz[k] = sc * az;
    }
    return s;
}

// ---------------------------------------------------------------------------
// Force model (force_model.hpp:14-142)
// ---------------------------------------------------------------------------
/// n_body_1pn = EXTENSION (BASELINE config 5; not in the reference): Newtonian
/// restricted N-body + the EIH first post-Newtonian correction (eih_correction).
enum class ForceKind { two_body, n_body, n_body_1pn };
inline bool has_bodies(ForceKind k) { return k != ForceKind::two_body; }
struct ForceConfig {
    ForceKind kind = ForceKind::two_body;
    double central_mu = 0.0;
    std::vector<Body> bodies;
    double proximity_floor_km = 1.0;
    double c_light = 299792.458;  // km/s (relativistic model only)
};

inline V3 central_acc(V3 r, double mu) {  // :26-32
    const double rn = r.norm();
    if (!(rn > 0.0)) throw SingularityError("central-body acceleration at zero radius");
    return (-mu / (rn * rn * rn)) * r;
}

inline V3 perturber_acc(V3 r, V3 rb, double mu_b, double floor_km, const std::string& name) {  // :40-52
    const V3 d = rb - r;
    const double dn = d.norm();
    if (dn < floor_km)
        throw SingularityError("close approach to body '" + name + "': distance " + std::to_string(dn) +
                                   " km below floor " + std::to_string(floor_km) + " km",
                               name);
    const double bn = rb.norm();
    const V3 direct = d / (dn * dn * dn);
    const V3 indirect = rb / (bn * bn * bn);
    return mu_b * (direct - indirect);
}

inline V3 table_acc(V3 r, Index node, const EphTable& t, ForceKind kind, double floor_km) {  // :57-69
    V3 a = central_acc(r, t.central_mu);
    if (has_bodies(kind)) {
        for (Index b = 0; b < t.n_bodies(); ++b) {
            const V3 rb{t.pos[b](node, 0), t.pos[b](node, 1), t.pos[b](node, 2)};
            a = a + perturber_acc(r, rb, t.mus[b], floor_km, t.names[b]);
        }
    }
    return a;
}

inline V3 acceleration_at(V3 r, double t, const ForceConfig& cfg) {  // :78-87
    V3 a = central_acc(r, cfg.central_mu);
    if (has_bodies(cfg.kind))
        for (const auto& b : cfg.bodies)
            a = a + perturber_acc(r, body_position(b, cfg.central_mu, t), b.mu, cfg.proximity_floor_km, b.name);
    return a;
}

/// EXTENSION: continuous-time acceleration of the relativistic model (RKF78 cross-check).
inline V3 acceleration_at(V3 r, V3 v, double t, const ForceConfig& cfg) {
    V3 a = acceleration_at(r, t, cfg);
    if (cfg.kind == ForceKind::n_body_1pn) {
        RelBodies q;
        for (const auto& b : cfg.bodies) {
            const auto [rb, vb] = body_state(b, cfg.central_mu, t);
            q.r.push_back(rb);
            q.v.push_back(vb);
            q.mu.push_back(b.mu);
        }
        rel_derive(q, cfg.central_mu);
        a = a + eih_correction(r, v, q, cfg.central_mu, cfg.c_light);
    }
    return a;
}

/// omega2-scaled derivative block of a component-major N x 6m state block (:93-142).
inline void eval_force_block(const Mat& y, Index m, const Grid& g, const EphTable& t, const ForceConfig& cfg,
                             Mat& force, Pool* pool = nullptr) {
    const Index n = g.n;
    if (y.r != n || y.c != state_dim * m)
        throw ShapeError("eval_force_block: state block is " + std::to_string(y.r) + "x" + std::to_string(y.c) +
                         ", expected " + std::to_string(n) + "x" + std::to_string(state_dim * m));
    if (static_cast<Index>(t.node_times.size()) != n)
        throw AlignmentError("eval_force_block: ephemeris table has " + std::to_string(t.node_times.size()) +
                             " nodes, grid has " + std::to_string(n));
    force.resize(n, state_dim * m);
    const double w2 = g.omega2;
    auto sample = [&](Index j, Index k) {
        const V3 r{y(j, k), y(j, m + k), y(j, 2 * m + k)};
        const V3 v{y(j, 3 * m + k), y(j, 4 * m + k), y(j, 5 * m + k)};
        V3 a;
        try {
            a = table_acc(r, j, t, cfg.kind, cfg.proximity_floor_km);
            if (t.rel) a = a + eih_correction(r, v, rel_cached(t, j), t.central_mu, t.c_light);
        } catch (const SingularityError& e) {
            throw SingularityError("node " + std::to_string(j) + ", trajectory " + std::to_string(k) + ": " + e.what(),
                                   e.body);
        }
        force(j, k) = w2 * v.x;
        force(j, m + k) = w2 * v.y;
        force(j, 2 * m + k) = w2 * v.z;
        force(j, 3 * m + k) = w2 * a.x;
        force(j, 4 * m + k) = w2 * a.y;
        force(j, 5 * m + k) = w2 * a.z;
    };
    const Index samples = n * m;
    if (pool && pool->size() > 1)
        pool->chunks(samples, [&](Index b, Index e) {
            for (Index s = b; s < e; ++s) sample(s / m, s % m);
        });
    else
        for (Index s = 0; s < samples; ++s) sample(s / m, s % m);
}

// ---------------------------------------------------------------------------
// Blocks and grouping (block.hpp:17-149)
// ---------------------------------------------------------------------------
struct Block {
    Index n = 0, m = 0;
    Mat data;
    std::vector<double> y0;
    static Index col(Index comp, Index traj, Index m) { return comp * m + traj; }
};

inline Block assemble_block(const State* states, Index m, const Grid& g, const Mat* guesses,
                            Index n_guesses) {  // :32-67
    if (m == 0 || m != n_guesses)
        throw ShapeError("assemble_block: need one guess per state, got " + std::to_string(n_guesses) +
                         " guesses for " + std::to_string(m) + " states");
    Block b;
    b.n = g.n;
    b.m = m;
    b.data.resize(g.n, state_dim * m);
    b.y0.assign(static_cast<std::size_t>(state_dim * m), 0.0);
    for (Index t = 0; t < m; ++t) {
        const Mat& gs = guesses[t];
        if (gs.r != g.n || gs.c != state_dim)
            throw AlignmentError("assemble_block: guess " + std::to_string(t) + " is " + std::to_string(gs.r) + "x" +
                                 std::to_string(gs.c) + ", expected " + std::to_string(g.n) + "x6");
        if (states[t].epoch != g.times[0])
            throw AlignmentError("assemble_block: state " + std::to_string(t) + " epoch " +
                                 std::to_string(states[t].epoch) + " does not match grid start " +
                                 std::to_string(g.times[0]));
        for (Index c = 0; c < state_dim; ++c) {
            const Index col = Block::col(c, t, m);
            for (Index j = 0; j < g.n; ++j) b.data(j, col) = gs(j, c);
            b.y0[col] = c < 3 ? states[t].r[static_cast<int>(c)] : states[t].v[static_cast<int>(c - 3)];
        }
    }
    return b;
}

inline std::vector<Mat> disassemble_block(const Block& b) {  // :70-80
    std::vector<Mat> out(static_cast<std::size_t>(b.m));
    for (Index t = 0; t < b.m; ++t) {
        out[t].resize(b.n, state_dim);
        for (Index c = 0; c < state_dim; ++c)
            for (Index j = 0; j < b.n; ++j) out[t](j, c) = b.data(j, Block::col(c, t, b.m));
    }
    return out;
}

struct Plan {  // :83-106
    Index total = 0;
    std::vector<Index> sizes, offsets, group_of, slot_of;
    Index groups() const { return static_cast<Index>(sizes.size()); }
    void rebuild() {
        offsets.assign(sizes.size(), 0);
        group_of.assign(static_cast<std::size_t>(total), 0);
        slot_of.assign(static_cast<std::size_t>(total), 0);
        Index at = 0;
        for (std::size_t g = 0; g < sizes.size(); ++g) {
            offsets[g] = at;
            for (Index s = 0; s < sizes[g]; ++s, ++at) {
                group_of[at] = static_cast<Index>(g);
                slot_of[at] = s;
            }
        }
    }
};

inline Plan split_groups(Index total, Index p) {  // :110-126
    if (total < 1 || p < 1 || p > total)
        throw InvalidPlanError("split_groups: cannot split " + std::to_string(total) + " states into " +
                               std::to_string(p) + " groups");
    Plan pl;
    pl.total = total;
    const Index base = total / p, rem = total % p;
    for (Index g = 0; g < p; ++g) pl.sizes.push_back(g < rem ? base + 1 : base);
    pl.rebuild();
    return pl;
}

inline Plan plan_from_sizes(std::vector<Index> sizes) {  // :134-149
    Index total = 0;
    for (Index s : sizes) {
        if (s < 1) throw InvalidPlanError("plan_from_sizes: group sizes must be positive");
        total += s;
    }
    if (total < 1) throw InvalidPlanError("plan_from_sizes: empty plan");
    Plan pl;
    pl.total = total;
    pl.sizes = std::move(sizes);
    pl.rebuild();
    return pl;
}

// ---------------------------------------------------------------------------
// Reductions (reduction.hpp:16-66)
// ---------------------------------------------------------------------------
inline int reduction_levels(std::size_t n) {
    if (n == 0) throw EmptyReductionError("reduction_levels: empty input");
    return static_cast<int>(std::bit_width(n - 1)) + 1;
}
inline double reduce_max(const double* v, std::size_t n) {
    if (n == 0) throw EmptyReductionError("reduce_max: empty input");
    double best = v[0];
    for (std::size_t i = 1; i < n; ++i) best = std::max(best, v[i]);
    return best;
}
inline double reduce_max_tree(const double* v, std::size_t n, Pool* pool = nullptr) {
    if (n == 0) throw EmptyReductionError("reduce_max_tree: empty input");
    std::vector<double> buf(v, v + n);
    Index len = static_cast<Index>(n);
    while (len > 1) {
        const Index pairs = len / 2;
        auto merge = [&](Index b, Index e) {
            for (Index i = b; i < e; ++i) buf[i] = std::max(buf[2 * i], buf[2 * i + 1]);
        };
        if (pool && pool->size() > 1 && pairs >= 1024)
            pool->chunks(pairs, merge);
        else
            merge(0, pairs);
        if (len % 2 == 1) {
            buf[pairs] = buf[len - 1];
            len = pairs + 1;
        } else {
            len = pairs;
        }
    }
    return buf[0];
}

// ---------------------------------------------------------------------------
// Convergence error (augment.hpp:32-104)
// ---------------------------------------------------------------------------
inline void sweep_error(const Mat& cur, const Mat& prev, Index m, ErrorMode mode, Index t0, Index t1,
                        std::vector<double>& worst) {  // :32-55
    for (Index j = 0; j < cur.r; ++j) {
        const double* c = cur.row(j);
        const double* p = prev.row(j);
        for (Index t = t0; t < t1; ++t) {
            double dr2 = 0, r2 = 0, dv2 = 0, v2 = 0;
            for (Index k = 0; k < 3; ++k) {
                const Index rc = k * m + t, vc = (k + 3) * m + t;
                const double dr = c[rc] - p[rc], dv = c[vc] - p[vc];
                dr2 += dr * dr;
                r2 += p[rc] * p[rc];
                dv2 += dv * dv;
                v2 += p[vc] * p[vc];
            }
            const double pos = component_error(std::sqrt(dr2), std::sqrt(r2), mode);
            const double vel = component_error(std::sqrt(dv2), std::sqrt(v2), mode);
            worst[t] = std::max(worst[t], std::max(pos, vel));
        }
    }
}

inline double block_max_error(const Mat& cur, const Mat& prev, Index m, ErrorMode mode,
                              Pool* pool = nullptr) {  // :61-77
    if (cur.r != prev.r || cur.c != prev.c || cur.c != state_dim * m) throw ShapeError("block_max_error: shape mismatch");
    std::vector<double> per(static_cast<std::size_t>(m), 0.0);
    if (pool && pool->size() > 1 && m >= 2) {
        pool->chunks(m, [&](Index b, Index e) { sweep_error(cur, prev, m, mode, b, e, per); });
        return reduce_max_tree(per.data(), per.size(), pool);
    }
    sweep_error(cur, prev, m, mode, 0, m, per);
    return reduce_max(per.data(), per.size());
}

inline std::vector<double> block_iteration_error(const Mat& cur, const Mat& prev, Index m, ErrorMode mode,
                                                 double* group_max) {  // :80-104
    if (cur.r != prev.r || cur.c != prev.c) throw ShapeError("block_iteration_error: block shapes do not match");
    std::vector<double> per(static_cast<std::size_t>(m), 0.0);
    sweep_error(cur, prev, m, mode, 0, m, per);
    if (group_max) *group_max = reduce_max(per.data(), per.size());
    return per;
}

// ---------------------------------------------------------------------------
// Fixed-point loop (picard.hpp:17-83) and group solve (augment.hpp:110-136)
// ---------------------------------------------------------------------------
struct Report {
    int iterations = 0;
    double final_error = std::numeric_limits<double>::infinity();
    bool converged = false;
    std::vector<double> history;
};

inline void throw_first_non_finite(const Mat& y) {  // picard.hpp:26-36
    for (Index j = 0; j < y.r; ++j)
        for (Index c = 0; c < y.c; ++c)
            if (!std::isfinite(y(j, c)))
                throw DivergenceError("picard iteration produced a non-finite value at node " + std::to_string(j) +
                                          ", column " + std::to_string(c),
                                      j, c);
}

template <typename Dyn, typename Err>
std::pair<Mat, Report> pc_solve(const Ops& o, Dyn&& dynamics, const Mat& y_init, const std::vector<double>& y0,
                                double tol, int max_it, Err&& error_fn, Pool* pool = nullptr) {  // :46-83
    if (tol <= 0.0) throw Error("pc_solve: tolerance must be positive");
    if (y_init.r != o.n || y_init.c != static_cast<Index>(y0.size()))
        throw ShapeError("pc_solve: initial block is " + std::to_string(y_init.r) + "x" + std::to_string(y_init.c) +
                         ", expected " + std::to_string(o.n) + "x" + std::to_string(y0.size()));
    Mat y = y_init, y_next(y.r, y.c), force(y.r, y.c);
    Report rep;
    for (int it = 1; it <= max_it; ++it) {
        dynamics(y, force);
        picard_update_into(o, force, y0, y_next, pool);
        if (!y_next.all_finite()) throw_first_non_finite(y_next);
        const double err = error_fn(y_next, y);
        std::swap(y, y_next);
        rep.iterations = it;
        rep.final_error = err;
        rep.history.push_back(err);
        if (err <= tol) {
            rep.converged = true;
            break;
        }
    }
    return {std::move(y), std::move(rep)};
}

using Clock = std::chrono::steady_clock;

inline std::pair<Block, Report> solve_group(Block block, const Grid& g, const Ops& o, const EphTable& t,
                                            const ForceConfig& cfg, double tol, int max_it,
                                            ErrorMode mode = ErrorMode::relative, Pool* inner = nullptr,
                                            int group_id = -1,
                                            Clock::time_point deadline = Clock::time_point::max()) {
    const Index m = block.m;
    auto dyn = [&](const Mat& y, Mat& f) {
        if (Clock::now() > deadline)
            throw TimeoutError("solve_group: wall-clock budget exhausted in group " + std::to_string(group_id));
        eval_force_block(y, m, g, t, cfg, f, inner);
    };
    auto err = [&](const Mat& c, const Mat& p) { return block_max_error(c, p, m, mode, inner); };
    try {
        auto [data, rep] = pc_solve(o, dyn, block.data, block.y0, tol, max_it, err, inner);
        block.data = std::move(data);
        return {std::move(block), std::move(rep)};
    } catch (const DivergenceError& e) {
        throw DivergenceError("group " + std::to_string(group_id) + ": " + e.what(), e.node, e.column);
    }
}

// ---------------------------------------------------------------------------
// Propagator (propagator.hpp:24-347)
// ---------------------------------------------------------------------------
/// hot = EXTENSION (BASELINE config 3; excluded by the reference): segment 0 is
/// warm; a later segment whose span equals the previous one starts from its own conic guess
/// plus the previous segment's (converged - starting guess) correction per node (Macomber's
/// hot start), otherwise warm.
enum class StartMode { warm, cold, hot };
enum class SegmentPolicy { single, per_orbit };
enum class Direction { forward, backward };

struct Segments {
    std::vector<double> boundaries;
    Index n_nodes = 200;
    Direction direction = Direction::forward;
    Index count() const { return static_cast<Index>(boundaries.size()) - 1; }
};

struct Config {  // :38-49
    Index n_nodes = 200;
    double tolerance = 1e-12;
    ErrorMode error_mode = ErrorMode::relative;
    int max_iterations = 100;
    StartMode start_mode = StartMode::warm;
    SegmentPolicy segment_policy = SegmentPolicy::single;
    double max_segment_periods = 1.0;
    ForceConfig force;
    Index p_groups = 1;
    double timeout_s = 0.0;
};

struct Exec {
    unsigned group_workers = 1, inner_workers = 1;
};

inline Mat cold_guess(const State& s, Index n) {  // :65-77
    Mat g(n, state_dim);
    for (Index j = 0; j < n; ++j) {
        g(j, 0) = s.r.x; g(j, 1) = s.r.y; g(j, 2) = s.r.z;
        g(j, 3) = s.v.x; g(j, 4) = s.v.y; g(j, 5) = s.v.z;
    }
    return g;
}

/// Conic guess per trajectory; non-elliptic states fall back to cold rows (:81-103).
inline Mat warm_guess(const State& s, const Grid& g, double mu, bool* fell_back) {
    Mat out(g.n, state_dim);
    *fell_back = false;
    try {
        for (Index j = 0; j < g.n; ++j) {
            const State sj = kepler_propagate(s, mu, g.times[j] - s.epoch);
            out(j, 0) = sj.r.x; out(j, 1) = sj.r.y; out(j, 2) = sj.r.z;
            out(j, 3) = sj.v.x; out(j, 4) = sj.v.y; out(j, 5) = sj.v.z;
        }
    } catch (const NonEllipticError&) {
        out = cold_guess(s, g.n);
        *fell_back = true;
    }
    return out;
}

/// EXTENSION: a hot start applies to segment seg >= 1 whose span equals the previous span
/// (to 1e-9 relative), so node j sits at the same phase of the representative orbit.
inline bool hot_applies(const Segments& sp, Index seg) {
    if (seg < 1) return false;
    const double a = sp.boundaries[seg + 1] - sp.boundaries[seg];
    const double b = sp.boundaries[seg] - sp.boundaries[seg - 1];
    return std::abs(a - b) <= 1e-9 * std::abs(b);
}

inline Segments plan_segments(const State& rep, double t0, double t1, double mu, SegmentPolicy policy, Index n,
                              double max_periods = 1.0) {  // :109-148
    if (t0 == t1) throw InvalidSpanError("plan_segments: degenerate span at t = " + std::to_string(t0));
    Segments p;
    p.n_nodes = n;
    p.direction = t1 > t0 ? Direction::forward : Direction::backward;
    const double span = t1 - t0;
    if (policy == SegmentPolicy::single) {
        std::optional<double> period;
        try {
            period = osculating_period(rep, mu);
        } catch (const NonEllipticError&) {
        }
        if (period && std::abs(span) > max_periods * (*period) * (1.0 + 1e-12))
            throw InvalidSpanError("plan_segments: span of " + std::to_string(std::abs(span)) + " s exceeds " +
                                   std::to_string(max_periods) + " nominal periods; use the per-orbit policy");
        p.boundaries = {t0, t1};
        return p;
    }
    const double period = osculating_period(rep, mu);
    const double step = std::copysign(max_periods * period, span);
    p.boundaries.push_back(t0);
    double at = t0;
    while ((t1 - at - step) * (span > 0 ? 1.0 : -1.0) > 1e-9 * period) {
        at += step;
        p.boundaries.push_back(at);
    }
    p.boundaries.push_back(t1);
    return p;
}

struct Result {  // :151-169
    std::vector<double> times;
    std::vector<Mat> trajectories;
    std::vector<State> terminal_states;
    std::vector<std::vector<Report>> reports;  // [segment][group]
    Plan plan;
    Segments segments;
    std::vector<std::string> warnings;
    int max_iterations_used() const {
        int w = 0;
        for (const auto& s : reports)
            for (const auto& r : s) w = std::max(w, r.iterations);
        return w;
    }
};

struct IncompleteError : Error {
    IncompleteError(const std::string& w, Index s, Index g, std::shared_ptr<const Result> p)
        : Error(w), segment(s), group(g), partial(std::move(p)) {}
    Index segment, group;
    std::shared_ptr<const Result> partial;
};

inline Result propagate(const std::vector<State>& states, const Plan& plan, const Segments& sp, const Config& cfg,
                        const Exec& exec = {}) {  // :192-347
    if (states.empty()) throw InvalidPlanError("propagate: empty batch");
    if (plan.total != static_cast<Index>(states.size()))
        throw InvalidPlanError("propagate: grouping plan covers " + std::to_string(plan.total) + " states, batch has " +
                               std::to_string(states.size()));
    if (sp.count() < 1) throw InvalidSpanError("propagate: empty segment plan");
    for (std::size_t i = 1; i < states.size(); ++i)
        if (states[i].epoch != states[0].epoch)
            throw AlignmentError("propagate: state " + std::to_string(i) + " epoch " + std::to_string(states[i].epoch) +
                                 " differs from shared epoch " + std::to_string(states[0].epoch));
    if (states[0].epoch != sp.boundaries.front())
        throw AlignmentError("propagate: batch epoch does not match the first segment boundary");

    const auto ops = cached_ops(sp.n_nodes);
    const Index n = sp.n_nodes, n_seg = sp.count(), n_traj = static_cast<Index>(states.size());
    const unsigned pool_size = std::max(exec.group_workers, exec.inner_workers);
    std::optional<Pool> pool;
    if (pool_size > 1) pool.emplace(pool_size);
    Pool* gpool = (pool && exec.group_workers > 1) ? &*pool : nullptr;
    Pool* ipool = (pool && exec.group_workers <= 1 && exec.inner_workers > 1) ? &*pool : nullptr;
    const auto deadline = cfg.timeout_s > 0.0
                              ? Clock::now() + std::chrono::duration_cast<Clock::duration>(
                                                   std::chrono::duration<double>(cfg.timeout_s))
                              : Clock::time_point::max();

    auto res = std::make_shared<Result>();
    res->plan = plan;
    res->segments = sp;
    const Index rows = 1 + n_seg * (n - 1);
    res->times.assign(static_cast<std::size_t>(rows), 0.0);
    res->trajectories.assign(static_cast<std::size_t>(n_traj), Mat(rows, state_dim));
    std::vector<State> cur(states);
    std::vector<Mat> base_prev(cfg.start_mode == StartMode::hot ? static_cast<std::size_t>(n_traj) : 0);

    for (Index seg = 0; seg < n_seg; ++seg) {
        const Grid g = build_grid(n, sp.boundaries[seg], sp.boundaries[seg + 1]);
        const EphTable tab =
            cfg.force.kind == ForceKind::n_body_1pn
                ? build_ephemeris_rel(cfg.force.bodies, g, cfg.force.central_mu, cfg.force.c_light)
                : build_ephemeris(has_bodies(cfg.force.kind) ? cfg.force.bodies : std::vector<Body>{}, g,
                                  cfg.force.central_mu);
        std::vector<Mat> guesses(static_cast<std::size_t>(n_traj));
        if (seg == 0 && cfg.start_mode == StartMode::cold) {
            for (Index i = 0; i < n_traj; ++i) guesses[i] = cold_guess(cur[i], n);
        } else {
            for (Index i = 0; i < n_traj; ++i) {
                bool fb = false;
                guesses[i] = warm_guess(cur[i], g, cfg.force.central_mu, &fb);
                if (fb)
                    res->warnings.push_back("segment " + std::to_string(seg) + ", trajectory " + std::to_string(i) +
                                            ": non-elliptic state, cold start used");
            }
        }
        // EXTENSION: hot start (see StartMode::hot)
        std::vector<Mat> base_now;
        if (cfg.start_mode == StartMode::hot) {
            base_now = guesses;
            if (hot_applies(sp, seg))
                for (Index i = 0; i < n_traj; ++i) {
                    const Mat& prev = res->trajectories[i];
                    const Index prow = (seg - 1) * (n - 1);
                    for (Index j = 0; j < n; ++j)
                        for (Index c = 0; c < state_dim; ++c)
                            guesses[i](j, c) += prev(prow + j, c) - base_prev[i](j, c);
                }
        }
        const Index P = plan.groups();
        std::vector<Block> blocks(static_cast<std::size_t>(P));
        std::vector<Report> reps(static_cast<std::size_t>(P));
        auto solve_one = [&](Index gi) {
            const Index off = plan.offsets[gi], sz = plan.sizes[gi];
            Block b = assemble_block(cur.data() + off, sz, g, guesses.data() + off, sz);
            auto [solved, rep] = solve_group(std::move(b), g, *ops, tab, cfg.force, cfg.tolerance, cfg.max_iterations,
                                             cfg.error_mode, ipool, static_cast<int>(gi), deadline);
            blocks[gi] = std::move(solved);
            reps[gi] = std::move(rep);
        };
        if (gpool)
            gpool->tasks(P, solve_one);
        else
            for (Index gi = 0; gi < P; ++gi) solve_one(gi);

        for (Index gi = 0; gi < P; ++gi) {
            if (!reps[gi].converged) {
                res->reports.push_back(reps);
                throw IncompleteError("propagate: group " + std::to_string(gi) + " did not converge in segment " +
                                          std::to_string(seg) + " (error " + std::to_string(reps[gi].final_error) +
                                          " after " + std::to_string(reps[gi].iterations) + " iterations)",
                                      seg, gi, res);
            }
        }
        res->reports.push_back(std::move(reps));
        const Index row0 = seg * (n - 1);
        for (Index j = (seg == 0 ? 0 : 1); j < n; ++j) res->times[row0 + j] = g.times[j];
        for (Index gi = 0; gi < P; ++gi) {
            const Block& b = blocks[gi];
            const Index off = plan.offsets[gi];
            for (Index s = 0; s < b.m; ++s) {
                Mat& tr = res->trajectories[off + s];
                for (Index j = (seg == 0 ? 0 : 1); j < n; ++j)
                    for (Index c = 0; c < state_dim; ++c) tr(row0 + j, c) = b.data(j, Block::col(c, s, b.m));
            }
        }
        for (Index i = 0; i < n_traj; ++i) {
            const Mat& tr = res->trajectories[i];
            const Index last = row0 + n - 1;
            cur[i].epoch = g.times[n - 1];
            cur[i].r = {tr(last, 0), tr(last, 1), tr(last, 2)};
            cur[i].v = {tr(last, 3), tr(last, 4), tr(last, 5)};
        }
        if (cfg.start_mode == StartMode::hot) base_prev = std::move(base_now);
    }
    res->terminal_states = std::move(cur);
    return std::move(*res);
}

// ---------------------------------------------------------------------------
// Runner (runner.hpp:21-159)
// ---------------------------------------------------------------------------
enum class RunMode { independent, augmented_sequential, augmented_parallel, grouped };

inline Plan grouping_for_mode(Index batch, RunMode mode, Index p) {  // :47-55
    switch (mode) {
    case RunMode::independent: return split_groups(batch, batch);
    case RunMode::augmented_sequential:
    case RunMode::augmented_parallel: return split_groups(batch, 1);
    case RunMode::grouped: return split_groups(batch, std::clamp<Index>(p, 1, batch));
    }
    throw InvalidPlanError("grouping_for_mode: invalid mode");
}

inline Result run_independent(const std::vector<State>& states, const Config& cfg, const Segments& sp,
                              unsigned workers) {  // :63-105
    const Index M = static_cast<Index>(states.size());
    std::vector<Result> singles(static_cast<std::size_t>(M));
    auto one = [&](Index i) {
        singles[i] = propagate(std::vector<State>{states[i]}, split_groups(1, 1), sp, cfg, {});
    };
    if (workers > 1) {
        Pool p(workers);
        p.tasks(M, one);
    } else {
        for (Index i = 0; i < M; ++i) one(i);
    }
    Result r;
    r.plan = split_groups(M, M);
    r.segments = sp;
    r.times = singles[0].times;
    r.reports.assign(static_cast<std::size_t>(sp.count()), std::vector<Report>(static_cast<std::size_t>(M)));
    for (Index i = 0; i < M; ++i) {
        r.trajectories.push_back(std::move(singles[i].trajectories[0]));
        r.terminal_states.push_back(singles[i].terminal_states[0]);
        for (Index s = 0; s < sp.count(); ++s) r.reports[s][i] = std::move(singles[i].reports[s][0]);
        for (auto& w : singles[i].warnings) r.warnings.push_back("trajectory " + std::to_string(i) + ": " + w);
    }
    return r;
}

struct Outcome {
    Result result;
    double wall_time_s = 0.0;
};

inline Outcome run_batch(const std::vector<State>& states, const Config& cfg, const Segments& sp, RunMode mode,
                         unsigned workers = 1) {  // :111-135
    if (workers < 1) throw InvalidPlanError("run_batch: need at least one worker");
    const auto t0 = Clock::now();
    Outcome o;
    if (mode == RunMode::independent) {
        o.result = run_independent(states, cfg, sp, workers);
    } else {
        const Plan plan = grouping_for_mode(static_cast<Index>(states.size()), mode, cfg.p_groups);
        Exec ex;
        if (mode == RunMode::augmented_parallel) ex = {1, workers};
        if (mode == RunMode::grouped) ex = {workers, 1};
        o.result = propagate(states, plan, sp, cfg, ex);
    }
    o.wall_time_s = std::chrono::duration<double>(Clock::now() - t0).count();
    return o;
}

inline double max_state_discrepancy(const Result& a, const Result& b) {  // :139-159
    if (a.trajectories.size() != b.trajectories.size()) throw ShapeError("max_state_discrepancy: different batch sizes");
    double worst = 0.0;
    for (std::size_t i = 0; i < a.trajectories.size(); ++i) {
        const Mat &ta = a.trajectories[i], &tb = b.trajectories[i];
        if (ta.r != tb.r) throw ShapeError("max_state_discrepancy: different sample counts");
        for (Index j = 0; j < ta.r; ++j) {
            const V3 ra{ta(j, 0), ta(j, 1), ta(j, 2)}, va{ta(j, 3), ta(j, 4), ta(j, 5)};
            const V3 rb{tb(j, 0), tb(j, 1), tb(j, 2)}, vb{tb(j, 3), tb(j, 4), tb(j, 5)};
            const double pos = component_error((ra - rb).norm(), rb.norm(), ErrorMode::relative);
            const double vel = component_error((va - vb).norm(), vb.norm(), ErrorMode::relative);
            worst = std::max(worst, std::max(pos, vel));
        }
    }
    return worst;
}

// ---------------------------------------------------------------------------
// Synthetic fixtures (synthetic.hpp:15-83) — reproduced bit-exactly
// ---------------------------------------------------------------------------
inline constexpr double mu_sun = 1.32712440018e11;

inline std::vector<Body> reference_bodies() {  // :19-29
    std::vector<Body> b(2);
    b[0].name = "venus-like";
    b[0].mu = 3.24858592e5;
    b[0].el = {1.08208e8, 0.0068, 0.0593, 1.338, 0.958, 2.10, 0.0};
    b[1].name = "earth-like";
    b[1].mu = 3.98600436e5;
    b[1].el = {1.495979e8, 0.0167, 0.0, 0.0, 1.796, 4.20, 0.0};
    return b;
}

inline State reference_state() {  // :31-34
    return elements_to_state({1.25e8, 0.12, 0.030, 0.30, 1.00, 0.0, 0.0}, mu_sun, 0.0);
}

inline ForceConfig reference_force(ForceKind kind = ForceKind::n_body) {  // :36-44
    ForceConfig c;
    c.kind = kind;
    c.central_mu = mu_sun;
    if (has_bodies(kind)) c.bodies = reference_bodies();
    return c;
}

inline std::uint64_t splitmix64(std::uint64_t& s) {  // :48-54
    s += 0x9e3779b97f4a7c15ULL;
    std::uint64_t z = s;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d649bb133111ebULL;
    return z ^ (z >> 31);
}
inline double symmetric_unit(std::uint64_t& s) {  // :57-59
    return 2.0 * (static_cast<double>(splitmix64(s) >> 11) * 0x1.0p-53) - 1.0;
}

inline std::vector<State> clone_batch(const State& base, Index count, double spread = 1e-5,
                                      std::uint64_t seed = 20220411ULL) {  // :66-83
    std::vector<State> out;
    out.reserve(static_cast<std::size_t>(count));
    std::uint64_t rng = seed;
    for (Index i = 0; i < count; ++i) {
        State s = base;
        if (i > 0) {
            for (int c = 0; c < 3; ++c) {
                s.r[c] *= 1.0 + spread * symmetric_unit(rng);
                s.v[c] *= 1.0 + spread * symmetric_unit(rng);
            }
        }
        out.push_back(s);
    }
    return out;
}

// ---------------------------------------------------------------------------
// Independent verifier: adaptive Fehlberg 7(8) (oracle.hpp:20-183)
// ---------------------------------------------------------------------------
struct RkConfig {
    double rel_tol = 1e-13, abs_tol = 1e-16;
    long max_steps = 4000000;
};

namespace rkf78 {
inline constexpr std::array<double, 13> c = {0.0,       2.0 / 27.0, 1.0 / 9.0, 1.0 / 6.0, 5.0 / 12.0, 0.5, 5.0 / 6.0,
                                             1.0 / 6.0, 2.0 / 3.0,  1.0 / 3.0, 1.0,       0.0,        1.0};
inline constexpr std::array<std::array<double, 12>, 13> a = {{
    {},
    {2.0 / 27.0},
    {1.0 / 36.0, 1.0 / 12.0},
    {1.0 / 24.0, 0.0, 1.0 / 8.0},
    {5.0 / 12.0, 0.0, -25.0 / 16.0, 25.0 / 16.0},
    {1.0 / 20.0, 0.0, 0.0, 1.0 / 4.0, 1.0 / 5.0},
    {-25.0 / 108.0, 0.0, 0.0, 125.0 / 108.0, -65.0 / 27.0, 125.0 / 54.0},
    {31.0 / 300.0, 0.0, 0.0, 0.0, 61.0 / 225.0, -2.0 / 9.0, 13.0 / 900.0},
    {2.0, 0.0, 0.0, -53.0 / 6.0, 704.0 / 45.0, -107.0 / 9.0, 67.0 / 90.0, 3.0},
    {-91.0 / 108.0, 0.0, 0.0, 23.0 / 108.0, -976.0 / 135.0, 311.0 / 54.0, -19.0 / 60.0, 17.0 / 6.0, -1.0 / 12.0},
    {2383.0 / 4100.0, 0.0, 0.0, -341.0 / 164.0, 4496.0 / 1025.0, -301.0 / 82.0, 2133.0 / 4100.0, 45.0 / 82.0,
     45.0 / 164.0, 18.0 / 41.0},
    {3.0 / 205.0, 0.0, 0.0, 0.0, 0.0, -6.0 / 41.0, -3.0 / 205.0, -3.0 / 41.0, 3.0 / 41.0, 6.0 / 41.0, 0.0},
    {-1777.0 / 4100.0, 0.0, 0.0, -341.0 / 164.0, 4496.0 / 1025.0, -289.0 / 82.0, 2193.0 / 4100.0, 51.0 / 82.0,
     33.0 / 164.0, 12.0 / 41.0, 0.0, 1.0},
}};
inline constexpr std::array<double, 13> b8 = {0.0,         0.0,         0.0,         0.0,       0.0,
                                              34.0 / 105.0, 9.0 / 35.0,  9.0 / 35.0,  9.0 / 280.0, 9.0 / 280.0,
                                              0.0,         41.0 / 840.0, 41.0 / 840.0};
}  // namespace rkf78

using S6 = std::array<double, 6>;

template <typename Deriv>
State rk_propagate(const State& start, Deriv&& deriv, double t_end, const RkConfig& cfg = {}) {  // :63-132
    if (!(cfg.rel_tol > 0.0) || !(cfg.abs_tol > 0.0)) throw OracleError("rk_propagate: tolerances must be positive");
    double t = start.epoch;
    const double span = t_end - t;
    if (span == 0.0) return start;
    S6 y{start.r.x, start.r.y, start.r.z, start.v.x, start.v.y, start.v.z};
    const double dir = span > 0.0 ? 1.0 : -1.0;
    double h = span / 50.0;
    long steps = 0;
    std::array<S6, 13> k{};
    while (t != t_end) {
        bool last = false;
        if ((t + h - t_end) * dir >= 0.0) {
            h = t_end - t;
            last = true;
        }
        for (int i = 0; i < 13; ++i) {
            S6 yi = y;
            for (int l = 0; l < i; ++l) {
                const double alk = rkf78::a[i][l];
                if (alk != 0.0) {
                    const double ha = h * alk;
                    for (int q = 0; q < 6; ++q) yi[q] += ha * k[l][q];
                }
            }
            k[i] = deriv(t + rkf78::c[i] * h, yi);
        }
        S6 y8 = y;
        for (int i = 0; i < 13; ++i) {
            if (rkf78::b8[i] != 0.0) {
                const double hb = h * rkf78::b8[i];
                for (int q = 0; q < 6; ++q) y8[q] += hb * k[i][q];
            }
        }
        double err = 0.0;
        const double hd = h * (41.0 / 840.0);
        for (int q = 0; q < 6; ++q) {
            const double defect = hd * (k[0][q] + k[10][q] - k[11][q] - k[12][q]);
            const double scale = cfg.abs_tol + cfg.rel_tol * std::max(std::abs(y[q]), std::abs(y8[q]));
            err = std::max(err, std::abs(defect) / scale);
        }
        if (err <= 1.0) {
            y = y8;
            t = last ? t_end : t + h;
        }
        const double factor = (err > 0.0) ? std::clamp(0.9 * std::pow(err, -1.0 / 8.0), 0.2, 4.0) : 4.0;
        h *= factor;
        if (t + h == t) throw OracleError("rk_propagate: step size underflow at t = " + std::to_string(t));
        if (++steps > cfg.max_steps) throw OracleError("rk_propagate: exceeded " + std::to_string(cfg.max_steps) + " steps");
    }
    State out;
    out.epoch = t_end;
    out.r = {y[0], y[1], y[2]};
    out.v = {y[3], y[4], y[5]};
    return out;
}

template <typename Deriv>
Mat rk_sample(const State& start, Deriv&& deriv, const std::vector<double>& times, const RkConfig& cfg = {}) {  // :136-150
    if (times.empty() || times[0] != start.epoch)
        throw OracleError("oracle_sample_trajectory: sample times must begin at the state epoch");
    Mat out(static_cast<Index>(times.size()), state_dim);
    State cur = start;
    auto put = [&](Index j) {
        out(j, 0) = cur.r.x; out(j, 1) = cur.r.y; out(j, 2) = cur.r.z;
        out(j, 3) = cur.v.x; out(j, 4) = cur.v.y; out(j, 5) = cur.v.z;
    };
    put(0);
    for (std::size_t j = 1; j < times.size(); ++j) {
        cur = rk_propagate(cur, deriv, times[j], cfg);
        put(static_cast<Index>(j));
    }
    return out;
}

/// Max over nodes of the relative position/velocity discrepancy (oracle.hpp:154-183).
inline double compare_trajectories(const Mat& cand, const Mat& ref) {
    if (cand.r != ref.r || cand.c != state_dim || ref.c != state_dim)
        throw ShapeError("compare_trajectories: sample shapes do not match");
    double worst = 0.0;
    for (Index j = 0; j < cand.r; ++j) {
        const V3 dr{cand(j, 0) - ref(j, 0), cand(j, 1) - ref(j, 1), cand(j, 2) - ref(j, 2)};
        const V3 dv{cand(j, 3) - ref(j, 3), cand(j, 4) - ref(j, 4), cand(j, 5) - ref(j, 5)};
        const double rn = std::max(V3{ref(j, 0), ref(j, 1), ref(j, 2)}.norm(), 1e-30);
        const double vn = std::max(V3{ref(j, 3), ref(j, 4), ref(j, 5)}.norm(), 1e-30);
        worst = std::max(worst, std::max(dr.norm() / rn, dv.norm() / vn));
    }
    return worst;
}

/// Newtonian derivative callback for rk_propagate (state -> [v, a(r, t)]).
inline auto nbody_deriv(const ForceConfig& cfg) {
    return [&cfg](double t, const S6& y) {
        const V3 a = acceleration_at({y[0], y[1], y[2]}, {y[3], y[4], y[5]}, t, cfg);
        return S6{y[3], y[4], y[5], a.x, a.y, a.z};
    };
}

}  // namespace pswarm_ref
