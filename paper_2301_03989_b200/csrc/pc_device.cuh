// Device building blocks of the B200 (sm_100a) augmented Picard–Chebyshev path.
//
//   * dmma()            FP64 tensor-core MMA (mma.sync m8n8k4 f64 -> SASS DMMA.8x8x4);
//                       tcgen05 has no f64 kind, so this is the FP64 tensor path on B200.
//   * conic_*/kepler_*  warm-start conic (kepler.hpp:26-98) evaluated per (node, trajectory).
//   * accel()           Newtonian restricted N-body acceleration with the reference's
//                       singularity guards (force_model.hpp:26-69), rsqrt formulation.
//   * tile GEMM         Y' = U'·F for one CTA tile: all N+1 rows (N nodes + the anchor
//                       row of pc_matrices.hpp:98-100) × 48 columns (8 trajectories × 6
//                       components), K = N, operator streamed from L2, F from smem.
//
// Layout conventions (DESIGN.md §Data layout):
//   Ybuf  smem  [node j][component c ^ (j&1)][slot t], row stride 48 doubles (the pair
//               swap on odd rows makes the double2 epilogue stores bank-conflict-free);
//   Fbuf  smem  fragment-native B operand: [kstep][ntile pair][lane][2] doubles, so every
//               B-fragment fetch of a warp is one contiguous 512-byte LDS.128;
//   Upack gmem  fragment-native A operand: [mtile][kstep pair][lane] double2 (LDG.128).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace pswarm_dev {

constexpr int SLOTS = 8;             // trajectories per CTA tile
constexpr int COLS = 6 * SLOTS;      // 48 block columns: column = comp*8 + slot
constexpr double PI = 3.141592653589793238462643383279502884;

// ---------------------------------------------------------------- DMMA ---
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
#ifdef PSWARM_DMMA_VOLATILE
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
#else  // pure register op: let the compiler schedule it against the operand loads
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
        : "+d"(c0), "+d"(c1)
        : "d"(a), "d"(b));
#endif
}

// ------------------------------------------------- bulk copy (TMA engine) ---
/// One-shot global -> shared staging through the TMA unit: cp.async.bulk (SASS UBLKCP)
/// completing on an mbarrier's transaction count.  One thread arms the barrier and issues
/// the copies; every consumer waits on phase 0.  Addresses 16-byte aligned, sizes
/// multiples of 16 bytes, at most 2^20 - 1 bytes per barrier phase.
__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned phase) {
    asm volatile(
        "{\n .reg .pred p;\n"
        "WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}
/// Stage `bytes` (multiple of 16) from global to shared memory in <= 64 KB bulk copies on
/// one barrier (thread `leader` issues; the caller waits with mbar_wait(bar, 0)).
__device__ __forceinline__ void bulk_stage(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    mbar_expect_tx(bar, bytes);
    for (unsigned o = 0; o < bytes; o += 65536u)
        bulk_g2s(static_cast<char*>(dst) + o, static_cast<const char*>(src) + o, min(65536u, bytes - o), bar);
}

__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// --------------------------------------------------------------- conics ---
enum ConicStatus : int { CONIC_OK = 0, CONIC_NON_ELLIPTIC = 1, CONIC_ZERO_RADIUS = 2, CONIC_SOLVER = 3 };

/// Newton solve of E - e sin E = M (kepler.hpp:26-42).
__device__ __forceinline__ int solve_kepler(double mean_anomaly, double ecc, double* e_out) {
    const double mw = remainder(mean_anomaly, 2.0 * PI);
    double e = (ecc < 0.8) ? mw : copysign(PI, mw);
    for (int it = 0; it < 50; ++it) {
        double s, c;
        sincos(e, &s, &c);
        const double f = e - ecc * s - mw;
        const double fp = 1.0 - ecc * c;
        const double step = f / fp;
        e -= step;
        if (fabs(step) <= 1e-14) {
            *e_out = e + (mean_anomaly - mw);
            return CONIC_OK;
        }
    }
    return CONIC_SOLVER;
}

/// Bound-conic test of kepler_propagate (kepler.hpp:60-79) independent of dt, so every
/// node of a trajectory reaches the same warm/cold decision (propagator.hpp:86-99).
__device__ __forceinline__ int conic_check(const double r[3], const double v[3], double mu) {
    const double r0n = sqrt(r[0] * r[0] + r[1] * r[1] + r[2] * r[2]);
    if (!(r0n > 0.0)) return CONIC_ZERO_RADIUS;
    const double energy = 0.5 * (v[0] * v[0] + v[1] * v[1] + v[2] * v[2]) - mu / r0n;
    if (!(energy < 0.0)) return CONIC_NON_ELLIPTIC;
    const double a = -mu / (2.0 * energy);
    const double esin = (r[0] * v[0] + r[1] * v[1] + r[2] * v[2]) / sqrt(mu * a);
    const double ecos = 1.0 - r0n / a;
    if (hypot(esin, ecos) >= 1.0 - 1e-8) return CONIC_NON_ELLIPTIC;
    return CONIC_OK;
}

/// Conic propagation by dt (kepler.hpp:59-98); caller has passed conic_check.
/// dt == 0 returns the input exactly (kepler.hpp:69-71).
__device__ __forceinline__ int kepler_propagate(const double r[3], const double v[3], double mu, double dt,
                                                double ro[3], double vo[3], double* m_fail, double* e_fail) {
    if (dt == 0.0) {
        for (int i = 0; i < 3; ++i) {
            ro[i] = r[i];
            vo[i] = v[i];
        }
        return CONIC_OK;
    }
    const double r0n = sqrt(r[0] * r[0] + r[1] * r[1] + r[2] * r[2]);
    const double energy = 0.5 * (v[0] * v[0] + v[1] * v[1] + v[2] * v[2]) - mu / r0n;
    const double a = -mu / (2.0 * energy);
    const double n = sqrt(mu / (a * a * a));
    const double esin = (r[0] * v[0] + r[1] * v[1] + r[2] * v[2]) / sqrt(mu * a);
    const double ecos = 1.0 - r0n / a;
    const double ecc = hypot(esin, ecos);
    const double e0 = atan2(esin, ecos);
    const double m1 = (e0 - esin) + n * dt;
    double e1;
    if (solve_kepler(m1, ecc, &e1) != CONIC_OK) {
        *m_fail = m1;
        *e_fail = ecc;
        return CONIC_SOLVER;
    }
    const double de = e1 - e0;
    double sde, cde;
    sincos(de, &sde, &cde);
    const double f = 1.0 - (a / r0n) * (1.0 - cde);
    const double g = dt + (sde - de) / n;
    const double r1n = a * (1.0 - ecc * cos(e1));
    const double fdot = -sqrt(mu * a) * sde / (r1n * r0n);
    const double gdot = 1.0 - (a / r1n) * (1.0 - cde);
    for (int i = 0; i < 3; ++i) {
        ro[i] = f * r[i] + g * v[i];
        vo[i] = fdot * r[i] + gdot * v[i];
    }
    return CONIC_OK;
}

/// Position of an analytic body at epoch t (elements_to_state, kepler.hpp:102-131); the
/// host has already validated the elements (bound conic).
__device__ __forceinline__ int elements_position(const double* el, double mu, double t, double out[3], double* m_fail) {
    const double a = el[0], e = el[1], inc = el[2], raan = el[3], argp = el[4], m0 = el[5], ep = el[6];
    const double n = sqrt(mu / (a * a * a));
    const double m = m0 + n * (t - ep);
    double ea;
    if (solve_kepler(m, e, &ea) != CONIC_OK) {
        *m_fail = m;
        return CONIC_SOLVER;
    }
    double se, ce, so, co, si, ci, sw, cw;
    sincos(ea, &se, &ce);
    sincos(raan, &so, &co);
    sincos(inc, &si, &ci);
    sincos(argp, &sw, &cw);
    const double beta = sqrt(1.0 - e * e);
    const double xp = a * (ce - e), yp = a * beta * se;
    const double p[3] = {co * cw - so * sw * ci, so * cw + co * sw * ci, sw * si};
    const double q[3] = {-co * sw - so * cw * ci, -so * sw + co * cw * ci, cw * si};
    for (int c = 0; c < 3; ++c) out[c] = xp * p[c] + yp * q[c];
    return CONIC_OK;
}

/// Position and velocity of an analytic body (elements_to_state, kepler.hpp:102-131);
/// the velocity feeds the relativistic model only (EXTENSION).
__device__ __forceinline__ int elements_state(const double* el, double mu, double t, double r[3], double v[3],
                                              double* m_fail) {
    const double a = el[0], e = el[1], inc = el[2], raan = el[3], argp = el[4], m0 = el[5], ep = el[6];
    const double n = sqrt(mu / (a * a * a));
    const double m = m0 + n * (t - ep);
    double ea;
    if (solve_kepler(m, e, &ea) != CONIC_OK) {
        *m_fail = m;
        return CONIC_SOLVER;
    }
    double se, ce, so, co, si, ci, sw, cw;
    sincos(ea, &se, &ce);
    sincos(raan, &so, &co);
    sincos(inc, &si, &ci);
    sincos(argp, &sw, &cw);
    const double beta = sqrt(1.0 - e * e);
    const double rn = a * (1.0 - e * ce);
    const double xp = a * (ce - e), yp = a * beta * se;
    const double vs = sqrt(mu * a) / rn;
    const double vxp = -vs * se, vyp = vs * beta * ce;
    const double p[3] = {co * cw - so * sw * ci, so * cw + co * sw * ci, sw * si};
    const double q[3] = {-co * sw - so * cw * ci, -so * sw + co * cw * ci, cw * si};
    for (int c = 0; c < 3; ++c) {
        r[c] = xp * p[c] + yp * q[c];
        v[c] = vxp * p[c] + vyp * q[c];
    }
    return CONIC_OK;
}

/// d/dx of a Chebyshev series: sum_k k c_k U_{k-1}(x) by Clenshaw on the U recurrence
/// (EXTENSION: velocities of tabulated bodies for the relativistic model).
__device__ __forceinline__ double clenshaw_deriv(const double* c, int nc, double x) {
    double b1 = 0.0, b2 = 0.0;
    for (int k = nc - 1; k >= 1; --k) {
        const double b0 = k * c[k] + 2.0 * x * b1 - b2;
        b2 = b1;
        b1 = b0;
    }
    return b1;
}

/// EXTENSION (hot start, StartMode::hot): the starting guess of a node is its conic (or
/// cold) base guess plus the previous segment's (converged - base) correction hb when the
/// segment spans match (apply); hb then keeps this segment's base for hot_retire_node.
__device__ __forceinline__ void hot_start_node(double* hb, int apply, double ro[3], double vo[3]) {
    const double base[6] = {ro[0], ro[1], ro[2], vo[0], vo[1], vo[2]};
    if (apply)
        for (int c = 0; c < 3; ++c) {
            ro[c] = base[c] + hb[c];
            vo[c] = base[3 + c] + hb[3 + c];
        }
    for (int c = 0; c < 6; ++c) hb[c] = base[c];
}

/// EXTENSION (hot start): correction carried to the next segment = converged - base.
__device__ __forceinline__ void hot_retire_node(double* hb, int c, double y) { hb[c] = y - hb[c]; }

/// Clenshaw evaluation of a Chebyshev series (ephemeris.hpp:29-38).
__device__ __forceinline__ double clenshaw(const double* c, int nc, double x) {
    double b1 = 0.0, b2 = 0.0;
    for (int k = nc - 1; k >= 1; --k) {
        const double b0 = c[k] + 2.0 * x * b1 - b2;
        b2 = b1;
        b1 = b0;
    }
    return c[0] + x * b1 - b2;
}

/// 1/sqrt(x) for normal positive x: MUFU.RSQ64H seed (rsqrt.approx.f64, ~2^-23) and
/// two Newton steps (error < 1 ulp level).  The force arguments are squared distances
/// of 1e-2..1e20 km^2, far from the denormal/overflow cases CUDA's rsqrt() guards
/// with a slow-path branch.
__device__ __forceinline__ double rsqrt_seed(double x) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    return y;
}

/// One Newton-Raphson step for 1/sqrt(x): y (1.5 - 0.5 x y^2).
__device__ __forceinline__ double rsqrt_newton(double x, double y) {
    return y * fma(-0.5 * x * y, y, 1.5);
}

/// mu / |d|^3 for a perturbing body from d2 = |d|^2, with the single Newton step of the
/// planet terms folded into the cube: e = 3 - d2 y0^2, y1 = y0 e / 2 (the Newton iterate),
/// mu y1^3 = (mu / 8) (y0 e)^3 — 2 DMUL + 1 DFMA for the step and 3 DMUL for the cube
/// (mu8 = mu / 8, exact).  Same iterate as rsqrt_newton up to rounding.
__device__ __forceinline__ double body_mu_ir3(double d2, double mu8) {
    const double y0 = rsqrt_seed(d2);
    const double y1h = y0 * fma(-d2 * y0, y0, 3.0);  // 2 / |d|
    return (mu8 * y1h) * (y1h * y1h);
}

/// d2 < bound for non-negative doubles (d2 is a sum of squares, bound >= 0) as a 64-bit
/// integer compare on the IEEE bits: the proximity pre-test stays off the FP64 pipe,
/// which the force shares with the DMMA stream.  NaN d2 compares false, as with <.
__device__ __forceinline__ bool below_bits(double d2, long long bound_bits) {
    return __double_as_longlong(d2) < bound_bits;
}

__device__ __forceinline__ double rsqrt_nr(double x) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    const double hx = 0.5 * x;
    y = y * fma(-hx * y, y, 1.5);
    y = y * fma(-hx * y, y, 1.5);
    return y;
}

// ---------------------------------------------------------------- force ---
/// Per-segment force data.  body_pos [N][B][3] frozen per node (ephemeris.hpp:89-107);
/// indirect [N][3] = sum_b mu_b r_b/|r_b|^3, the node-constant half of
/// perturber_acceleration (force_model.hpp:50-51), built on the host.
struct ForceData {
    const double* body_pos;
    const double* body_mu;
    const double* indirect;
    double central_mu;
    double floor_km;
    double floor2_hi;  // floor^2 * (1 + 1e-9): cheap pre-test before the exact sqrt compare
    long long floor2_hi_bits;  // its IEEE bits (integer pre-test, below_bits)
    int n_bodies;      // 0 for two-body
    int rel;           // 1: n_body_1pn (EXTENSION) -> add rel_correction()
    double ic2;        // 1 / c^2 (km^-2 s^2)
    const double* rel_tab;  // [N][rel_stride(B)]: Sun + bodies + indirect term at each node (k_ephemeris)
    const double* eph_t;    // [3B + 3][eph_ld(N)]: positions (3b + c) then the indirect term, node-contiguous
};

// ------------------------------------------------------- relativistic (EXTENSION) ---
/// Row of the per-node relativistic table: massive body A (A = 0 Sun at the origin)
/// position, velocity, Newtonian heliocentric acceleration, mu and
/// K_A = (2 v_A^2 - phi_A) / c^2 with phi_A the potential of the other massive bodies at A.
constexpr int REL_W = 12;
/// Node stride of the relativistic table (doubles): B + 1 rows of REL_W, then the node's
/// indirect term [3]; odd, so consecutive nodes (the force threads of a warp) fall in
/// distinct shared-memory banks when the table is staged.
__host__ __device__ constexpr int rel_stride(int B) { return (B + 1) * REL_W + 3; }
/// Row length of the node-contiguous ephemeris eph_t (N rounded up to even: 16-byte rows).
__host__ __device__ constexpr int eph_ld(int N) { return (N + 1) & ~1; }
/// Doubles of the per-segment table a slot kernel stages in shared memory (16-byte multiple).
__host__ __device__ constexpr size_t eph_stage_doubles(int N, int B, bool rel) {
    return rel ? ((static_cast<size_t>(N) * rel_stride(B) + 1) & ~static_cast<size_t>(1))
               : static_cast<size_t>(3 * B + 3) * eph_ld(N);
}

/// First post-Newtonian (EIH, beta = gamma = 1) correction for a massless particle
/// (Explanatory Supplement 1992 eq. 8.1) in one pass over the massive
/// bodies: the -4U/c^2 and v^2/c^2 terms factor out of the Newtonian sum, so
///   da = (v^2 - 4U)/c^2 a_N + sum_A g_A [K_A - (4 v.v_A + 1.5 (d.v_A)^2/rho^2 - 0.5 d.a_A)/c^2] d
///        + 1/c^2 sum_A g_A (-d.(4v - 3v_A)) (v - v_A) + 3.5/c^2 sum_A mu_A a_A / rho,
/// d = r_A - r, g_A = mu_A / rho^3.  The oracle evaluates the textbook two-pass form.
static __device__ __noinline__ void rel_correction(double rx, double ry, double rz, double vx, double vy, double vz,
                                            const double* __restrict__ tab, int nb1, double ic2, double* out) {
    double U = 0.0, nx = 0.0, ny = 0.0, nz = 0.0, bx = 0.0, by = 0.0, bz = 0.0;
    double wx = 0.0, wy = 0.0, wz = 0.0, qx = 0.0, qy = 0.0, qz = 0.0;
    for (int A = 0; A < nb1; ++A) {
        const double* t = tab + A * REL_W;
        const double dx = t[0] - rx, dy = t[1] - ry, dz = t[2] - rz;
        const double d2 = dx * dx + dy * dy + dz * dz;
        const double ir = rsqrt_nr(d2);
        const double mu = t[9];
        const double g = mu * ir * ir * ir;
        U += mu * ir;
        nx += g * dx;
        ny += g * dy;
        nz += g * dz;
        const double vax = t[3], vay = t[4], vaz = t[5];
        const double vva = vx * vax + vy * vay + vz * vaz;
        const double dva = dx * vax + dy * vay + dz * vaz;
        const double daa = dx * t[6] + dy * t[7] + dz * t[8];
        const double br = g * (t[10] - ic2 * (4.0 * vva + 1.5 * dva * dva * (ir * ir) - 0.5 * daa));
        bx += br * dx;
        by += br * dy;
        bz += br * dz;
        const double w = -g * (dx * (4.0 * vx - 3.0 * vax) + dy * (4.0 * vy - 3.0 * vay) + dz * (4.0 * vz - 3.0 * vaz));
        wx += w * (vx - vax);
        wy += w * (vy - vay);
        wz += w * (vz - vaz);
        const double m = mu * ir;
        qx += m * t[6];
        qy += m * t[7];
        qz += m * t[8];
    }
    const double f = ic2 * (vx * vx + vy * vy + vz * vz - 4.0 * U);
    out[0] = f * nx + bx + ic2 * wx + 3.5 * ic2 * qx;
    out[1] = f * ny + by + ic2 * wy + 3.5 * ic2 * qy;
    out[2] = f * nz + bz + ic2 * wz + 3.5 * ic2 * qz;
}

/// Acceleration at node j (force_model.hpp:57-69).  Returns -1 when finite and legal,
/// else the index of the first failing check in reference order: 0 = central body
/// (|r| not > 0, force_model.hpp:28), 1 + b = body b closer than the floor (:44).
/// `bp` = this node's [B][3] body positions, `ind` = its indirect term (shared or global).
__device__ __forceinline__ int accel(double rx, double ry, double rz, const double* bp, const double* ind,
                                     const ForceData& fd, double& ax, double& ay, double& az) {
    const double r2 = rx * rx + ry * ry + rz * rz;
    if (!(r2 > 0.0)) return 0;
    const double ir = rsqrt(r2);
    const double s = -fd.central_mu * (ir * ir * ir);
    ax = s * rx;
    ay = s * ry;
    az = s * rz;
    const int B = fd.n_bodies;
    if (B > 0) {
        int fail = -1;
        for (int b = 0; b < B; ++b) {
            const double dx = bp[3 * b + 0] - rx;
            const double dy = bp[3 * b + 1] - ry;
            const double dz = bp[3 * b + 2] - rz;
            const double d2 = dx * dx + dy * dy + dz * dz;
            if (d2 < fd.floor2_hi && fail < 0 && sqrt(d2) < fd.floor_km) fail = 1 + b;
            const double id = rsqrt(d2);
            const double k = __ldg(fd.body_mu + b) * (id * id * id);
            ax += k * dx;
            ay += k * dy;
            az += k * dz;
        }
        ax -= ind[0];
        ay -= ind[1];
        az -= ind[2];
        return fail;
    }
    return -1;
}

/// Distance behind a failing check (for the SingularityError message, force_model.hpp:44-49).
__device__ __forceinline__ double check_distance(double rx, double ry, double rz, int j, int check,
                                                 const ForceData& fd) {
    if (check <= 0) return sqrt(rx * rx + ry * ry + rz * rz);
    const double* bp = fd.body_pos + (static_cast<size_t>(j) * fd.n_bodies + (check - 1)) * 3;  // global copy
    const double dx = bp[0] - rx, dy = bp[1] - ry, dz = bp[2] - rz;
    return sqrt(dx * dx + dy * dy + dz * dz);
}

// ----------------------------------------------------------- tile GEMM ---
/// Ybuf address of (node j, component c, slot t): components of odd rows are
/// pair-swapped so the 8 rows of an MMA fragment hit two 64-byte bank windows
/// (conflict-free double2 epilogue stores with a 48-double row stride).
__device__ __forceinline__ int yidx(int j, int c, int t) { return j * COLS + ((c ^ (j & 1)) << 3) + t; }

/// Fragment-native index of B element (k, n) in Fbuf (doubles): B fragment of
/// mma.m8n8k4 holds B[k = lane%4][n = lane/4]; two n-tiles share one double2.
__device__ __forceinline__ int fbuf_index(int k, int n) {
    const int ks = k >> 2, kk = k & 3, nt = n >> 3, nn = n & 7;
    return (((ks * 3 + (nt >> 1)) * 32) + (nn * 4 + kk)) * 2 + (nt & 1);
}

/// Warp work plan of the 8-row x 8-column output tiles (mtiles x 6 n-tiles).
/// Warp w owns `main` full-width m-tiles [w*main, w*main+main) plus up to XMAX single
/// extra tiles e = w + k*warps (< extras): m-tile mb + e/6, n-tile e%6.  The host picks
/// warps as a multiple of 4 so every SM sub-partition (SMSP) issues the same number of
/// DMMAs — the DMMA pipe is per SMSP, so an uneven warp count idles three of them.
struct GemmPlan {
    int warps;   // multiple of 4
    int main;    // full-width m-tiles per warp (0..2)
    int mb;      // first extra m-tile = main*warps
    int extras;  // number of extra (m-tile, n-tile) tiles
    int mtiles;  // ceil((N+1)/8), row N is the anchor row
    int xmax;    // extra tiles per warp the kernel variant holds (XMAX or XMAX_SMALL)
};
constexpr int XMAX = 2;        // extra tiles per warp, large-N kernels
constexpr int XMAX_SMALL = 6;  // extra tiles per warp, N < 63 (fewer than 8 m-tiles)

/// Per-warp operator pointers (one per owned tile row-block), hoisted out of the
/// k loop; pair kp of a tile is at ptr + kp*32.
template <int XM>
struct AWarp {
    const double2* m0;
    const double2* m1;
    const double2* x[XM];
    int xoff[XM];  // B-fragment double offset of the extra tile's n-tile within a k-step
    bool hx[XM];
};

template <int XM>
__device__ __forceinline__ AWarp<XM> a_warp(const double2* __restrict__ upack, int nkp, const GemmPlan& gp, int warp,
                                            int lane) {
    AWarp<XM> w;
    w.m0 = upack + static_cast<size_t>(warp * gp.main) * nkp * 32 + lane;
    w.m1 = w.m0 + static_cast<size_t>(nkp) * 32;
#pragma unroll
    for (int x = 0; x < XM; ++x) {
        const int e = warp + x * gp.warps;
        w.hx[x] = e < gp.extras;
        const int mt = w.hx[x] ? gp.mb + e / 6 : 0;
        w.x[x] = upack + static_cast<size_t>(mt) * nkp * 32 + lane;
        const int n = e % 6;
        w.xoff[x] = ((n >> 1) * 32 + lane) * 2 + (n & 1);  // + ks*192 per k-step
    }
    return w;
}

template <int XM>
struct APair {  // one k-step pair of A fragments for every tile the warp owns
    double2 m0, m1, x[XM];
};

template <int XM>
__device__ __forceinline__ void load_apair(const AWarp<XM>& w, int nmain, int kp, APair<XM>& p) {
    if (nmain > 0) p.m0 = __ldg(w.m0 + kp * 32);
    if (nmain > 1) p.m1 = __ldg(w.m1 + kp * 32);
#pragma unroll
    for (int x = 0; x < XM; ++x)
        if (w.hx[x]) p.x[x] = __ldg(w.x[x] + kp * 32);
}

/// Prefetched first k-step pair (issued before the force phase to hide L2 latency).
template <int XM>
struct APrefetch {
    APair<XM> p;
};

template <int XM>
__device__ __forceinline__ APrefetch<XM> gemm_prefetch(const double2* __restrict__ upack, int nkp, const GemmPlan& gp,
                                                       int warp, int lane) {
    APrefetch<XM> f;
    const AWarp<XM> w = a_warp<XM>(upack, nkp, gp, warp, lane);
    load_apair<XM>(w, gp.main, 0, f.p);
    return f;
}

/// Two k-steps (one operator pair) of the warp's tiles.
template <int XM>
__device__ __forceinline__ void gemm_pair(const double* fbuf, const AWarp<XM>& w, int nmain, int lane, int kp,
                                          const APair<XM>& c, double (&acc)[2][6][2], double (&xacc)[XM][2]) {
    const double2* fb = reinterpret_cast<const double2*>(fbuf) + lane;
#pragma unroll
    for (int s = 0; s < 2; ++s) {
        const int ks = 2 * kp + s;
        const double2 b01 = fb[(ks * 3 + 0) * 32];
        const double2 b23 = fb[(ks * 3 + 1) * 32];
        const double2 b45 = fb[(ks * 3 + 2) * 32];
        const double bv[6] = {b01.x, b01.y, b23.x, b23.y, b45.x, b45.y};
        double bx[XM];
#pragma unroll
        for (int x = 0; x < XM; ++x) bx[x] = w.hx[x] ? fbuf[ks * 192 + w.xoff[x]] : 0.0;
        if (nmain > 0) {
            const double a0 = s ? c.m0.y : c.m0.x;
#pragma unroll
            for (int n = 0; n < 6; ++n) dmma(acc[0][n][0], acc[0][n][1], a0, bv[n]);
        }
        if (nmain > 1) {
            const double a1 = s ? c.m1.y : c.m1.x;
#pragma unroll
            for (int n = 0; n < 6; ++n) dmma(acc[1][n][0], acc[1][n][1], a1, bv[n]);
        }
#pragma unroll
        for (int x = 0; x < XM; ++x)
            if (w.hx[x]) dmma(xacc[x][0], xacc[x][1], s ? c.x[x].y : c.x[x].x, bx[x]);
    }
}

/// One warp's share of Y' = [U; anchor]·F: `main` full-width m-tiles (acc) and up to
/// XM extra tiles (xacc).  Operator pairs come from L2 as LDG.128, triple-buffered in
/// registers; B fragments are contiguous LDS.128 from the fragment-native Fbuf.
template <int XM>
__device__ __forceinline__ void warp_gemm(const double2* __restrict__ upack, int nkp, const double* fbuf,
                                          const GemmPlan& gp, int warp, int lane, APrefetch<XM> pre,
                                          double (&acc)[2][6][2], double (&xacc)[XM][2]) {
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int n = 0; n < 6; ++n) acc[i][n][0] = acc[i][n][1] = 0.0;
#pragma unroll
    for (int x = 0; x < XM; ++x) xacc[x][0] = xacc[x][1] = 0.0;
    const AWarp<XM> w = a_warp<XM>(upack, nkp, gp, warp, lane);
    const int nmain = gp.main;
    // three register buffers, two operator pairs in flight (L2 latency under full-chip
    // load exceeds one pair of DMMA issue time)
    APair<XM> p0 = pre.p, p1, p2;
    if (nkp > 1) load_apair<XM>(w, nmain, 1, p1);
    int kp = 0;
    for (; kp + 2 < nkp; kp += 3) {
        load_apair<XM>(w, nmain, kp + 2, p2);
        gemm_pair<XM>(fbuf, w, nmain, lane, kp, p0, acc, xacc);
        if (kp + 3 < nkp) load_apair<XM>(w, nmain, kp + 3, p0);
        gemm_pair<XM>(fbuf, w, nmain, lane, kp + 1, p1, acc, xacc);
        if (kp + 4 < nkp) load_apair<XM>(w, nmain, kp + 4, p1);
        gemm_pair<XM>(fbuf, w, nmain, lane, kp + 2, p2, acc, xacc);
    }
    if (kp < nkp) gemm_pair<XM>(fbuf, w, nmain, lane, kp, p0, acc, xacc);
    if (kp + 1 < nkp) gemm_pair<XM>(fbuf, w, nmain, lane, kp + 1, p1, acc, xacc);
}

}  // namespace pswarm_dev
