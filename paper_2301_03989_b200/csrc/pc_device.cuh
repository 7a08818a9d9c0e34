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
//   Ybuf  smem  [node j][component c][slot t], row stride YS doubles (bank-conflict-free
//               double2 epilogue stores);
//   Fbuf  smem  fragment-native B operand: [kstep][ntile pair][lane][2] doubles, so every
//               B-fragment fetch of a warp is one contiguous 512-byte LDS.128;
//   Upack gmem  fragment-native A operand: [mtile][kstep pair][lane] double2 (LDG.128).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace pswarm_dev {

constexpr int SLOTS = 8;             // trajectories per CTA tile
constexpr int COLS = 6 * SLOTS;      // 48 block columns: column = comp*8 + slot
constexpr int YS = 56;               // Ybuf row stride in doubles (48 + 8 pad)
constexpr double PI = 3.141592653589793238462643383279502884;

// ---------------------------------------------------------------- DMMA ---
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
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
    int n_bodies;      // 0 for two-body
};

/// Acceleration at node j (force_model.hpp:57-69).  Returns -1 when finite and legal,
/// else the index of the first failing check in reference order: 0 = central body
/// (|r| not > 0, force_model.hpp:28), 1 + b = body b closer than the floor (:44).
__device__ __forceinline__ int accel(double rx, double ry, double rz, int j, const ForceData& fd, double& ax,
                                     double& ay, double& az) {
    const double r2 = rx * rx + ry * ry + rz * rz;
    if (!(r2 > 0.0)) return 0;
    const double ir = rsqrt(r2);
    const double s = -fd.central_mu * (ir * ir * ir);
    ax = s * rx;
    ay = s * ry;
    az = s * rz;
    const int B = fd.n_bodies;
    if (B > 0) {
        const double* bp = fd.body_pos + static_cast<size_t>(j) * B * 3;
        for (int b = 0; b < B; ++b) {
            const double dx = __ldg(bp + 3 * b + 0) - rx;
            const double dy = __ldg(bp + 3 * b + 1) - ry;
            const double dz = __ldg(bp + 3 * b + 2) - rz;
            const double d2 = dx * dx + dy * dy + dz * dz;
            if (d2 < fd.floor2_hi && sqrt(d2) < fd.floor_km) return 1 + b;
            const double id = rsqrt(d2);
            const double k = __ldg(fd.body_mu + b) * (id * id * id);
            ax += k * dx;
            ay += k * dy;
            az += k * dz;
        }
        const double* ind = fd.indirect + 3 * j;
        ax -= __ldg(ind + 0);
        ay -= __ldg(ind + 1);
        az -= __ldg(ind + 2);
    }
    return -1;
}

/// Distance behind a failing check (for the SingularityError message, force_model.hpp:44-49).
__device__ __forceinline__ double check_distance(double rx, double ry, double rz, int j, int check,
                                                 const ForceData& fd) {
    if (check <= 0) return sqrt(rx * rx + ry * ry + rz * rz);
    const double* bp = fd.body_pos + (static_cast<size_t>(j) * fd.n_bodies + (check - 1)) * 3;
    const double dx = bp[0] - rx, dy = bp[1] - ry, dz = bp[2] - rz;
    return sqrt(dx * dx + dy * dy + dz * dz);
}

// ----------------------------------------------------------- tile GEMM ---
/// Fragment-native index of B element (k, n) in Fbuf (doubles): B fragment of
/// mma.m8n8k4 holds B[k = lane%4][n = lane/4]; two n-tiles share one double2.
__device__ __forceinline__ int fbuf_index(int k, int n) {
    const int ks = k >> 2, kk = k & 3, nt = n >> 3, nn = n & 7;
    return (((ks * 3 + (nt >> 1)) * 32) + (nn * 4 + kk)) * 2 + (nt & 1);
}

/// One warp's share of Y' = U'·F: m-tiles 2w and 2w+1 (16 rows) × 48 columns.
/// Operator pairs (two k-steps) arrive as one LDG.128 per m-tile from L2 with a
/// two-deep register prefetch; B fragments are LDS.128 from the fragment-native Fbuf.
__device__ __forceinline__ void warp_gemm(const double2* __restrict__ upack, int nkp, const double* fbuf,
                                          int warp, int lane, double (&acc)[2][6][2]) {
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int n = 0; n < 6; ++n) acc[i][n][0] = acc[i][n][1] = 0.0;
    const double2* a0 = upack + static_cast<size_t>(2 * warp) * nkp * 32 + lane;
    const double2* a1 = a0 + static_cast<size_t>(nkp) * 32;
    const double2* fb = reinterpret_cast<const double2*>(fbuf) + lane;
    double2 p0 = __ldg(a0), p1 = __ldg(a1);
    double2 q0 = p0, q1 = p1;
    if (nkp > 1) {
        q0 = __ldg(a0 + 32);
        q1 = __ldg(a1 + 32);
    }
    for (int kp = 0; kp < nkp; ++kp) {
        const double2 c0 = p0, c1 = p1;
        p0 = q0;
        p1 = q1;
        if (kp + 2 < nkp) {
            q0 = __ldg(a0 + (kp + 2) * 32);
            q1 = __ldg(a1 + (kp + 2) * 32);
        }
#pragma unroll
        for (int s = 0; s < 2; ++s) {
            const int ks = 2 * kp + s;
            const double2 b01 = fb[(ks * 3 + 0) * 32];
            const double2 b23 = fb[(ks * 3 + 1) * 32];
            const double2 b45 = fb[(ks * 3 + 2) * 32];
            const double bv[6] = {b01.x, b01.y, b23.x, b23.y, b45.x, b45.y};
            const double av0 = s ? c0.y : c0.x;
            const double av1 = s ? c1.y : c1.x;
#pragma unroll
            for (int n = 0; n < 6; ++n) {
                dmma(acc[0][n][0], acc[0][n][1], av0, bv[n]);
                dmma(acc[1][n][0], acc[1][n][1], av1, bv[n]);
            }
        }
    }
}

}  // namespace pswarm_dev
