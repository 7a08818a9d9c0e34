// Batched independent verifier on the device: the reference's adaptive
// Fehlberg 7(8) oracle (oracle.hpp:63-132) sampled at the result's node epochs
// (oracle_sample_trajectory, oracle.hpp:136-150) and compared node by node
// (compare_trajectories, oracle.hpp:154-183), one thread per trajectory, so the CLI's
// --oracle-check (cli.hpp:238-261) scales to 1e5-1e6 trajectories.  The derivative is
// the continuous-time force (acceleration_at, force_model.hpp:78-87): body positions
// are evaluated at every stage epoch (conic solve / Clenshaw), not frozen per node, so
// it shares no numerics with the Picard-Chebyshev path.
#include <climits>

#include "pc_kernels.cuh"

namespace pswarm_dev {

namespace {

__constant__ double RK_C[13] = {0.0,       2.0 / 27.0, 1.0 / 9.0, 1.0 / 6.0, 5.0 / 12.0, 0.5, 5.0 / 6.0,
                                1.0 / 6.0, 2.0 / 3.0,  1.0 / 3.0, 1.0,       0.0,        1.0};
__constant__ double RK_A[13][12] = {
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
};
// eighth-order weights; the 7th-order defect is 41/840 (k0 + k10 - k11 - k12)
__constant__ double RK_B8[13] = {0.0,          0.0,         0.0,         0.0,         0.0,
                                 34.0 / 105.0, 9.0 / 35.0,  9.0 / 35.0,  9.0 / 280.0, 9.0 / 280.0,
                                 0.0,          41.0 / 840.0, 41.0 / 840.0};

constexpr int MAX_RK_BODIES = 16;

/// Position (and velocity) of body b at epoch t (ephemeris.hpp:58-73): CONIC_OK, or
/// 1 = not covered (CoverageError), CONIC_SOLVER.
__device__ int body_at(const BodyTable& bt, int b, double mu_c, double t, double p[3], double v[3], bool want_v) {
    double mf;
    if (bt.kind[b] == 0) {
        if (want_v) return elements_state(bt.elements + 7 * b, mu_c, t, p, v, &mf);
        return elements_position(bt.elements + 7 * b, mu_c, t, p, &mf);
    }
    for (int sg = bt.seg_off[b]; sg < bt.seg_off[b + 1]; ++sg) {
        const double t0 = bt.seg_bounds[2 * sg], t1 = bt.seg_bounds[2 * sg + 1];
        const bool fwd = t0 <= t1;
        if ((fwd && t >= t0 && t <= t1) || (!fwd && t <= t0 && t >= t1)) {
            const double tau = (2.0 * t - (t0 + t1)) / (t1 - t0);
            const int nc = bt.ncoef[b];
            const double* c = bt.coeffs + bt.coeff_off[sg];
            for (int k = 0; k < 3; ++k) p[k] = clenshaw(c + k * nc, nc, tau);
            if (want_v)
                for (int k = 0; k < 3; ++k) v[k] = (2.0 / (t1 - t0)) * clenshaw_deriv(c + k * nc, nc, tau);
            return CONIC_OK;
        }
    }
    return 1;
}

/// y' = [v, a(r, v, t)] with the reference's guards (force_model.hpp:26-52); fault codes:
/// 0 ok, 1 central zero radius, 2 + b close approach to body b, 100 + b ephemeris failure.
__device__ int rk_deriv(const RkArgs& a, double t, const double y[6], double dy[6]) {
    const double r[3] = {y[0], y[1], y[2]}, v[3] = {y[3], y[4], y[5]};
    const double rn = sqrt(r[0] * r[0] + r[1] * r[1] + r[2] * r[2]);
    if (!(rn > 0.0)) return 1;
    double acc[3];
    const double sc = -a.central_mu / (rn * rn * rn);
    for (int c = 0; c < 3; ++c) acc[c] = sc * r[c];
    const int B = a.bt.B;
    double pb[MAX_RK_BODIES][3], vb[MAX_RK_BODIES][3];
    for (int b = 0; b < B; ++b) {
        if (body_at(a.bt, b, a.central_mu, t, pb[b], vb[b], a.rel != 0) != CONIC_OK) return 100 + b;
        const double d[3] = {pb[b][0] - r[0], pb[b][1] - r[1], pb[b][2] - r[2]};
        const double dn = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
        if (dn < a.floor_km) return 2 + b;
        const double bn = sqrt(pb[b][0] * pb[b][0] + pb[b][1] * pb[b][1] + pb[b][2] * pb[b][2]);
        const double mu = a.bt.mu[b];
        for (int c = 0; c < 3; ++c) acc[c] += mu * (d[c] / (dn * dn * dn) - pb[b][c] / (bn * bn * bn));
    }
    if (a.rel) {  // EXTENSION: EIH 1PN, textbook two-pass form (oracle eih_correction)
        double ab[MAX_RK_BODIES][3], phi[MAX_RK_BODIES], phi_sun = 0.0;
        for (int b = 0; b < B; ++b) {
            const double rb = sqrt(pb[b][0] * pb[b][0] + pb[b][1] * pb[b][1] + pb[b][2] * pb[b][2]);
            phi_sun += a.bt.mu[b] / rb;
            const double k0 = -(a.central_mu + a.bt.mu[b]) / (rb * rb * rb);
            for (int c = 0; c < 3; ++c) ab[b][c] = k0 * pb[b][c];
            phi[b] = a.central_mu / rb;
            for (int k = 0; k < B; ++k) {
                if (k == b) continue;
                const double d[3] = {pb[k][0] - pb[b][0], pb[k][1] - pb[b][1], pb[k][2] - pb[b][2]};
                const double dn = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
                const double rk = sqrt(pb[k][0] * pb[k][0] + pb[k][1] * pb[k][1] + pb[k][2] * pb[k][2]);
                for (int c = 0; c < 3; ++c) ab[b][c] += a.bt.mu[k] * (d[c] / (dn * dn * dn) - pb[k][c] / (rk * rk * rk));
                phi[b] += a.bt.mu[k] / dn;
            }
        }
        const double c2 = a.c_light * a.c_light;
        double U = 0.0;
        for (int A = 0; A <= B; ++A) {
            const double* rA = A == 0 ? nullptr : pb[A - 1];
            const double dx = (A ? rA[0] : 0.0) - r[0], dy_ = (A ? rA[1] : 0.0) - r[1], dz = (A ? rA[2] : 0.0) - r[2];
            U += (A ? a.bt.mu[A - 1] : a.central_mu) / sqrt(dx * dx + dy_ * dy_ + dz * dz);
        }
        const double v2 = v[0] * v[0] + v[1] * v[1] + v[2] * v[2];
        for (int A = 0; A <= B; ++A) {
            double rA[3] = {0.0, 0.0, 0.0}, vA[3] = {0.0, 0.0, 0.0}, aA[3] = {0.0, 0.0, 0.0};
            double muA = a.central_mu, phiA = phi_sun;
            if (A > 0) {
                for (int c = 0; c < 3; ++c) {
                    rA[c] = pb[A - 1][c];
                    vA[c] = vb[A - 1][c];
                    aA[c] = ab[A - 1][c];
                }
                muA = a.bt.mu[A - 1];
                phiA = phi[A - 1];
            }
            const double d[3] = {rA[0] - r[0], rA[1] - r[1], rA[2] - r[2]};
            const double rho = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
            const double rho3 = rho * rho * rho;
            const double proj = -(d[0] * vA[0] + d[1] * vA[1] + d[2] * vA[2]) / rho;
            const double vA2 = vA[0] * vA[0] + vA[1] * vA[1] + vA[2] * vA[2];
            const double vvA = v[0] * vA[0] + v[1] * vA[1] + v[2] * vA[2];
            const double daA = d[0] * aA[0] + d[1] * aA[1] + d[2] * aA[2];
            const double br = -4.0 * U / c2 - phiA / c2 + v2 / c2 + 2.0 * vA2 / c2 - 4.0 * vvA / c2 -
                              1.5 * proj * proj / c2 + 0.5 * daA / c2;
            const double w = -(d[0] * (4.0 * v[0] - 3.0 * vA[0]) + d[1] * (4.0 * v[1] - 3.0 * vA[1]) +
                               d[2] * (4.0 * v[2] - 3.0 * vA[2]));
            for (int c = 0; c < 3; ++c)
                acc[c] += muA / rho3 * br * d[c] + muA / rho3 * w / c2 * (v[c] - vA[c]) + 3.5 * muA / rho / c2 * aA[c];
        }
    }
    for (int c = 0; c < 3; ++c) {
        dy[c] = v[c];
        dy[3 + c] = acc[c];
    }
    return 0;
}

/// rk_propagate (oracle.hpp:63-132) of y from t to t_end; returns 0, or a fault code
/// (rk_deriv codes, 200 step underflow, 201 step budget).
__device__ int rk_propagate_dev(const RkArgs& a, double& t, double y[6], double t_end, double (*k)[6]) {
    const double span = t_end - t;
    if (span == 0.0) return 0;
    const double dir = span > 0.0 ? 1.0 : -1.0;
    double h = span / 50.0;
    long long steps = 0;
    while (t != t_end) {
        bool last = false;
        if ((t + h - t_end) * dir >= 0.0) {
            h = t_end - t;
            last = true;
        }
        for (int i = 0; i < 13; ++i) {
            double yi[6];
            for (int q = 0; q < 6; ++q) yi[q] = y[q];
            for (int l = 0; l < i; ++l) {
                const double alk = RK_A[i][l];
                if (alk != 0.0) {
                    const double ha = h * alk;
                    for (int q = 0; q < 6; ++q) yi[q] += ha * k[l][q];
                }
            }
            const int f = rk_deriv(a, t + RK_C[i] * h, yi, k[i]);
            if (f) return f;
        }
        double y8[6];
        for (int q = 0; q < 6; ++q) y8[q] = y[q];
        for (int i = 0; i < 13; ++i)
            if (RK_B8[i] != 0.0) {
                const double hb = h * RK_B8[i];
                for (int q = 0; q < 6; ++q) y8[q] += hb * k[i][q];
            }
        double err = 0.0;
        const double hd = h * (41.0 / 840.0);
        for (int q = 0; q < 6; ++q) {
            const double defect = hd * (k[0][q] + k[10][q] - k[11][q] - k[12][q]);
            const double scale = a.abs_tol + a.rel_tol * fmax(fabs(y[q]), fabs(y8[q]));
            err = fmax(err, fabs(defect) / scale);
        }
        if (err <= 1.0) {
            for (int q = 0; q < 6; ++q) y[q] = y8[q];
            t = last ? t_end : t + h;
        }
        const double factor = (err > 0.0) ? fmin(fmax(0.9 * pow(err, -1.0 / 8.0), 0.2), 4.0) : 4.0;
        h *= factor;
        if (t + h == t) return 200;
        if (++steps > a.max_steps) return 201;
    }
    return 0;
}

__global__ void k_rk_check(RkArgs a) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= a.M) return;
    double k[13][6];
    double y[6];
    for (int q = 0; q < 6; ++q) y[q] = a.states[static_cast<size_t>(i) * 7 + 1 + q];
    double t = a.states[static_cast<size_t>(i) * 7];
    double worst = 0.0;
    int fault = 0, fault_node = 0;
    for (int j = 0; j < a.R; ++j) {
        if (j > 0) {
            fault = rk_propagate_dev(a, t, y, a.times[j], k);
            if (fault) {
                fault_node = j;
                break;
            }
        }
        const size_t o = (static_cast<size_t>(i) * a.R + j) * 6;
        if (a.samples_out)
            for (int q = 0; q < 6; ++q) a.samples_out[o + q] = y[q];
        if (a.candidate) {  // compare_trajectories: the RK reference normalises (oracle.hpp:154-183)
            const double* c = a.candidate + o;
            double dr2 = 0.0, dv2 = 0.0, rn2 = 0.0, vn2 = 0.0;
            for (int q = 0; q < 3; ++q) {
                dr2 += (c[q] - y[q]) * (c[q] - y[q]);
                dv2 += (c[3 + q] - y[3 + q]) * (c[3 + q] - y[3 + q]);
                rn2 += y[q] * y[q];
                vn2 += y[3 + q] * y[3 + q];
            }
            const double e = fmax(sqrt(dr2) / fmax(sqrt(rn2), 1e-30), sqrt(dv2) / fmax(sqrt(vn2), 1e-30));
            if (a.node_err) a.node_err[static_cast<size_t>(i) * a.R + j] = e;
            worst = fmax(worst, e);
        }
    }
    if (a.max_err) a.max_err[i] = worst;
    if (fault) {
        atomicMin(a.fault_key, static_cast<unsigned long long>(i) << 24 | static_cast<unsigned long long>(fault) << 16 |
                                   static_cast<unsigned long long>(fault_node & 0xffff));
        a.fault_t[i] = t;
    }
}

}  // namespace

cudaError_t launch_rk_check(const RkArgs& a, cudaStream_t s) {
    if (a.bt.B > MAX_RK_BODIES) return cudaErrorNotSupported;
    const int threads = 64;
    k_rk_check<<<(a.M + threads - 1) / threads, threads, 0, s>>>(a);
    return cudaGetLastError();
}

}  // namespace pswarm_dev
