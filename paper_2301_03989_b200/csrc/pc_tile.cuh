// Tile-level device routines shared by the persistent slot kernel (pc_kernels.cu)
// (groups wider than a CTA run on the same kernels in member-level rounds).
#pragma once

#include <climits>

#include "pc_device.cuh"

namespace pswarm_dev {

/// Per-sample finite check (picard.hpp:26-36) and convergence error of one (node, slot)
/// against the previous iterate (augment.hpp:38-51, component_error of
/// error_metric.hpp:15-23).  The squared ratio max(|dr|^2/|r|^2, |dv|^2/|v|^2) is kept as
/// a (numerator, denominator) pair and maximised by cross-multiplication, so a lane
/// pays one division for all its samples; max commutes with the final sqrt.
__device__ __forceinline__ void update_sample(const double (&yn)[6], const double (&yo)[6], int j, int error_mode,
                                              double& bn, double& bd, int& nf) {
#pragma unroll
    for (int c = 5; c >= 0; --c)  // finite <=> exponent field != 0x7ff: integer test, off the FP64 pipe
        if ((__double2hiint(yn[c]) & 0x7ff00000) == 0x7ff00000) nf = min(nf, j * 8 + c);
    double dr2 = 0.0, r2 = 0.0, dv2 = 0.0, v2 = 0.0;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        const double dr = yn[c] - yo[c], dv = yn[c + 3] - yo[c + 3];
        dr2 += dr * dr;
        r2 += yo[c] * yo[c];
        dv2 += dv * dv;
        v2 += yo[c + 3] * yo[c + 3];
    }
    if (error_mode == 1) {
        r2 = 1.0;
        v2 = 1.0;
    } else {
        r2 = fmax(r2, 1e-60);
        v2 = fmax(v2, 1e-60);
    }
    if (dr2 * bd > bn * r2) {
        bn = dr2;
        bd = r2;
    }
    if (dv2 * bd > bn * v2) {
        bn = dv2;
        bd = v2;
    }
}

/// Force for FS slots of node jq (+ optionally one extra sample (jx, tx)) as
/// independent chains: a = -mu r/|r|^3 + sum_b mu_b (d_b/|d_b|^3) - indirect(j),
/// F = omega2 [v; a] written in MMA B-fragment order (force_model.hpp:93-142).
/// Singularity guards run exactly, in reference order, on a rare slow path.
template <int FS, bool X, bool REL = false>
__device__ __forceinline__ void force_chains(const ForceData& fd, double w2, const double* ybuf, double* fbuf,
                                             int* sing_key, const double* pos_base, const double* ind_base, int act,
                                             int jq, int t0, int jx, int tx) {
    constexpr int K = FS + (X ? 1 : 0);
    const int B = fd.n_bodies;
    int jj[K], tt[K];
    double rx[K], ry[K], rz[K], ax[K], ay[K], az[K];
    bool on[K];
    bool flag = false;
    double r2[K], ir[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
        jj[k] = k < FS ? jq : jx;
        tt[k] = k < FS ? t0 + k : tx;
        on[k] = (act >> tt[k]) & 1;
        rx[k] = on[k] ? ybuf[yidx(jj[k], 0, tt[k])] : 1.0e8;  // benign stand-in keeps idle slots finite
        ry[k] = on[k] ? ybuf[yidx(jj[k], 1, tt[k])] : 0.0;
        rz[k] = on[k] ? ybuf[yidx(jj[k], 2, tt[k])] : 0.0;
    }
#pragma unroll
    for (int k = 0; k < K; ++k) {
        r2[k] = rx[k] * rx[k] + ry[k] * ry[k] + rz[k] * rz[k];
        flag |= !(r2[k] > 0.0);
    }
#pragma unroll
    for (int k = 0; k < K; ++k) ir[k] = rsqrt_seed(r2[k]);
#pragma unroll
    for (int k = 0; k < K; ++k) ir[k] = rsqrt_newton(r2[k], rsqrt_newton(r2[k], ir[k]));  // central: full precision
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const double sc = -fd.central_mu * (ir[k] * ir[k] * ir[k]);
        ax[k] = sc * rx[k];
        ay[k] = sc * ry[k];
        az[k] = sc * rz[k];
    }
    const double* bq = pos_base + static_cast<size_t>(jq) * 3 * B;
    const double* bx_ = pos_base + static_cast<size_t>(jx) * 3 * B;
    for (int b = 0; b < B; ++b) {
        const double mu_b = __ldg(fd.body_mu + b);
        const double qx = bq[3 * b], qy = bq[3 * b + 1], qz = bq[3 * b + 2];
        double ex = 0.0, ey = 0.0, ez = 0.0;
        if (X) {
            ex = bx_[3 * b];
            ey = bx_[3 * b + 1];
            ez = bx_[3 * b + 2];
        }
        // stage-by-stage over the chains so their dependency chains interleave
        double dx[K], dy[K], dz[K], d2[K], y[K];
#pragma unroll
        for (int k = 0; k < K; ++k) {
            dx[k] = (k < FS ? qx : ex) - rx[k];
            dy[k] = (k < FS ? qy : ey) - ry[k];
            dz[k] = (k < FS ? qz : ez) - rz[k];
        }
#pragma unroll
        for (int k = 0; k < K; ++k) {
            d2[k] = dx[k] * dx[k] + dy[k] * dy[k] + dz[k] * dz[k];
            flag |= d2[k] < fd.floor2_hi;
        }
#pragma unroll
        for (int k = 0; k < K; ++k) y[k] = rsqrt_seed(d2[k]);
        // one Newton step (rel. error ~1e-14 on a perturbation that is <1e-3 of the
        // central term, i.e. far below the FP64 resolution of the total acceleration)
#pragma unroll
        for (int k = 0; k < K; ++k) y[k] = rsqrt_newton(d2[k], y[k]);
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const double kk = mu_b * (y[k] * y[k] * y[k]);
            ax[k] += kk * dx[k];
            ay[k] += kk * dy[k];
            az[k] += kk * dz[k];
        }
    }
    if (B > 0) {
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const double* ind = ind_base + 3 * jj[k];
            ax[k] -= ind[0];
            ay[k] -= ind[1];
            az[k] -= ind[2];
        }
    }
    if (REL) {  // EXTENSION: EIH 1PN correction (n_body_1pn)
        for (int k = 0; k < K; ++k) {
            if (!on[k]) continue;
            double o[3];
            rel_correction(rx[k], ry[k], rz[k], ybuf[yidx(jj[k], 3, tt[k])], ybuf[yidx(jj[k], 4, tt[k])],
                           ybuf[yidx(jj[k], 5, tt[k])], fd.rel_tab + static_cast<size_t>(jj[k]) * rel_stride(B),
                           B + 1, fd.ic2, o);
            ax[k] += o[0];
            ay[k] += o[1];
            az[k] += o[2];
        }
    }
    if (flag) {  // rare: exact guard order of table_acceleration (force_model.hpp:57-69)
#pragma unroll
        for (int k = 0; k < K; ++k) {
            if (!on[k]) continue;
            int fail = (rx[k] * rx[k] + ry[k] * ry[k] + rz[k] * rz[k] > 0.0) ? -1 : 0;
            const double* bp = pos_base + static_cast<size_t>(jj[k]) * 3 * B;
            for (int b = 0; b < B && fail < 0; ++b) {
                const double dx = bp[3 * b] - rx[k], dy = bp[3 * b + 1] - ry[k], dz = bp[3 * b + 2] - rz[k];
                if (sqrt(dx * dx + dy * dy + dz * dz) < fd.floor_km) fail = 1 + b;
            }
            if (fail >= 0) atomicMin(&sing_key[tt[k]], jj[k] * (B + 1) + fail);
        }
    }
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const int j = jj[k], t = tt[k];
        fbuf[fbuf_index(j, 0 * 8 + t)] = on[k] ? w2 * ybuf[yidx(j, 3, t)] : 0.0;
        fbuf[fbuf_index(j, 1 * 8 + t)] = on[k] ? w2 * ybuf[yidx(j, 4, t)] : 0.0;
        fbuf[fbuf_index(j, 2 * 8 + t)] = on[k] ? w2 * ybuf[yidx(j, 5, t)] : 0.0;
        fbuf[fbuf_index(j, 3 * 8 + t)] = on[k] ? w2 * ax[k] : 0.0;
        fbuf[fbuf_index(j, 4 * 8 + t)] = on[k] ? w2 * ay[k] : 0.0;
        fbuf[fbuf_index(j, 5 * 8 + t)] = on[k] ? w2 * az[k] : 0.0;
    }
}

}  // namespace pswarm_dev
