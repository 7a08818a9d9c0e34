// Wide-group path: groups larger than the 8 trajectory slots of one CTA
// (RunMode::augmented_* with M > 8, grouped mode with big groups).
//
// A group converges only when the max error over ALL its members is <= tol
// (augment.hpp:106-109, picard.hpp:77), so the members of a wide group must
// iterate in lockstep across CTAs.  The state block of every trajectory stays in
// HBM between iterations ([tile][N][48] with the same swizzled layout as the
// slot kernel's shared-memory block); one launch of k_wide_iter advances every
// tile of every still-active group by one Picard iteration (force -> DMMA update
// -> error), and k_wide_finalize applies the stopping rule per group.  The host
// keeps at most two iterations in flight and stops launching when the device
// reports no active group (SURVEY.md §8a a9 loop control).
#include <climits>

#include "pc_kernels.cuh"
#include "pc_tile.cuh"

namespace pswarm_dev {

namespace {

struct WideSmem {
    double y0[SLOTS][6];
    double b0h[COLS];
    unsigned long long slot_err[SLOTS];
    int sing_key[SLOTS];
    int nf_key[SLOTS];
    int slot_group[SLOTS];
    int slot_member[SLOTS];
    int slot_size[SLOTS];
};

__host__ __device__ inline size_t wide_smem_bytes(int N, int nkp, int xrows) {
    return sizeof(double) * (static_cast<size_t>(N) * COLS + static_cast<size_t>(8 * nkp) * COLS +
                             static_cast<size_t>(xrows) * COLS) +
           sizeof(WideSmem);
}

}  // namespace

size_t wide_iter_smem_bytes(int N, int nkp, int xrows) { return wide_smem_bytes(N, nkp, xrows); }

/// Warm (conic) or cold start of every trajectory into the HBM state blocks.
__global__ void k_wide_start(WideArgs a) {
    const long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= static_cast<long long>(a.M) * a.N) return;
    const int tr = static_cast<int>(idx / a.N), j = static_cast<int>(idx % a.N);
    const double* s = a.state_in + static_cast<size_t>(tr) * 6;
    const double r[3] = {s[0], s[1], s[2]}, v[3] = {s[3], s[4], s[5]};
    double ro[3] = {r[0], r[1], r[2]}, vo[3] = {v[0], v[1], v[2]};
    if (!a.cold_start) {
        const int chk = conic_check(r, v, a.fd.central_mu);
        if (chk == CONIC_ZERO_RADIUS) {
            atomicMin(a.warm_key, static_cast<unsigned long long>(tr) * 4ull + CONIC_ZERO_RADIUS);
        } else if (chk == CONIC_OK) {
            double mf, ef;
            if (kepler_propagate(r, v, a.fd.central_mu, a.times[j] - a.epoch, ro, vo, &mf, &ef) != CONIC_OK)
                atomicMin(a.warm_key, static_cast<unsigned long long>(tr) * 4ull + CONIC_SOLVER);
        }
        if (j == 0 && a.cold_fallback) a.cold_fallback[tr] = chk == CONIC_NON_ELLIPTIC ? 1 : 0;
    }
    if (a.hot) hot_start_node(a.hot + (static_cast<size_t>(tr) * a.N + j) * 6, a.hot_apply, ro, vo);
    double* y = a.Y + static_cast<size_t>(tr >> 3) * a.N * COLS;
    const int t = tr & 7;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        y[yidx(j, c, t)] = ro[c];
        y[yidx(j, c + 3, t)] = vo[c];
    }
}

/// One Picard iteration of every tile whose slots belong to active groups.
template <int MAXT, int XM, bool REL>
__global__ void __launch_bounds__(MAXT, 1) k_wide_iter(WideArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int N = a.N, B = a.fd.n_bodies;
    const GemmPlan gp = a.gp;
    double* ybuf = reinterpret_cast<double*>(smem_raw);
    double* fbuf = ybuf + static_cast<size_t>(N) * COLS;
    double* xstage = fbuf + static_cast<size_t>(8 * a.nkp) * COLS;
    WideSmem& ws = *reinterpret_cast<WideSmem*>(xstage + static_cast<size_t>(a.xrows) * COLS);
    const int tid = threadIdx.x, nthr = blockDim.x, warp = tid >> 5, lane = tid & 31;
    const int g = lane >> 2, q = lane & 3;
    const int tiles = (a.M + SLOTS - 1) / SLOTS;
    const int KP = 8 * a.nkp;
    for (int i = tid; i < KP * COLS; i += nthr) fbuf[i] = 0.0;

    for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
        __syncthreads();
        if (tid < SLOTS) {
            const int tr = tile * SLOTS + tid;
            int grp = -1;
            if (tr < a.M) {
                grp = a.traj_group[tr];
                if (!a.g_active[grp]) grp = -1;
            }
            ws.slot_group[tid] = grp;
            ws.slot_member[tid] = grp >= 0 ? tr - static_cast<int>(a.group_off[grp]) : 0;
            ws.slot_size[tid] = grp >= 0 ? static_cast<int>(a.group_off[grp + 1] - a.group_off[grp]) : 1;
            ws.slot_err[tid] = 0ull;
            ws.sing_key[tid] = INT_MAX;
            ws.nf_key[tid] = INT_MAX;
        }
        __syncthreads();
        int act = 0;
#pragma unroll
        for (int t = 0; t < SLOTS; ++t) act |= (ws.slot_group[t] >= 0) << t;
        if (act == 0) continue;
        const double* ysrc = a.Y + static_cast<size_t>(tile) * N * COLS;
        for (int i = tid; i < N * COLS / 2; i += nthr)
            reinterpret_cast<double2*>(ybuf)[i] = reinterpret_cast<const double2*>(ysrc)[i];
        for (int i = tid; i < SLOTS * 6; i += nthr) {
            const int s = i / 6, c = i % 6, tr = tile * SLOTS + s;
            ws.y0[s][c] = tr < a.M ? a.state_in[static_cast<size_t>(tr) * 6 + c] : 0.0;
        }
        __syncthreads();

        // force -> Fbuf (same tile routine as the slot kernel)
        {
            constexpr int FS = 4;
            const int items = N * (SLOTS / FS);
            const int extra = items > nthr ? (items - nthr) * FS : 0;
            for (int it0 = tid; it0 < (items > nthr ? nthr : items); it0 += nthr) {
                const int jq = it0 / (SLOTS / FS), t0 = (it0 % (SLOTS / FS)) * FS;
                if (tid < extra) {
                    const int sx = nthr * FS + tid;
                    force_chains<FS, true, REL>(a.fd, a.omega2, ybuf, fbuf, ws.sing_key, a.fd.body_pos, a.fd.indirect, act,
                                           jq, t0, sx >> 3, sx & 7);
                } else {
                    force_chains<FS, false, REL>(a.fd, a.omega2, ybuf, fbuf, ws.sing_key, a.fd.body_pos, a.fd.indirect, act,
                                            jq, t0, 0, 0);
                }
            }
        }
        const APrefetch<XM> pre = gemm_prefetch<XM>(a.upack, a.nkp, gp, warp, lane);
        __syncthreads();
        if (tid < SLOTS && ws.sing_key[tid] != INT_MAX) {  // rare: record the failing sample
            const int t = tid, key = ws.sing_key[t], j = key / (B + 1), chk = key % (B + 1);
            const int tr = tile * SLOTS + t, size = ws.slot_size[t], mbr = ws.slot_member[t];
            const unsigned long long gkey =
                ((static_cast<unsigned long long>(j) * size + mbr) << 6) | static_cast<unsigned long long>(chk);
            a.t_sing_key[tr] = gkey;
            a.t_sing_val[tr] = check_distance(ybuf[yidx(j, 0, t)], ybuf[yidx(j, 1, t)], ybuf[yidx(j, 2, t)], j, chk, a.fd);
            atomicMin(a.g_sing + ws.slot_group[t], gkey);
        }

        double acc[2][6][2], xacc[XM][2];
        warp_gemm<XM>(a.upack, a.nkp, fbuf, gp, warp, lane, pre, acc, xacc);
        {
            const int amt = N >> 3;
            if (g == (N & 7)) {
#pragma unroll
                for (int i = 0; i < 2; ++i)
                    if (i < gp.main && warp * gp.main + i == amt)
#pragma unroll
                        for (int c = 0; c < 6; ++c)
#pragma unroll
                            for (int h = 0; h < 2; ++h) {
                                const int t = 2 * q + h;
                                const double an = i ? acc[1][c][h] : acc[0][c][h];
                                ws.b0h[c * 8 + t] = 0.5 * (an + 2.0 * ws.y0[t][c]);
                            }
#pragma unroll
                for (int x = 0; x < XM; ++x) {
                    const int e = warp + x * gp.warps;
                    if (e < gp.extras && gp.mb + e / 6 == amt)
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            const int t = 2 * q + h, c = e % 6;
                            ws.b0h[c * 8 + t] = 0.5 * (xacc[x][h] + 2.0 * ws.y0[t][c]);
                        }
                }
            }
        }
        __syncthreads();
        {  // epilogue: main rows
            double bn[2] = {0.0, 0.0}, bd[2] = {1.0, 1.0};
            int nf[2] = {INT_MAX, INT_MAX};
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                if (i >= gp.main) continue;
                const int j = (warp * gp.main + i) * 8 + g;
                if (j >= N) continue;
                double yn[2][6], yo[2][6];
#pragma unroll
                for (int c = 0; c < 6; ++c) {
                    const double2 prev = *reinterpret_cast<const double2*>(ybuf + yidx(j, c, 2 * q));
                    yo[0][c] = prev.x;
                    yo[1][c] = prev.y;
                    yn[0][c] = acc[i][c][0] + ws.b0h[c * 8 + 2 * q];
                    yn[1][c] = acc[i][c][1] + ws.b0h[c * 8 + 2 * q + 1];
                }
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    if (!((act >> (2 * q + h)) & 1)) {
#pragma unroll
                        for (int c = 0; c < 6; ++c) yn[h][c] = yo[h][c];
                        continue;
                    }
                    update_sample(yn[h], yo[h], j, a.error_mode, bn[h], bd[h], nf[h]);
                }
#pragma unroll
                for (int c = 0; c < 6; ++c)
                    *reinterpret_cast<double2*>(ybuf + yidx(j, c, 2 * q)) = make_double2(yn[0][c], yn[1][c]);
            }
#pragma unroll
            for (int x = 0; x < XM; ++x) {
                const int e = warp + x * gp.warps;
                if (e >= gp.extras) continue;
                const int j = (gp.mb + e / 6) * 8 + g, c = e % 6;
                if (j >= N) continue;
#pragma unroll
                for (int h = 0; h < 2; ++h)
                    xstage[(j - gp.mb * 8) * COLS + c * 8 + 2 * q + h] = xacc[x][h] + ws.b0h[c * 8 + 2 * q + h];
            }
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                double e2 = bn[h] / bd[h];
#pragma unroll
                for (int off = 4; off < 32; off <<= 1) {
                    e2 = fmax(e2, __shfl_xor_sync(0xffffffffu, e2, off));
                    nf[h] = min(nf[h], __shfl_xor_sync(0xffffffffu, nf[h], off));
                }
                const int t = 2 * q + h;
                if (g == 0 && gp.main > 0 && ((act >> t) & 1)) {
                    atomicMax(&ws.slot_err[t], static_cast<unsigned long long>(__double_as_longlong(e2)));
                    if (nf[h] != INT_MAX) atomicMin(&ws.nf_key[t], nf[h]);
                }
            }
        }
        __syncthreads();
        // every staged row (up to 31 x 8 items on the 128-thread small-N plan)
        for (int i = tid; i < a.xrows * SLOTS; i += blockDim.x) {  // epilogue: staged rows
            const int r = i >> 3, t = i & 7, j = gp.mb * 8 + r;
            if ((act >> t) & 1) {
                double yn[6], yo[6];
#pragma unroll
                for (int c = 0; c < 6; ++c) {
                    yn[c] = xstage[r * COLS + c * 8 + t];
                    yo[c] = ybuf[yidx(j, c, t)];
                }
                double bn = 0.0, bd = 1.0;
                int nf = INT_MAX;
                update_sample(yn, yo, j, a.error_mode, bn, bd, nf);
#pragma unroll
                for (int c = 0; c < 6; ++c) ybuf[yidx(j, c, t)] = yn[c];
                atomicMax(&ws.slot_err[t], static_cast<unsigned long long>(__double_as_longlong(bn / bd)));
                if (nf != INT_MAX) atomicMin(&ws.nf_key[t], nf);
            }
        }
        __syncthreads();
        // publish: per-group max error and first non-finite (node, column); write Y' back
        if (tid < SLOTS && ((act >> tid) & 1)) {
            const int t = tid, grp = ws.slot_group[t];
            atomicMax(a.g_err2 + grp, ws.slot_err[t]);
            if (ws.nf_key[t] != INT_MAX) {
                const unsigned long long size = ws.slot_size[t], mbr = ws.slot_member[t];
                const unsigned long long key = static_cast<unsigned long long>(ws.nf_key[t] >> 3) * 6ull * size +
                                               static_cast<unsigned long long>(ws.nf_key[t] & 7) * size + mbr;
                atomicMin(a.g_nf + grp, key);
            }
        }
        double* ydst = a.Y + static_cast<size_t>(tile) * N * COLS;
        for (int i = tid; i < N * COLS / 2; i += nthr)
            reinterpret_cast<double2*>(ydst)[i] = reinterpret_cast<const double2*>(ybuf)[i];
    }
}

/// Stopping rule per group (picard.hpp:66-81) after one k_wide_iter launch.
__global__ void k_wide_finalize(WideArgs a) {
    const int gid = blockIdx.x * blockDim.x + threadIdx.x;
    if (gid >= a.P || !a.g_active[gid]) return;
    const int it = ++a.g_iter[gid];
    GroupFault* fl = a.faults + gid;
    bool retire = false, conv = false;
    const double gerr = sqrt(__longlong_as_double(static_cast<long long>(a.g_err2[gid])));
    if (a.g_sing[gid] != ~0ull) {
        const unsigned long long key = a.g_sing[gid];
        const long long size = a.group_off[gid + 1] - a.group_off[gid];
        const long long smp = static_cast<long long>(key >> 6);
        fl->status = FAULT_SINGULARITY;
        fl->iteration = it;
        fl->node = smp / size;
        fl->trajectory = smp % size;
        fl->body = static_cast<int>(key & 63) - 1;
        fl->value = a.t_sing_val[a.group_off[gid] + smp % size];
        retire = true;
    } else if (a.g_nf[gid] != ~0ull) {
        const long long size = a.group_off[gid + 1] - a.group_off[gid];
        fl->status = FAULT_DIVERGENCE;
        fl->iteration = it;
        fl->node = static_cast<long long>(a.g_nf[gid] / (6ull * size));
        fl->column = static_cast<long long>(a.g_nf[gid] % (6ull * size));
        retire = true;
    } else {
        if (a.rep_hist) a.rep_hist[static_cast<size_t>(gid) * a.max_it + (it - 1)] = gerr;
        if (gerr <= a.tol) retire = conv = true;
        else if (it >= a.max_it) retire = true;
    }
    a.rep_iter[gid] = it;
    a.rep_err[gid] = gerr;
    a.rep_conv[gid] = conv ? 1 : 0;
    a.g_err2[gid] = 0ull;
    a.g_nf[gid] = ~0ull;
    a.g_sing[gid] = ~0ull;
    if (retire) a.g_active[gid] = 0;
    else atomicAdd(a.active_count, 1);
}

/// Terminal rows (chaining) and node samples of every trajectory after the loop.
__global__ void k_wide_output(WideArgs a) {
    const long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= static_cast<long long>(a.M) * a.N) return;
    const int tr = static_cast<int>(idx / a.N), j = static_cast<int>(idx % a.N);
    const double* y = a.Y + static_cast<size_t>(tr >> 3) * a.N * COLS;
    const int t = tr & 7;
    if (a.samples && j >= (a.seg == 0 ? 0 : 1)) {
        double* o = a.samples + (static_cast<size_t>(tr) * a.R + a.row0 + j) * 6;
#pragma unroll
        for (int c = 0; c < 6; ++c) o[c] = y[yidx(j, c, t)];
    }
    if (j == a.N - 1) {
#pragma unroll
        for (int c = 0; c < 6; ++c) a.state_out[static_cast<size_t>(tr) * 6 + c] = y[yidx(j, c, t)];
    }
    if (a.hot)
        for (int c = 0; c < 6; ++c)
            hot_retire_node(a.hot + (static_cast<size_t>(tr) * a.N + j) * 6, c, y[yidx(j, c, t)]);
}

cudaError_t launch_wide_start(const WideArgs& a, cudaStream_t s) {
    const long long n = static_cast<long long>(a.M) * a.N;
    k_wide_start<<<static_cast<unsigned>((n + 127) / 128), 128, 0, s>>>(a);
    return cudaGetLastError();
}

template <int MAXT, int XM>
static cudaError_t launch_wide_iter_t(const WideArgs& a, int grid, size_t smem, cudaStream_t s) {
    auto kern = a.fd.rel ? k_wide_iter<MAXT, XM, true> : k_wide_iter<MAXT, XM, false>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    kern<<<grid, 32 * a.gp.warps, smem, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_wide_iter(const WideArgs& a, int grid, cudaStream_t s) {
    const size_t smem = wide_smem_bytes(a.N, a.nkp, a.xrows);
    if (a.gp.xmax == XMAX_SMALL) return launch_wide_iter_t<128, XMAX_SMALL>(a, grid, smem, s);
    if (a.gp.warps <= 12) return launch_wide_iter_t<384, XMAX>(a, grid, smem, s);
    return launch_wide_iter_t<512, XMAX>(a, grid, smem, s);
}

cudaError_t launch_wide_finalize(const WideArgs& a, cudaStream_t s) {
    k_wide_finalize<<<(a.P + 127) / 128, 128, 0, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_wide_output(const WideArgs& a, cudaStream_t s) {
    const long long n = static_cast<long long>(a.M) * a.N;
    k_wide_output<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(a);
    return cudaGetLastError();
}

}  // namespace pswarm_dev
