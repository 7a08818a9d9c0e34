// CUDA kernels of the B200-native augmented Picard–Chebyshev propagator (sm_100a).
//
// k_pc_segment   persistent slot kernel: one CTA per SM owns SLOTS = 8 trajectory
//                slots and runs the WHOLE fixed-point loop of pc_solve
//                (picard.hpp:46-83) for every group it claims, with the state block
//                resident in shared memory across iterations:
//                  warm start (kepler.hpp:59-98) -> [force (force_model.hpp:93-142)
//                  -> DMMA update (pc_matrices.hpp:123-151) -> finite check
//                  (picard.hpp:69-71) -> convergence error (augment.hpp:32-77)
//                  -> group decision (picard.hpp:73-79)]*  -> retire + refill.
//                Converged groups leave the CTA immediately and their slots are
//                refilled from a global work queue, so converged trajectories are
//                masked out of further iterations without wasting tensor-core work.
// k_picard_update / k_force_block / k_block_error / k_warm_start
//                standalone operator kernels behind the operator-level C-ABI
//                (per-kernel parity against the oracle).
#include <climits>

#include "pc_kernels.cuh"

namespace pswarm_dev {

namespace {

struct CtaState {
    int slot_traj[SLOTS];      // batch index, -1 = free
    int slot_grp[SLOTS];       // local group index
    int slot_member[SLOTS];    // member index within its group
    int sing_key[SLOTS];       // min j*(B+1)+check this tick
    int nf_key[SLOTS];         // min j*8+c non-finite this tick
    int warm_key[SLOTS];       // min node with a warm-start fault
    int warm_kind[SLOTS];
    unsigned long long slot_err[SLOTS];
    double sing_val[SLOTS];
    double warm_val[SLOTS][2];
    double y0[SLOTS][6];
    double b0h[COLS];
    int grp_id[SLOTS];         // global group id, -1 = free
    int grp_size[SLOTS];
    int grp_iter[SLOTS];
    int active_mask;
    int new_mask;
    int retire_mask;           // slots whose results are written out this tick
    int free_mask;             // slots released this tick (retired or failed)
    int queue_done;
    int timeout;
};

__device__ __forceinline__ int popc(int x) { return __popc(static_cast<unsigned>(x)); }

}  // namespace

size_t segment_smem_bytes(int N, int nkp) {
    return sizeof(double) * (static_cast<size_t>(N) * YS + static_cast<size_t>(8 * nkp) * COLS) + sizeof(CtaState);
}

int segment_threads(int N) {
    const int mt = (N + 1 + 7) / 8;
    return 32 * ((mt + 1) / 2);
}

template <int MAXT>
__global__ void __launch_bounds__(MAXT, 1) k_pc_segment(const SegArgs a) {
    extern __shared__ __align__(16) double smem[];
    const int N = a.N;
    double* ybuf = smem;
    double* fbuf = ybuf + static_cast<size_t>(N) * YS;
    const int KP = 8 * a.nkp;
    CtaState& st = *reinterpret_cast<CtaState*>(fbuf + static_cast<size_t>(KP) * COLS);
    const int tid = threadIdx.x, nthr = blockDim.x, warp = tid >> 5, lane = tid & 31;
    const int B = a.fd.n_bodies;

    for (int i = tid; i < KP * COLS; i += nthr) fbuf[i] = 0.0;
    if (tid == 0) {
        for (int t = 0; t < SLOTS; ++t) {
            st.slot_traj[t] = -1;
            st.grp_id[t] = -1;
        }
        st.active_mask = 0;
        st.queue_done = 0;
        st.timeout = 0;
    }
    __syncthreads();

    for (;;) {
        // ------------------------------------------------ claim + bookkeeping
        if (tid == 0) {
            st.new_mask = 0;
            int free_slots = SLOTS - popc(st.active_mask);
            if (!st.queue_done && free_slots >= a.gmax) {
                const int k = free_slots / a.gmax;
                const int g0 = atomicAdd(a.queue, k);
                const int g1 = min(g0 + k, a.P);
                if (g0 + k >= a.P) st.queue_done = 1;
                for (int g = g0; g < g1; ++g) {
                    int lg = 0;
                    while (st.grp_id[lg] >= 0) ++lg;
                    const int off = static_cast<int>(a.group_off[g]);
                    const int size = static_cast<int>(a.group_off[g + 1]) - off;
                    st.grp_id[lg] = g;
                    st.grp_size[lg] = size;
                    st.grp_iter[lg] = 0;
                    int t = 0;
                    for (int mbr = 0; mbr < size; ++mbr) {
                        while ((st.active_mask >> t) & 1) ++t;
                        st.active_mask |= 1 << t;
                        st.new_mask |= 1 << t;
                        st.slot_traj[t] = off + mbr;
                        st.slot_grp[t] = lg;
                        st.slot_member[t] = mbr;
                        st.warm_key[t] = INT_MAX;
                    }
                }
            }
            if (a.deadline_ns != 0ull && globaltimer_ns() > a.deadline_ns) st.timeout = 1;
            for (int t = 0; t < SLOTS; ++t) {
                st.slot_err[t] = 0ull;
                st.sing_key[t] = INT_MAX;
                st.nf_key[t] = INT_MAX;
            }
            st.retire_mask = 0;
            st.free_mask = 0;
        }
        __syncthreads();
        if (st.active_mask == 0) break;
        if (st.timeout) {
            if (tid == 0) {
                for (int lg = 0; lg < SLOTS; ++lg) {
                    const int g = st.grp_id[lg];
                    if (g < 0) continue;
                    a.faults[g].status = FAULT_TIMEOUT;
                    a.faults[g].iteration = st.grp_iter[lg];
                    a.rep_iter[g] = st.grp_iter[lg];
                    a.rep_conv[g] = 0;
                }
            }
            break;
        }

        // ------------------------------------------------ load + warm start
        const int new_mask = st.new_mask;
        if (new_mask) {
            for (int t = tid; t < SLOTS * 6; t += nthr) {
                const int s = t / 6, c = t % 6;
                if ((new_mask >> s) & 1) st.y0[s][c] = a.state_in[static_cast<size_t>(st.slot_traj[s]) * 6 + c];
            }
            __syncthreads();
            for (int i = tid; i < N * SLOTS; i += nthr) {
                const int j = i >> 3, t = i & 7;
                if (!((new_mask >> t) & 1)) continue;
                const double r[3] = {st.y0[t][0], st.y0[t][1], st.y0[t][2]};
                const double v[3] = {st.y0[t][3], st.y0[t][4], st.y0[t][5]};
                double ro[3] = {r[0], r[1], r[2]}, vo[3] = {v[0], v[1], v[2]};
                if (!a.cold_start) {
                    const int chk = conic_check(r, v, a.fd.central_mu);
                    if (chk == CONIC_ZERO_RADIUS) {
                        atomicMin(&st.warm_key[t], j * 4 + CONIC_ZERO_RADIUS);
                    } else if (chk == CONIC_OK) {
                        double mf, ef;
                        if (kepler_propagate(r, v, a.fd.central_mu, a.times[j] - a.epoch, ro, vo, &mf, &ef) !=
                            CONIC_OK)
                            atomicMin(&st.warm_key[t], j * 4 + CONIC_SOLVER);
                    }
                    if (j == 0 && a.cold_fallback)
                        a.cold_fallback[st.slot_traj[t]] = (chk == CONIC_NON_ELLIPTIC) ? 1 : 0;
                }
                double* yp = ybuf + static_cast<size_t>(j) * YS + t;
                yp[0] = ro[0];
                yp[8] = ro[1];
                yp[16] = ro[2];
                yp[24] = vo[0];
                yp[32] = vo[1];
                yp[40] = vo[2];
            }
            __syncthreads();
            // rare path: describe warm-start faults (re-evaluate the failing node)
            if (tid < SLOTS && ((new_mask >> tid) & 1) && st.warm_key[tid] != INT_MAX) {
                const int t = tid, j = st.warm_key[t] / 4;
                st.warm_kind[t] = st.warm_key[t] % 4;
                const double r[3] = {st.y0[t][0], st.y0[t][1], st.y0[t][2]};
                const double v[3] = {st.y0[t][3], st.y0[t][4], st.y0[t][5]};
                double ro[3], vo[3], mf = 0.0, ef = 0.0;
                if (st.warm_kind[t] == CONIC_SOLVER)
                    kepler_propagate(r, v, a.fd.central_mu, a.times[j] - a.epoch, ro, vo, &mf, &ef);
                st.warm_val[t][0] = mf;
                st.warm_val[t][1] = ef;
            }
            __syncthreads();
        }

        // ------------------------------------------------ force -> Fbuf
        const int act = st.active_mask;
        const double w2 = a.omega2;
        for (int i = tid; i < N * SLOTS; i += nthr) {
            const int j = i >> 3, t = i & 7;
            double f[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
            if ((act >> t) & 1) {
                const double* yp = ybuf + static_cast<size_t>(j) * YS + t;
                const double rx = yp[0], ry = yp[8], rz = yp[16];
                double ax = 0.0, ay = 0.0, az = 0.0;
                const int chk = accel(rx, ry, rz, j, a.fd, ax, ay, az);
                if (chk >= 0) atomicMin(&st.sing_key[t], j * (B + 1) + chk);
                f[0] = w2 * yp[24];
                f[1] = w2 * yp[32];
                f[2] = w2 * yp[40];
                f[3] = w2 * ax;
                f[4] = w2 * ay;
                f[5] = w2 * az;
            }
#pragma unroll
            for (int c = 0; c < 6; ++c) fbuf[fbuf_index(j, c * 8 + t)] = f[c];
        }
        __syncthreads();
        if (tid < SLOTS && st.sing_key[tid] != INT_MAX) {
            const int t = tid, key = st.sing_key[t], j = key / (B + 1), chk = key % (B + 1);
            const double* yp = ybuf + static_cast<size_t>(j) * YS + t;
            st.sing_val[t] = check_distance(yp[0], yp[8], yp[16], j, chk, a.fd);
        }

        // ------------------------------------------------ DMMA update
        double acc[2][6][2];
        warp_gemm(a.upack, a.nkp, fbuf, warp, lane, acc);
        {
            const int amt = N >> 3, ag = N & 7;
            if (warp == (amt >> 1) && (lane >> 2) == ag) {
                const int i = amt & 1, q = lane & 3;
#pragma unroll
                for (int c = 0; c < 6; ++c)
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int t = 2 * q + h;
                        const double an = i ? acc[1][c][h] : acc[0][c][h];  // static register selection
                        st.b0h[c * 8 + t] = 0.5 * (an + 2.0 * st.y0[t][c]);
                    }
            }
        }
        __syncthreads();

        // ------------------------------------------------ epilogue: Y' , finite, error
        {
            const int g = lane >> 2, q = lane & 3;
            double emax[2] = {0.0, 0.0};
            int nf[2] = {INT_MAX, INT_MAX};
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                const int j = (2 * warp + i) * 8 + g;
                if (j >= N) continue;
                double* yrow = ybuf + static_cast<size_t>(j) * YS + 2 * q;
                double yn[2][6], yo[2][6];
#pragma unroll
                for (int c = 0; c < 6; ++c) {
                    const double2 prev = *reinterpret_cast<const double2*>(yrow + c * 8);
                    yo[0][c] = prev.x;
                    yo[1][c] = prev.y;
                    yn[0][c] = acc[i][c][0] + st.b0h[c * 8 + 2 * q];
                    yn[1][c] = acc[i][c][1] + st.b0h[c * 8 + 2 * q + 1];
                }
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int t = 2 * q + h;
                    if (!((act >> t) & 1)) {
#pragma unroll
                        for (int c = 0; c < 6; ++c) yn[h][c] = yo[h][c];
                        continue;
                    }
#pragma unroll
                    for (int c = 5; c >= 0; --c)
                        if (!isfinite(yn[h][c])) nf[h] = min(nf[h], j * 8 + c);
                    double dr2 = 0.0, r2 = 0.0, dv2 = 0.0, v2 = 0.0;
#pragma unroll
                    for (int c = 0; c < 3; ++c) {
                        const double dr = yn[h][c] - yo[h][c], dv = yn[h][c + 3] - yo[h][c + 3];
                        dr2 += dr * dr;
                        r2 += yo[h][c] * yo[h][c];
                        dv2 += dv * dv;
                        v2 += yo[h][c + 3] * yo[h][c + 3];
                    }
                    double pos, vel;
                    if (a.error_mode == 1) {
                        pos = sqrt(dr2);
                        vel = sqrt(dv2);
                    } else {
                        pos = sqrt(dr2) / fmax(sqrt(r2), 1e-30);
                        vel = sqrt(dv2) / fmax(sqrt(v2), 1e-30);
                    }
                    emax[h] = fmax(emax[h], fmax(pos, vel));
                }
#pragma unroll
                for (int c = 0; c < 6; ++c)
                    *reinterpret_cast<double2*>(yrow + c * 8) = make_double2(yn[0][c], yn[1][c]);
            }
#pragma unroll
            for (int h = 0; h < 2; ++h) {
#pragma unroll
                for (int off = 4; off < 32; off <<= 1) {
                    emax[h] = fmax(emax[h], __shfl_xor_sync(0xffffffffu, emax[h], off));
                    nf[h] = min(nf[h], __shfl_xor_sync(0xffffffffu, nf[h], off));
                }
            }
            if (g == 0) {
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int t = 2 * q + h;
                    if ((act >> t) & 1) {
                        atomicMax(&st.slot_err[t], static_cast<unsigned long long>(__double_as_longlong(emax[h])));
                        if (nf[h] != INT_MAX) atomicMin(&st.nf_key[t], nf[h]);
                    }
                }
            }
        }
        __syncthreads();

        // ------------------------------------------------ group decisions
        if (tid == 0) {
            for (int lg = 0; lg < SLOTS; ++lg) {
                const int gid = st.grp_id[lg];
                if (gid < 0) continue;
                const int size = st.grp_size[lg];
                double gerr = 0.0;
                long long sing_s = LLONG_MAX;
                int sing_t = -1;
                long long nf_key = LLONG_MAX;
                long long warm_k = LLONG_MAX;
                int warm_t = -1;
                for (int t = 0; t < SLOTS; ++t) {
                    if (!((st.active_mask >> t) & 1) || st.slot_grp[t] != lg) continue;
                    const int mbr = st.slot_member[t];
                    gerr = fmax(gerr, __longlong_as_double(static_cast<long long>(st.slot_err[t])));
                    if (((new_mask >> t) & 1) && st.warm_key[t] != INT_MAX) {
                        // warm_start walks trajectories in batch order (propagator.hpp:86)
                        if (st.slot_traj[t] < warm_k) {
                            warm_k = st.slot_traj[t];
                            warm_t = t;
                        }
                    }
                    if (st.sing_key[t] != INT_MAX) {
                        const long long j = st.sing_key[t] / (B + 1);
                        const long long s = j * size + mbr;  // sample order s = j*m + t
                        if (s < sing_s) {
                            sing_s = s;
                            sing_t = t;
                        }
                    }
                    if (st.nf_key[t] != INT_MAX) {
                        const long long j = st.nf_key[t] >> 3, c = st.nf_key[t] & 7;
                        const long long key = j * (6LL * size) + c * size + mbr;  // row-major (j, col)
                        nf_key = min(nf_key, key);
                    }
                }
                GroupFault* fl = a.faults + gid;
                int it = st.grp_iter[lg];
                bool retire = false, ok = false, conv = false;
                if (warm_t >= 0) {
                    const int t = warm_t;
                    fl->status = st.warm_kind[t] == CONIC_ZERO_RADIUS ? FAULT_WARM_ZERO_RADIUS : FAULT_WARM_SOLVER;
                    fl->iteration = 0;
                    fl->trajectory = st.slot_traj[t];
                    fl->node = st.warm_key[t] / 4;
                    fl->value = st.warm_val[t][0];
                    fl->value2 = st.warm_val[t][1];
                    retire = true;
                } else {
                    it += 1;
                    st.grp_iter[lg] = it;
                    if (sing_t >= 0) {
                        const int key = st.sing_key[sing_t];
                        fl->status = FAULT_SINGULARITY;
                        fl->iteration = it;
                        fl->node = key / (B + 1);
                        fl->body = key % (B + 1) - 1;
                        fl->trajectory = st.slot_member[sing_t];
                        fl->value = st.sing_val[sing_t];
                        retire = true;
                    } else if (nf_key != LLONG_MAX) {
                        fl->status = FAULT_DIVERGENCE;
                        fl->iteration = it;
                        fl->node = nf_key / (6LL * size);
                        fl->column = nf_key % (6LL * size);
                        retire = true;
                    } else {
                        if (a.rep_hist) a.rep_hist[static_cast<size_t>(gid) * a.max_it + (it - 1)] = gerr;
                        if (gerr <= a.tol) {
                            retire = ok = conv = true;
                        } else if (it >= a.max_it) {
                            retire = ok = true;
                        }
                    }
                }
                if (retire) {
                    a.rep_iter[gid] = it;
                    a.rep_err[gid] = gerr;
                    a.rep_conv[gid] = conv ? 1 : 0;
                    for (int t = 0; t < SLOTS; ++t) {
                        if (!((st.active_mask >> t) & 1) || st.slot_grp[t] != lg) continue;
                        st.free_mask |= 1 << t;
                        if (ok) st.retire_mask |= 1 << t;
                    }
                    st.grp_id[lg] = -1;
                }
            }
        }
        __syncthreads();

        // ------------------------------------------------ retire: samples + chained state
        const int retire = st.retire_mask;
        if (retire) {
            const int j_begin = a.seg == 0 ? 0 : 1;
            for (int i = tid; i < N * SLOTS; i += nthr) {
                const int j = i >> 3, t = i & 7;
                if (!((retire >> t) & 1)) continue;
                const double* yp = ybuf + static_cast<size_t>(j) * YS + t;
                const size_t tr = static_cast<size_t>(st.slot_traj[t]);
                if (a.samples && j >= j_begin) {
                    double* o = a.samples + (tr * a.R + a.row0 + j) * 6;
#pragma unroll
                    for (int c = 0; c < 6; ++c) o[c] = yp[c * 8];
                }
                if (j == N - 1) {
#pragma unroll
                    for (int c = 0; c < 6; ++c) a.state_out[tr * 6 + c] = yp[c * 8];
                }
            }
        }
        if (tid == 0) {
            st.active_mask &= ~st.free_mask;
            for (int t = 0; t < SLOTS; ++t)
                if ((st.free_mask >> t) & 1) st.slot_traj[t] = -1;
        }
        __syncthreads();
    }
}

template <int MAXT>
static cudaError_t launch_segment_t(const SegArgs& a, int grid, cudaStream_t s) {
    const size_t smem = segment_smem_bytes(a.N, a.nkp);
    cudaError_t e = cudaFuncSetAttribute(k_pc_segment<MAXT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    k_pc_segment<MAXT><<<grid, 32 * a.warps, smem, s>>>(a);
    return cudaGetLastError();
}

/// Two register budgets: up to 13 warps (N <= 207, e.g. the default N = 200) the
/// kernel gets 128+ registers per thread; up to 17 warps (N <= 264) it gets 120.
cudaError_t launch_segment(const SegArgs& a, int grid, cudaStream_t s) {
    if (32 * a.warps <= 416) return launch_segment_t<416>(a, grid, s);
    return launch_segment_t<544>(a, grid, s);
}

// ===================================================================== ops ==

/// Y = [U; anchor]·F tile per CTA (48 arbitrary columns), all W warps in one CTA.
__global__ void __launch_bounds__(544, 1)
    k_picard_update(int N, int nkp, int C, const double* __restrict__ F, const double* __restrict__ y0,
                    double* __restrict__ out, const double2* __restrict__ upack) {
    extern __shared__ __align__(16) double smem[];
    double* fbuf = smem;
    double* b0h = fbuf + static_cast<size_t>(8 * nkp) * COLS;
    const int KP = 8 * nkp;
    const int col0 = blockIdx.x * COLS;
    const int tid = threadIdx.x, nthr = blockDim.x, warp = tid >> 5, lane = tid & 31;
    for (int i = tid; i < KP * COLS; i += nthr) {
        const int k = i / COLS, n = i % COLS, col = col0 + n;
        fbuf[fbuf_index(k, n)] = (k < N && col < C) ? F[static_cast<size_t>(k) * C + col] : 0.0;
    }
    __syncthreads();
    double acc[2][6][2];
    warp_gemm(upack, nkp, fbuf, warp, lane, acc);
    const int g = lane >> 2, q = lane & 3;
    const int amt = N >> 3, ag = N & 7;
    if (warp == (amt >> 1) && g == ag) {
        const int i = amt & 1;
#pragma unroll
        for (int c = 0; c < 6; ++c)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int n = c * 8 + 2 * q + h, col = col0 + n;
                const double an = i ? acc[1][c][h] : acc[0][c][h];
                b0h[n] = col < C ? 0.5 * (an + 2.0 * y0[col]) : 0.0;
            }
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        const int j = (2 * warp + i) * 8 + g;
        if (j >= N) continue;
#pragma unroll
        for (int c = 0; c < 6; ++c)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int n = c * 8 + 2 * q + h, col = col0 + n;
                if (col < C) out[static_cast<size_t>(j) * C + col] = acc[i][c][h] + b0h[n];
            }
    }
}

cudaError_t launch_picard_update(int N, int nkp, int C, const double* F, const double* y0, double* out,
                                 const double2* upack, cudaStream_t s) {
    const size_t smem = sizeof(double) * (static_cast<size_t>(8 * nkp) * COLS + COLS);
    cudaError_t e = cudaFuncSetAttribute(k_picard_update, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    const int threads = segment_threads(N);
    k_picard_update<<<(C + COLS - 1) / COLS, threads, smem, s>>>(N, nkp, C, F, y0, out, upack);
    return cudaGetLastError();
}

/// Force block over a reference-layout N x 6m state block, one thread per sample.
__global__ void k_force_block(int N, int m, const double* __restrict__ y, double omega2, ForceData fd,
                              double* __restrict__ force, unsigned long long* fault_key) {
    const long long s = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (s >= static_cast<long long>(N) * m) return;
    const int j = static_cast<int>(s / m), t = static_cast<int>(s % m);
    const size_t row = static_cast<size_t>(j) * 6 * m;
    const double rx = y[row + t], ry = y[row + m + t], rz = y[row + 2 * m + t];
    double ax = 0.0, ay = 0.0, az = 0.0;
    const int chk = accel(rx, ry, rz, j, fd, ax, ay, az);
    if (chk >= 0) atomicMin(fault_key, static_cast<unsigned long long>(s) * 64ull + static_cast<unsigned long long>(chk));
    force[row + t] = omega2 * y[row + 3 * m + t];
    force[row + m + t] = omega2 * y[row + 4 * m + t];
    force[row + 2 * m + t] = omega2 * y[row + 5 * m + t];
    force[row + 3 * m + t] = omega2 * ax;
    force[row + 4 * m + t] = omega2 * ay;
    force[row + 5 * m + t] = omega2 * az;
}

cudaError_t launch_force_block(int N, int m, const double* y, double omega2, const ForceData& fd, int kind_nbody,
                               double* force, unsigned long long* fault_key, cudaStream_t s) {
    ForceData f = fd;
    if (!kind_nbody) f.n_bodies = 0;
    const long long n = static_cast<long long>(N) * m;
    k_force_block<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(N, m, y, omega2, f, force, fault_key);
    return cudaGetLastError();
}

/// Per-trajectory max over nodes of the iteration error (augment.hpp:32-55).
__global__ void k_block_error(int N, int m, const double* __restrict__ cur, const double* __restrict__ prev, int mode,
                              unsigned long long* per_state_bits) {
    const long long s = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (s >= static_cast<long long>(N) * m) return;
    const int j = static_cast<int>(s / m), t = static_cast<int>(s % m);
    const size_t row = static_cast<size_t>(j) * 6 * m;
    double dr2 = 0.0, r2 = 0.0, dv2 = 0.0, v2 = 0.0;
    for (int c = 0; c < 3; ++c) {
        const size_t rc = row + static_cast<size_t>(c) * m + t, vc = row + static_cast<size_t>(c + 3) * m + t;
        const double dr = cur[rc] - prev[rc], dv = cur[vc] - prev[vc];
        dr2 += dr * dr;
        r2 += prev[rc] * prev[rc];
        dv2 += dv * dv;
        v2 += prev[vc] * prev[vc];
    }
    double pos, vel;
    if (mode == 1) {
        pos = sqrt(dr2);
        vel = sqrt(dv2);
    } else {
        pos = sqrt(dr2) / fmax(sqrt(r2), 1e-30);
        vel = sqrt(dv2) / fmax(sqrt(v2), 1e-30);
    }
    const double e = fmax(pos, vel);
    atomicMax(per_state_bits + t, static_cast<unsigned long long>(__double_as_longlong(e)));
}

cudaError_t launch_block_error(int N, int m, const double* cur, const double* prev, int mode,
                               unsigned long long* per_state_bits, cudaStream_t s) {
    const long long n = static_cast<long long>(N) * m;
    k_block_error<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(N, m, cur, prev, mode, per_state_bits);
    return cudaGetLastError();
}

/// Conic warm start, one thread per (trajectory, node) (propagator.hpp:81-103).
__global__ void k_warm_start(int M, const double* __restrict__ states, int N, const double* __restrict__ times,
                             double mu, double* __restrict__ guesses, uint8_t* fallback,
                             unsigned long long* fault_key, double* fault_vals, int describe) {
    const long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= static_cast<long long>(M) * N) return;
    const int i = static_cast<int>(idx / N), j = static_cast<int>(idx % N);
    const double* s = states + static_cast<size_t>(i) * 7;
    const double r[3] = {s[1], s[2], s[3]}, v[3] = {s[4], s[5], s[6]};
    double ro[3] = {r[0], r[1], r[2]}, vo[3] = {v[0], v[1], v[2]};
    const int chk = conic_check(r, v, mu);
    double mf = 0.0, ef = 0.0;
    int fail = -1;
    if (chk == CONIC_ZERO_RADIUS) {
        fail = CONIC_ZERO_RADIUS;
    } else if (chk == CONIC_OK) {
        if (kepler_propagate(r, v, mu, times[j] - s[0], ro, vo, &mf, &ef) != CONIC_OK) fail = CONIC_SOLVER;
    }
    if (describe) {
        if (fail >= 0 && static_cast<unsigned long long>(idx) * 4ull + fail == *fault_key) {
            fault_vals[0] = mf;
            fault_vals[1] = ef;
        }
        return;
    }
    if (fail >= 0) atomicMin(fault_key, static_cast<unsigned long long>(idx) * 4ull + static_cast<unsigned long long>(fail));
    if (j == 0 && fallback) fallback[i] = chk == CONIC_NON_ELLIPTIC ? 1 : 0;
    double* o = guesses + static_cast<size_t>(idx) * 6;
    o[0] = ro[0];
    o[1] = ro[1];
    o[2] = ro[2];
    o[3] = vo[0];
    o[4] = vo[1];
    o[5] = vo[2];
}

cudaError_t launch_warm_start(int M, const double* states, int N, const double* times, double mu, double* guesses,
                              uint8_t* fallback, unsigned long long* fault_key, double* fault_vals, cudaStream_t s) {
    const long long n = static_cast<long long>(M) * N;
    const unsigned blocks = static_cast<unsigned>((n + 127) / 128);
    k_warm_start<<<blocks, 128, 0, s>>>(M, states, N, times, mu, guesses, fallback, fault_key, fault_vals, 0);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess || fault_vals == nullptr) return e;
    k_warm_start<<<blocks, 128, 0, s>>>(M, states, N, times, mu, guesses, fallback, fault_key, fault_vals, 1);
    return cudaGetLastError();
}

}  // namespace pswarm_dev
