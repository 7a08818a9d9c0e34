#include <algorithm>
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
#include "pc_tile.cuh"

namespace pswarm_dev {

namespace {

struct CtaState {
    int slot_traj[SLOTS];      // batch index, -1 = free
    int slot_grp[SLOTS];       // local group index
    int slot_member[SLOTS];    // member index within its group
    int sing_key[SLOTS];       // min j*(B+1)+check this tick
    int nf_key[SLOTS];         // min j*8+c non-finite this tick
    int warm_key[SLOTS];       // min node*4+kind with a warm-start fault
    int warm_kind[SLOTS];
    unsigned long long slot_err[SLOTS];  // max squared error ratio (bit pattern)
    double sing_val[SLOTS];
    double warm_val[SLOTS][2];
    double y0[SLOTS][6];
    double b0h[COLS];
    int grp_id[SLOTS];         // global group id, -1 = free
    int grp_size[SLOTS];
    int grp_iter[SLOTS];
    int grp_floor[SLOTS];  // wide-group round: converge only at it >= floor
    int grp_cap[SLOTS];    // stop at it >= cap (max_iterations, or a round's target)
    unsigned long long grp_t0[SLOTS];  // %globaltimer at the claim (per-trajectory budgets only)
    int active_mask;
    int new_mask;
    int retire_mask;           // slots whose results are written out this tick
    int free_mask;             // slots released this tick (retired or failed)
    int queue_done;
    int timeout;
};

__device__ __forceinline__ int popc(int x) { return __popc(static_cast<unsigned>(x)); }

// Optional per-phase cycle accounting (pswarm_set_option "profile_phases"): thread 0
// stamps clock64() at phase ends; the sums land in a.phase_cycles[PHASES].
#define PHASE(k)                                            \
    do {                                                    \
        if (prof && tid == 0) {                             \
            const long long now_ = clock64();               \
            pc[(k)] += now_ - t_prev;                       \
            t_prev = now_;                                  \
        }                                                   \
    } while (0)


struct SmemLayout {
    size_t ybuf, fbuf, xstage, eph, state, total;  // byte offsets
};

__host__ __device__ inline SmemLayout smem_layout(int N, int nkp, int xrows, int B, int stage_eph) {
    SmemLayout L;
    L.ybuf = 0;
    L.fbuf = L.ybuf + sizeof(double) * static_cast<size_t>(N) * COLS;
    L.xstage = L.fbuf + sizeof(double) * static_cast<size_t>(8 * nkp) * COLS;
    L.eph = L.xstage + sizeof(double) * static_cast<size_t>(xrows) * COLS;
    L.state = L.eph + (stage_eph ? sizeof(double) * static_cast<size_t>(N) * (3 * B + 3) : 0);
    L.total = L.state + sizeof(CtaState);
    return L;
}

}  // namespace

size_t segment_smem_bytes(int N, int nkp, int xrows, int B, int stage_eph) {
    return smem_layout(N, nkp, xrows, B, stage_eph).total;
}

GemmPlan make_gemm_plan(int N) {
    GemmPlan gp{};
    gp.mtiles = (N + 1 + 7) / 8;
    if (gp.mtiles < 8) {  // small N: 4 warps, up to XMAX_SMALL single tiles each
        gp.warps = 4;
        gp.main = gp.mtiles / 4;
        gp.mb = gp.main * 4;
        gp.extras = (gp.mtiles - gp.mb) * 6;
        gp.xmax = XMAX_SMALL;
        return gp;
    }
    for (int w = 4 * (gp.mtiles / 8); w <= 16; w += 4) {  // the kernels launch at most 16 warps
        const int main = gp.mtiles / w < 2 ? gp.mtiles / w : 2;
        const int extras = (gp.mtiles - main * w) * 6;
        if ((extras + w - 1) / w <= XMAX) {
            gp.warps = w;
            gp.main = main;
            gp.mb = main * w;
            gp.extras = extras;
            gp.xmax = XMAX;
            return gp;
        }
    }
    // 29-31 m-tiles (N = 225..247): no 16-warp plan with <= XMAX extras per warp; pad the
    // operator to 32 m-tiles (zero rows past N, never written back): 16 warps x 2 full tiles
    if (gp.mtiles <= 32) {
        gp.mtiles = 32;
        gp.warps = 16;
        gp.main = 2;
        gp.mb = 32;
        gp.extras = 0;
        gp.xmax = XMAX;
        return gp;
    }
    gp.warps = 0;  // no plan: N beyond the device path (rejected by the host)
    return gp;
}

int extra_rows(int N, const GemmPlan& gp) {
    const int r = N - gp.mb * 8;
    return r > 0 ? r : 0;
}

template <int MAXT, int XM, bool STAGE, int FS, bool REL>
__global__ void __launch_bounds__(MAXT, 1) k_pc_segment(const SegArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int N = a.N;
    const int B = a.fd.n_bodies;
    const GemmPlan gp = a.gp;
    const SmemLayout L = smem_layout(N, a.nkp, a.xrows, B, a.stage_eph);
    double* ybuf = reinterpret_cast<double*>(smem_raw + L.ybuf);
    double* fbuf = reinterpret_cast<double*>(smem_raw + L.fbuf);
    double* xstage = reinterpret_cast<double*>(smem_raw + L.xstage);
    double* eph = reinterpret_cast<double*>(smem_raw + L.eph);
    CtaState& st = *reinterpret_cast<CtaState*>(smem_raw + L.state);
    const int KP = 8 * a.nkp;
    const int tid = threadIdx.x, nthr = blockDim.x, warp = tid >> 5, lane = tid & 31;
    const int g = lane >> 2, q = lane & 3;
    const bool prof = a.phase_cycles != nullptr;
    long long pc[PHASES] = {};
    long long t_prev = clock64();

    for (int i = tid; i < KP * COLS; i += nthr) fbuf[i] = 0.0;
    // frozen per-segment ephemeris [N][B][3] + indirect [N][3] staged once per launch
    if (STAGE && B > 0) {
        for (int i = tid; i < N * 3 * B; i += nthr) eph[i] = a.fd.body_pos[i];
        for (int i = tid; i < N * 3; i += nthr) eph[N * 3 * B + i] = a.fd.indirect[i];
    }
    const double* pos_base = STAGE ? eph : a.fd.body_pos;
    const double* ind_base = STAGE ? eph + N * 3 * B : a.fd.indirect;
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
            int new_mask = 0;
            int am = st.active_mask;
            const int free_slots = SLOTS - popc(am);
            if (!st.queue_done && free_slots >= a.gmax) {
                const int k = free_slots / a.gmax;
                const int g0 = atomicAdd(a.queue, k);
                const int g1 = min(g0 + k, a.P);
                if (g0 + k >= a.P) st.queue_done = 1;
                for (int gi = g0; gi < g1; ++gi) {
                    int lg = 0;
                    while (st.grp_id[lg] >= 0) ++lg;
                    int off, size, gid;
                    claim_group(a, gi, off, size, gid);
                    st.grp_id[lg] = gid;
                    st.grp_size[lg] = size;
                    st.grp_iter[lg] = start_iteration(a, off);
                    st.grp_floor[lg] = claim_floor(a, gid);
                    st.grp_cap[lg] = claim_cap(a, gid);
                    if (a.traj_ns) st.grp_t0[lg] = globaltimer_ns();
                    int t = 0;
                    for (int mbr = 0; mbr < size; ++mbr) {
                        while ((am >> t) & 1) ++t;
                        am |= 1 << t;
                        new_mask |= 1 << t;
                        st.slot_traj[t] = off + mbr;
                        st.slot_grp[t] = lg;
                        st.slot_member[t] = mbr;
                        st.warm_key[t] = INT_MAX;
                    }
                }
            }
            st.active_mask = am;
            st.new_mask = new_mask;
            if (a.deadline_ns != 0ull && globaltimer_ns() > a.deadline_ns) st.timeout = 1;
        }
        if (tid < SLOTS) {
            st.slot_err[tid] = 0ull;
            st.sing_key[tid] = INT_MAX;
            st.nf_key[tid] = INT_MAX;
        }
        __syncthreads();
        PHASE(0);
        if (st.active_mask == 0) break;
        if (st.timeout) {
            if (tid == 0) {
                for (int lg = 0; lg < SLOTS; ++lg) {
                    const int gi = st.grp_id[lg];
                    if (gi < 0) continue;
                    a.faults[gi].status = FAULT_TIMEOUT;
                    a.faults[gi].iteration = st.grp_iter[lg];
                    a.rep_iter[gi] = st.grp_iter[lg];
                    a.rep_conv[gi] = 0;
                }
            }
            break;
        }

        // ------------------------------------------------ load + warm start
        const int new_mask = st.new_mask;
        if (new_mask) {
            for (int i = tid; i < SLOTS * 6; i += nthr) {
                const int s = i / 6, c = i % 6;
                if ((new_mask >> s) & 1) st.y0[s][c] = a.state_in[static_cast<size_t>(st.slot_traj[s]) * 6 + c];
            }
            __syncthreads();
            for (int i = tid; i < N * SLOTS; i += nthr) {
                const int j = i >> 3, t = i & 7;
                if (!((new_mask >> t) & 1)) continue;
                const double r[3] = {st.y0[t][0], st.y0[t][1], st.y0[t][2]};
                const double v[3] = {st.y0[t][3], st.y0[t][4], st.y0[t][5]};
                double ro[3] = {r[0], r[1], r[2]}, vo[3] = {v[0], v[1], v[2]};
                if (start_iteration(a, st.slot_traj[t]) > 0) {  // wide-group round: resume the saved iterate
                    resume_node(a, st.slot_traj[t], j, ro, vo);
                } else {
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
                    if (a.hot)
                        hot_start_node(a.hot + (static_cast<size_t>(st.slot_traj[t]) * N + j) * 6, a.hot_apply, ro, vo);
                }
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    ybuf[yidx(j, c, t)] = ro[c];
                    ybuf[yidx(j, c + 3, t)] = vo[c];
                }
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
        }
        PHASE(1);

        // ------------------------------------------------ force -> Fbuf
        // Thread = one node x FS slots (body positions read once, FS independent
        // dependency chains); when N*8/FS exceeds the thread count the leftover
        // samples ride along as one extra chain in the first warps, so every warp is
        // busy for a single pass (the force shares the FP64 pipe with DMMA).
        const int act = st.active_mask;
        {
            const int items = N * (SLOTS / FS);
            const int extra = items > nthr ? (items - nthr) * FS : 0;  // leftover single samples
            for (int it0 = tid; it0 < (items > nthr ? nthr : items); it0 += nthr) {
                const int jq = it0 / (SLOTS / FS), t0 = (it0 % (SLOTS / FS)) * FS;
                if (tid < extra) {
                    const int sx = nthr * FS + tid;
                    force_chains<FS, true, REL>(a.fd, a.omega2, ybuf, fbuf, st.sing_key, pos_base, ind_base, act, jq, t0,
                                           sx >> 3, sx & 7);
                } else {
                    force_chains<FS, false, REL>(a.fd, a.omega2, ybuf, fbuf, st.sing_key, pos_base, ind_base, act, jq, t0,
                                            0, 0);
                }
            }
        }
        // operator prefetch (L2 -> registers) overlaps the barrier wait
        const APrefetch<XM> pre = gemm_prefetch<XM>(a.upack, a.nkp, gp, warp, lane);
        PHASE(2);
        __syncthreads();
        if (tid < SLOTS && st.sing_key[tid] != INT_MAX) {
            const int t = tid, key = st.sing_key[t], j = key / (B + 1), chk = key % (B + 1);
            st.sing_val[t] = check_distance(ybuf[yidx(j, 0, t)], ybuf[yidx(j, 1, t)], ybuf[yidx(j, 2, t)], j, chk, a.fd);
        }

        // ------------------------------------------------ DMMA update
        double acc[2][6][2], xacc[XM][2];
        warp_gemm<XM>(a.upack, a.nkp, fbuf, gp, warp, lane, pre, acc, xacc);
        PHASE(3);
        // anchor row N -> b0/2 = (anchor_op·F + 2 y0)/2 (pc_matrices.hpp:138, :145)
        {
            const int amt = N >> 3;
            if (g == (N & 7)) {
#pragma unroll
                for (int i = 0; i < 2; ++i) {
                    if (i < gp.main && warp * gp.main + i == amt) {
#pragma unroll
                        for (int c = 0; c < 6; ++c)
#pragma unroll
                            for (int h = 0; h < 2; ++h) {
                                const int t = 2 * q + h;
                                const double an = i ? acc[1][c][h] : acc[0][c][h];
                                st.b0h[c * 8 + t] = 0.5 * (an + 2.0 * st.y0[t][c]);
                            }
                    }
                }
#pragma unroll
                for (int x = 0; x < XM; ++x) {
                    const int e = warp + x * gp.warps;
                    if (e < gp.extras && gp.mb + e / 6 == amt) {
                        const int c = e % 6;
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            const int t = 2 * q + h;
                            st.b0h[c * 8 + t] = 0.5 * (xacc[x][h] + 2.0 * st.y0[t][c]);
                        }
                    }
                }
            }
        }
        __syncthreads();
        PHASE(4);

        // ------------------------------------------------ epilogue: main rows in registers
        {
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
                    yn[0][c] = acc[i][c][0] + st.b0h[c * 8 + 2 * q];
                    yn[1][c] = acc[i][c][1] + st.b0h[c * 8 + 2 * q + 1];
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
            // extra tiles: one component per tile -> stage Y' for the cross-warp epilogue
#pragma unroll
            for (int x = 0; x < XM; ++x) {
                const int e = warp + x * gp.warps;
                if (e >= gp.extras) continue;
                const int j = (gp.mb + e / 6) * 8 + g, c = e % 6;
                if (j >= N) continue;
#pragma unroll
                for (int h = 0; h < 2; ++h)
                    xstage[(j - gp.mb * 8) * COLS + c * 8 + 2 * q + h] = xacc[x][h] + st.b0h[c * 8 + 2 * q + h];
            }
            double emax[2];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                emax[h] = bn[h] / bd[h];
#pragma unroll
                for (int off = 4; off < 32; off <<= 1) {
                    emax[h] = fmax(emax[h], __shfl_xor_sync(0xffffffffu, emax[h], off));
                    nf[h] = min(nf[h], __shfl_xor_sync(0xffffffffu, nf[h], off));
                }
            }
            if (g == 0 && gp.main > 0) {
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
        PHASE(5);

        // ------------------------------------------------ epilogue: extra rows from the stage
        // every staged row (up to 31 x 8 items on the 128-thread small-N plan)
        for (int i = tid; i < a.xrows * SLOTS; i += blockDim.x) {
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
                const double e2 = bn / bd;
#pragma unroll
                for (int c = 0; c < 6; ++c) ybuf[yidx(j, c, t)] = yn[c];
                atomicMax(&st.slot_err[t], static_cast<unsigned long long>(__double_as_longlong(e2)));
                if (nf != INT_MAX) atomicMin(&st.nf_key[t], nf);
            }
        }
        __syncthreads();
        PHASE(6);

        // ------------------------------------------------ group decisions (warp 0, lane = slot)
        // The lowest active slot of each group leads it: gathers the member maxima /
        // first-fault keys, applies the stopping rule of pc_solve (picard.hpp:66-81)
        // and writes the group's report.  Leaders of different groups run in parallel.
        if (warp == 0) {
            const int am = st.active_mask;
            const int t = lane;
            const bool act_t = t < SLOTS && ((am >> t) & 1);
            // each lane loads its own slot record once; leaders gather with shuffles
            const int my_grp = act_t ? st.slot_grp[t] : -1;
            const int my_mbr = act_t ? st.slot_member[t] : 0;
            const double my_e2 = act_t ? __longlong_as_double(static_cast<long long>(st.slot_err[t])) : 0.0;
            const int my_sk = act_t ? st.sing_key[t] : INT_MAX;
            const int my_nk = act_t ? st.nf_key[t] : INT_MAX;
            const int my_wk = (act_t && ((new_mask >> t) & 1)) ? st.warm_key[t] : INT_MAX;
            const int my_tr = act_t ? st.slot_traj[t] : INT_MAX;
            const int lg = my_grp;
            const int gid = act_t ? st.grp_id[lg] : -1;
            const int size = act_t ? st.grp_size[lg] : 1;
            int it = act_t ? st.grp_iter[lg] : 0;
            bool leader = act_t;
            double gerr2 = 0.0;
            long long sing_s = LLONG_MAX, nf_best = LLONG_MAX;
            int sing_t = -1, warm_t = -1, warm_tr = INT_MAX, members = 0;
            if (a.gmax == 1) {  // singleton groups (independent mode): each lane owns its group
                members = act_t ? 1 << t : 0;
                gerr2 = my_e2;
                if (my_wk != INT_MAX) warm_t = t;
                if (my_sk != INT_MAX) sing_t = t;
                if (my_nk != INT_MAX) nf_best = static_cast<long long>(my_nk >> 3) * 6 + (my_nk & 7);
            } else
#pragma unroll
            for (int u = 0; u < SLOTS; ++u) {
                const int ug = __shfl_sync(0xffffffffu, my_grp, u);
                const int um = __shfl_sync(0xffffffffu, my_mbr, u);
                const double ue = __shfl_sync(0xffffffffu, my_e2, u);
                const int usk = __shfl_sync(0xffffffffu, my_sk, u);
                const int unk = __shfl_sync(0xffffffffu, my_nk, u);
                const int uwk = __shfl_sync(0xffffffffu, my_wk, u);
                const int utr = __shfl_sync(0xffffffffu, my_tr, u);
                if (!act_t || ug != lg) continue;
                if (u < t) leader = false;
                members |= 1 << u;
                gerr2 = fmax(gerr2, ue);
                if (uwk != INT_MAX && utr < warm_tr) {  // warm_start walks the batch in order (propagator.hpp:86)
                    warm_tr = utr;
                    warm_t = u;
                }
                if (usk != INT_MAX) {
                    const long long smp = static_cast<long long>(usk / (B + 1)) * size + um;  // s = j*m + t
                    if (smp < sing_s) {
                        sing_s = smp;
                        sing_t = u;
                    }
                }
                if (unk != INT_MAX) {  // row-major (node, column = comp*m + member)
                    const long long key = static_cast<long long>(unk >> 3) * (6LL * size) +
                                          static_cast<long long>(unk & 7) * size + um;
                    nf_best = min(nf_best, key);
                }
            }
            __syncwarp();  // every lane has read the slot / group records the leader rewrites
            int free_bits = 0, retire_bits = 0;
            if (leader) {
                const double gerr = sqrt(gerr2);
                GroupFault* fl = a.faults + gid;
                bool retire = false, ok = false, conv = false;
                if (warm_t >= 0) {
                    fl->status = st.warm_kind[warm_t] == CONIC_ZERO_RADIUS ? FAULT_WARM_ZERO_RADIUS : FAULT_WARM_SOLVER;
                    fl->iteration = 0;
                    fl->trajectory = st.slot_traj[warm_t];
                    fl->node = st.warm_key[warm_t] / 4;
                    fl->value = st.warm_val[warm_t][0];
                    fl->value2 = st.warm_val[warm_t][1];
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
                    } else if (nf_best != LLONG_MAX) {
                        fl->status = FAULT_DIVERGENCE;
                        fl->iteration = it;
                        fl->node = nf_best / (6LL * size);
                        fl->column = nf_best % (6LL * size);
                        retire = true;
                    } else {
                        if (a.rep_hist) a.rep_hist[static_cast<size_t>(gid) * a.hist_stride + (it - 1)] = gerr;
                        if (gerr <= a.tol && it >= st.grp_floor[lg]) {
                            retire = ok = conv = true;
                        } else if (it >= st.grp_cap[lg]) {
                            retire = ok = true;
                        }
                    }
                }
                if (a.traj_ns && traj_budget_spent(a, st.slot_traj[t], st.grp_t0[lg], retire)) {  // singleton groups
                    fl->status = FAULT_TIMEOUT;
                    fl->iteration = it;
                    retire = true;
                }
                if (retire) {
                    a.rep_iter[gid] = it;
                    a.rep_err[gid] = gerr;
                    a.rep_conv[gid] = conv ? 1 : 0;
                    free_bits = members;
                    retire_bits = ok ? members : 0;
                    st.grp_id[lg] = -1;
                }
            }
            free_bits = __reduce_or_sync(0xffffffffu, static_cast<unsigned>(free_bits));
            retire_bits = __reduce_or_sync(0xffffffffu, static_cast<unsigned>(retire_bits));
            if (lane == 0) {
                st.free_mask = free_bits;
                st.retire_mask = retire_bits;
            }
        }
        __syncthreads();
        PHASE(7);

        // ------------------------------------------------ retire: samples + chained state
        const int retire = st.retire_mask;
        if (retire) {
            const int j_begin = a.seg == 0 ? 0 : 1;
            for (int i = tid; i < N * SLOTS; i += nthr) {
                const int j = i >> 3, t = i & 7;
                if (!((retire >> t) & 1)) continue;
                const size_t tr = static_cast<size_t>(st.slot_traj[t]);
                if (a.samples && j >= j_begin) {
                    double* o = a.samples + (tr * a.R + a.row0 + j) * 6;
#pragma unroll
                    for (int c = 0; c < 6; ++c) o[c] = ybuf[yidx(j, c, t)];
                }
                if (a.hot)
                    for (int c = 0; c < 6; ++c) hot_retire_node(a.hot + (tr * N + j) * 6, c, ybuf[yidx(j, c, t)]);
                if (a.blk)  // wide-group round: the full iterate (resume source)
                    for (int c = 0; c < 6; ++c) a.blk[(tr * N + j) * 6 + c] = ybuf[yidx(j, c, t)];
                if (j == N - 1) {
#pragma unroll
                    for (int c = 0; c < 6; ++c) a.state_out[tr * 6 + c] = ybuf[yidx(j, c, t)];
                }
            }
            __syncthreads();  // slot_traj is cleared below
        }
        if (tid == 0) {
            const int fm = st.free_mask;
            st.active_mask &= ~fm;
            for (int t = 0; t < SLOTS; ++t)
                if ((fm >> t) & 1) st.slot_traj[t] = -1;
        }
        __syncthreads();
        PHASE(8);
    }
    if (prof && tid == 0) {
        pc[PHASES - 1] += 1;  // CTA count
        for (int k = 0; k < PHASES; ++k) atomicAdd(a.phase_cycles + k, static_cast<unsigned long long>(pc[k]));
    }
}

template <int MAXT, int XM, int FS>
static cudaError_t launch_segment_t(const SegArgs& a, int grid, size_t smem, cudaStream_t s) {
    auto kern = a.fd.rel ? k_pc_segment<MAXT, XM, false, FS, true>
                         : (a.stage_eph ? k_pc_segment<MAXT, XM, true, FS, false> : k_pc_segment<MAXT, XM, false, FS, false>);
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    kern<<<grid, 32 * a.gp.warps, smem, s>>>(a);
    return cudaGetLastError();
}

/// Register budgets: up to 12 warps (N <= 207, e.g. the default N = 200) the kernel gets
/// up to 168 registers per thread; up to 16 warps (N <= 264) 128; small N (< 63) runs
/// 4 warps with up to 6 single tiles each.
cudaError_t launch_segment(const SegArgs& a, int grid, cudaStream_t s) {
    const size_t smem = segment_smem_bytes(a.N, a.nkp, a.xrows, a.fd.n_bodies, a.stage_eph);
    if (a.gp.xmax == XMAX_SMALL) return launch_segment_t<128, XMAX_SMALL, 4>(a, grid, smem, s);
    if (a.gp.warps <= 12) return launch_segment_t<384, XMAX, 4>(a, grid, smem, s);
    return launch_segment_t<512, XMAX, 4>(a, grid, smem, s);
}

// ============================================================== ephemeris ==

__global__ void k_ephemeris(int N, const double* __restrict__ times, double central_mu, BodyTable bt,
                            double* __restrict__ pos, double* __restrict__ indirect, unsigned long long* fault_key,
                            double* __restrict__ vel, double* __restrict__ rel_tab, double ic2,
                            double* __restrict__ eph_t) {
    const int j = blockIdx.x, b = threadIdx.x;
    const double t = times[j];
    const bool rel = rel_tab != nullptr;
    if (b < bt.B) {
        double p[3] = {0.0, 0.0, 0.0}, v[3] = {0.0, 0.0, 0.0};
        if (bt.kind[b] == 0) {
            double mf;
            const int st = rel ? elements_state(bt.elements + 7 * b, central_mu, t, p, v, &mf)
                               : elements_position(bt.elements + 7 * b, central_mu, t, p, &mf);
            if (st != CONIC_OK) atomicMin(fault_key, (static_cast<unsigned long long>(b) * N + j) * 4ull + 3ull);
        } else {
            int hit = -1;
            for (int sg = bt.seg_off[b]; sg < bt.seg_off[b + 1]; ++sg) {
                const double t0 = bt.seg_bounds[2 * sg], t1 = bt.seg_bounds[2 * sg + 1];
                const bool fwd = t0 <= t1;
                if ((fwd && t >= t0 && t <= t1) || (!fwd && t <= t0 && t >= t1)) {
                    hit = sg;
                    break;
                }
            }
            if (hit < 0) {
                atomicMin(fault_key, (static_cast<unsigned long long>(b) * N + j) * 4ull + 1ull);
            } else {
                const double t0 = bt.seg_bounds[2 * hit], t1 = bt.seg_bounds[2 * hit + 1];
                const double tau = (2.0 * t - (t0 + t1)) / (t1 - t0);
                const int nc = bt.ncoef[b];
                const double* c = bt.coeffs + bt.coeff_off[hit];
                for (int k = 0; k < 3; ++k) p[k] = clenshaw(c + k * nc, nc, tau);
                if (rel)
                    for (int k = 0; k < 3; ++k) v[k] = (2.0 / (t1 - t0)) * clenshaw_deriv(c + k * nc, nc, tau);
            }
        }
        double* o = pos + (static_cast<size_t>(j) * bt.B + b) * 3;
        o[0] = p[0];
        o[1] = p[1];
        o[2] = p[2];
        if (eph_t)  // node-contiguous copy for the slot kernels' bulk staging
            for (int c = 0; c < 3; ++c) eph_t[static_cast<size_t>(3 * b + c) * eph_ld(N) + j] = p[c];
        if (rel) {
            double* w = vel + (static_cast<size_t>(j) * bt.B + b) * 3;
            w[0] = v[0];
            w[1] = v[1];
            w[2] = v[2];
        }
    }
    __syncthreads();
    if (b == 0) {  // fixed summation order over bodies (deterministic)
        double s[3] = {0.0, 0.0, 0.0};
        for (int k = 0; k < bt.B; ++k) {
            const double* q = pos + (static_cast<size_t>(j) * bt.B + k) * 3;
            const double bn = sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2]);
            const double bn3 = bn * bn * bn;
            const double mu = bt.mu[k];
            for (int c = 0; c < 3; ++c) s[c] += mu * (q[c] / bn3);
        }
        for (int c = 0; c < 3; ++c) indirect[j * 3 + c] = s[c];
        if (eph_t)
            for (int c = 0; c < 3; ++c) eph_t[static_cast<size_t>(3 * bt.B + c) * eph_ld(N) + j] = s[c];
        if (rel)  // the node row of the relativistic table ends with the indirect term
            for (int c = 0; c < 3; ++c) rel_tab[static_cast<size_t>(j) * rel_stride(bt.B) + (bt.B + 1) * REL_W + c] = s[c];
    }
    if (rel && b <= bt.B) {
        // EXTENSION: relativistic node table row A = b (0 = Sun): Newtonian heliocentric
        // acceleration of body A and the potential of the other massive bodies at A
        const double* P = pos + static_cast<size_t>(j) * bt.B * 3;
        double* row = rel_tab + static_cast<size_t>(j) * rel_stride(bt.B) + b * REL_W;
        double r[3] = {0.0, 0.0, 0.0}, v[3] = {0.0, 0.0, 0.0}, acc[3] = {0.0, 0.0, 0.0}, phi = 0.0, mu = central_mu;
        if (b == 0) {
            for (int k = 0; k < bt.B; ++k) {
                const double* q = P + 3 * k;
                phi += bt.mu[k] / sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2]);
            }
        } else {
            const int bb = b - 1;
            mu = bt.mu[bb];
            for (int c = 0; c < 3; ++c) {
                r[c] = P[3 * bb + c];
                v[c] = vel[(static_cast<size_t>(j) * bt.B + bb) * 3 + c];
            }
            const double rb = sqrt(r[0] * r[0] + r[1] * r[1] + r[2] * r[2]);
            const double k0 = -(central_mu + mu) / (rb * rb * rb);
            for (int c = 0; c < 3; ++c) acc[c] = k0 * r[c];
            phi = central_mu / rb;
            for (int k = 0; k < bt.B; ++k) {
                if (k == bb) continue;
                const double* q = P + 3 * k;
                const double d[3] = {q[0] - r[0], q[1] - r[1], q[2] - r[2]};
                const double dn = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
                const double rk = sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2]);
                for (int c = 0; c < 3; ++c) acc[c] += bt.mu[k] * (d[c] / (dn * dn * dn) - q[c] / (rk * rk * rk));
                phi += bt.mu[k] / dn;
            }
        }
        for (int c = 0; c < 3; ++c) {
            row[c] = r[c];
            row[3 + c] = v[c];
            row[6 + c] = acc[c];
        }
        row[9] = mu;
        row[10] = ic2 * (2.0 * (v[0] * v[0] + v[1] * v[1] + v[2] * v[2]) - phi);
        row[11] = 0.0;
    }
}

/// Batch states [M][7] = (epoch, r, v) as the caller passed them -> the solver's [M][6]:
/// the host copies the caller's buffer as is (one DMA, no host repacking pass).
__global__ void k_repack_states(const double* __restrict__ s7, double* __restrict__ s6, long long M) {
    const long long n = M * 6;
    for (long long k = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; k < n;
         k += static_cast<long long>(gridDim.x) * blockDim.x)
        s6[k] = s7[(k / 6) * 7 + 1 + k % 6];
}

/// Terminal states [M][6] -> the caller's [M][7] = (epoch, r, v) layout on the device, so one
/// DMA lands them in a page-locked caller buffer.
__global__ void k_pack_states7(const double* __restrict__ s6, double epoch, double* __restrict__ s7, long long M) {
    for (long long k = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; k < M * 7;
         k += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long i = k / 7, c = k % 7;
        s7[k] = c == 0 ? epoch : s6[i * 6 + c - 1];
    }
}

cudaError_t launch_pack_states7(const double* s6, double epoch, double* s7, long long M, cudaStream_t s) {
    const long long n = M * 7;
    const int grid = static_cast<int>(std::max<long long>(1, std::min<long long>((n + 255) / 256, 148 * 16)));
    k_pack_states7<<<grid, 256, 0, s>>>(s6, epoch, s7, M);
    return cudaGetLastError();
}

cudaError_t launch_repack_states(const double* s7, double* s6, long long M, cudaStream_t s) {
    const long long n = M * 6;
    const int grid = static_cast<int>(std::min<long long>((n + 255) / 256, 148 * 16));
    k_repack_states<<<grid, 256, 0, s>>>(s7, s6, M);
    return cudaGetLastError();
}

/// Trajectory list 0..n-1 (first member-level round of the wide-group path).
__global__ void k_iota(int32_t* out, int n) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) out[i] = i;
}

cudaError_t launch_iota(int32_t* out, int n, cudaStream_t s) {
    const int grid = std::max(1, std::min((n + 255) / 256, 148 * 8));
    k_iota<<<grid, 256, 0, s>>>(out, n);
    return cudaGetLastError();
}

/// Group error history of a wide-group segment (augment.hpp:137 via pc_solve's history): the
/// group's error at iteration k is the max over its members (block_max_error), k < K[g].
/// Block = a chunk of HIST_CHUNK consecutive members, thread = iteration k (coalesced rows of
/// the member history); each thread keeps the running max of the current group and flushes it
/// with one atomicMax when the group changes or the chunk ends.  Non-negative doubles order
/// like their IEEE bits.  gh [P][stride] must be zero on entry; k_group_hist_fill writes NaN
/// past each K[g].
constexpr int HIST_CHUNK = 256;
__global__ void k_group_hist(const double* __restrict__ mh, int stride, const int64_t* __restrict__ group_off, int P,
                             const int32_t* __restrict__ gK, int M, unsigned long long* gh) {
    const int lo = blockIdx.x * HIST_CHUNK, hi = min(lo + HIST_CHUNK, M);
    if (lo >= hi) return;
    int g0 = 0, gh_ = P;  // group of member lo: upper_bound over the offsets
    while (gh_ - g0 > 1) {
        const int mid = (g0 + gh_) / 2;
        if (group_off[mid] <= lo) g0 = mid; else gh_ = mid;
    }
    for (int k = threadIdx.x; k < stride; k += blockDim.x) {
        int g = g0;
        long long gend = group_off[g + 1];
        unsigned long long run = 0ull;
        for (int m = lo; m < hi; ++m) {
            if (m >= gend) {  // next group: flush the finished one
                if (k < gK[g]) atomicMax(gh + static_cast<size_t>(g) * stride + k, run);
                run = 0ull;
                while (m >= gend) gend = group_off[++g + 1];
            }
            if (k < gK[g])
                run = max(run, static_cast<unsigned long long>(__double_as_longlong(mh[static_cast<size_t>(m) * stride + k])));
        }
        if (k < gK[g]) atomicMax(gh + static_cast<size_t>(g) * stride + k, run);
    }
}

__global__ void k_group_hist_fill(int stride, const int32_t* __restrict__ gK, int P, unsigned long long* gh) {
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < static_cast<long long>(P) * stride;
         i += static_cast<long long>(gridDim.x) * blockDim.x)
        if (i % stride >= gK[i / stride]) gh[i] = ~0ull;
}

cudaError_t launch_group_hist(const double* mh, int stride, const int64_t* group_off, int P, const int32_t* gK, int M,
                              double* gh, cudaStream_t s) {
    auto* ghb = reinterpret_cast<unsigned long long*>(gh);
    const int threads = std::min(256, 32 * ((stride + 31) / 32));
    k_group_hist<<<(M + HIST_CHUNK - 1) / HIST_CHUNK, threads, 0, s>>>(mh, stride, group_off, P, gK, M, ghb);
    const long long n = static_cast<long long>(P) * stride;
    k_group_hist_fill<<<static_cast<int>(std::max<long long>(1, std::min<long long>((n + 255) / 256, 148 * 8))), 256, 0,
                        s>>>(stride, gK, P, ghb);
    return cudaGetLastError();
}

cudaError_t launch_ephemeris(int N, const double* times, double central_mu, const BodyTable& bt, double* pos,
                             double* indirect, unsigned long long* fault_key, double* vel, double* rel_tab, double ic2,
                             double* eph_t, cudaStream_t s) {
    if (bt.B <= 0 && rel_tab == nullptr) return cudaSuccess;
    const int threads = 32 * ((bt.B + 1 + 31) / 32);
    k_ephemeris<<<N, threads, 0, s>>>(N, times, central_mu, bt, pos, indirect, fault_key, vel, rel_tab, ic2, eph_t);
    return cudaGetLastError();
}

// ===================================================================== ops ==

/// Y = [U; anchor]·F tile per CTA (48 arbitrary columns), same warp plan as the
/// segment kernel; every output element is written straight from its fragment.
template <int MAXT, int XM>
__global__ void __launch_bounds__(MAXT, 1)
    k_picard_update(int N, int nkp, GemmPlan gp, int C, const double* __restrict__ F, const double* __restrict__ y0,
                    double* __restrict__ out, const double2* __restrict__ upack) {
    extern __shared__ __align__(16) double smem[];
    double* fbuf = smem;
    double* b0h = fbuf + static_cast<size_t>(8 * nkp) * COLS;
    const int KP = 8 * nkp;
    const int col0 = blockIdx.x * COLS;
    const int tid = threadIdx.x, nthr = blockDim.x, warp = tid >> 5, lane = tid & 31;
    const int g = lane >> 2, q = lane & 3;
    for (int i = tid; i < KP * COLS; i += nthr) {
        const int k = i / COLS, n = i % COLS, col = col0 + n;
        fbuf[fbuf_index(k, n)] = (k < N && col < C) ? F[static_cast<size_t>(k) * C + col] : 0.0;
    }
    const APrefetch<XM> pre = gemm_prefetch<XM>(upack, nkp, gp, warp, lane);
    __syncthreads();
    double acc[2][6][2], xacc[XM][2];
    warp_gemm<XM>(upack, nkp, fbuf, gp, warp, lane, pre, acc, xacc);
    const int amt = N >> 3;
    if (g == (N & 7)) {
#pragma unroll
        for (int i = 0; i < 2; ++i)
            if (i < gp.main && warp * gp.main + i == amt)
#pragma unroll
                for (int c = 0; c < 6; ++c)
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int n = c * 8 + 2 * q + h, col = col0 + n;
                        const double an = i ? acc[1][c][h] : acc[0][c][h];
                        b0h[n] = col < C ? 0.5 * (an + 2.0 * y0[col]) : 0.0;
                    }
#pragma unroll
        for (int x = 0; x < XM; ++x) {
            const int e = warp + x * gp.warps;
            if (e < gp.extras && gp.mb + e / 6 == amt)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int n = (e % 6) * 8 + 2 * q + h, col = col0 + n;
                    b0h[n] = col < C ? 0.5 * (xacc[x][h] + 2.0 * y0[col]) : 0.0;
                }
        }
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        if (i >= gp.main) continue;
        const int j = (warp * gp.main + i) * 8 + g;
        if (j >= N) continue;
#pragma unroll
        for (int c = 0; c < 6; ++c)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int n = c * 8 + 2 * q + h, col = col0 + n;
                if (col < C) out[static_cast<size_t>(j) * C + col] = acc[i][c][h] + b0h[n];
            }
    }
#pragma unroll
    for (int x = 0; x < XM; ++x) {
        const int e = warp + x * gp.warps;
        if (e >= gp.extras) continue;
        const int j = (gp.mb + e / 6) * 8 + g;
        if (j >= N) continue;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int n = (e % 6) * 8 + 2 * q + h, col = col0 + n;
            if (col < C) out[static_cast<size_t>(j) * C + col] = xacc[x][h] + b0h[n];
        }
    }
}

cudaError_t launch_picard_update(int N, int nkp, int C, const double* F, const double* y0, double* out,
                                 const double2* upack, cudaStream_t s) {
    const GemmPlan gp = make_gemm_plan(N);
    const size_t smem = sizeof(double) * (static_cast<size_t>(8 * nkp) * COLS + COLS);
    auto kern = gp.xmax == XMAX_SMALL ? k_picard_update<128, XMAX_SMALL> : k_picard_update<512, XMAX>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    kern<<<(C + COLS - 1) / COLS, 32 * gp.warps, smem, s>>>(N, nkp, gp, C, F, y0, out, upack);
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
    const int chk = accel(rx, ry, rz, fd.body_pos + static_cast<size_t>(j) * 3 * fd.n_bodies, fd.indirect + 3 * j, fd,
                          ax, ay, az);
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
