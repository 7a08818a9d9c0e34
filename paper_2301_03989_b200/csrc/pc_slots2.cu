// Slot kernels of the persistent solve for groups of at most 4 trajectories
// (independent mode = singleton groups): the warp-specialised k_pc_ws (dense update, or
// mirror-folded when N % 8 == 0 — the default path) and the unified k_pc_uni.
//
// k_pc_ws: the 8 trajectory slots of a CTA are split into two halves of 4.  Sixteen warps
// form two groups that run the halves out of phase:
//   MMA group (warps 0-7):  [DMMA update of half h] -> [epilogue of half h: + b0/2,
//                           finite check, error] -> (folded) [staged rows, decisions]
//                           -> signal "Y_h ready"
//   FP group  (warps 8-15): [(dense) decisions / retire / refill / warm start of half h]
//                           -> [force of half h (folded: mirrored node pairs)] -> b0
//                           -> signal "F_h ready"
// On B200 the DMMA and DFMA paths share one FP64 datapath (tools/fp64_peak.cu,
// tools/ws_mix.cu), so the two groups' FP64 work largely serialises; the split still
// hides the integer / shared-memory latency of one phase under the other.
// Hand-off is through named barriers (bar.arrive / bar.sync).  Semantics are identical to
// k_pc_segment (pc_kernels.cu): pc_solve's loop (picard.hpp:66-81) per group with
// per-trajectory masking and refill.
//
// Half layout (per half: 4 slots x 6 components = 24 block columns = 3 MMA n-tiles):
//   n-tile p holds components 2p, 2p+1; column within the tile = slot*2 + (comp & 1),
//   so C-fragment lane (g, q) holds all six components of slot q of row g.
#include <algorithm>
#include <climits>

#ifndef PSWARM_ABLATE
#define PSWARM_ABLATE 0  // diagnostic builds only (tools/ablate.sh)
#endif

#include "pc_kernels.cuh"
#include "pc_tile.cuh"

namespace pswarm_dev {
// The same source compiles twice (csrc/Makefile): the default 512-thread kernels (8 MMA + 8 FP
// warps, one CTA per SM) and, with -DPSWARM_SLOTS_SMALL, 256-thread kernels (4 + 4 warps) that
// run two CTAs per SM for small N, in namespace pswarm_dev::small.
#ifdef PSWARM_SLOTS_SMALL
namespace small {
#endif

namespace {

constexpr int HS = 4;            // slots per half
constexpr int HC = 6 * HS;       // columns per half
// Ybuf row stride 52 doubles (= 4 mod 16): a half-warp touching 4 rows x 4 slots (epilogue,
// retire, warm start) covers 16 distinct banks; the slot index is XOR-swizzled with
// (j >> 2) & 3 so the force's 16 consecutive rows of one column do as well.
constexpr int YS2 = 2 * HC + 4;
#ifndef PSWARM_MMA_WARPS
#define PSWARM_MMA_WARPS 8
#endif
#ifndef PSWARM_FP_WARPS
#define PSWARM_FP_WARPS 8
#endif
#ifndef PSWARM_MIN_BLOCKS
#define PSWARM_MIN_BLOCKS 1  // CTAs per SM the launch bounds promise (2 for the small variant)
#endif
constexpr int MMA_WARPS = PSWARM_MMA_WARPS, FP_WARPS = PSWARM_FP_WARPS;
constexpr int MMA_THREADS = 32 * MMA_WARPS, FP_THREADS = 32 * FP_WARPS, WS_THREADS = MMA_THREADS + FP_THREADS;
constexpr int BAR_F0 = 1, BAR_Y0 = 3, BAR_MMA = 5, BAR_FP = 6, BAR_B0 = 7;  // F_h = 1+h, Y_h = 3+h, B_h = 7+h

__device__ __forceinline__ int y2(int j, int h, int c, int s) {
    return j * YS2 + h * HC + c * HS + (s ^ ((j >> 2) & 3));
}
/// B-fragment index of F(node j, comp c, slot s) within a half's Fbuf: per k-step (4 nodes)
/// three 32-double fragments (one per n-tile) + 4 doubles of padding, so the force
/// threads' stores (consecutive nodes j, bank set by j & 3 and the k-step) spread over
/// all banks instead of 4.
constexpr int FKS = 3 * 32 + 4;  // doubles per k-step
#ifndef PSWARM_FP_UNROLL
#define PSWARM_FP_UNROLL 2
#endif
constexpr int kForceUnroll = PSWARM_FP_UNROLL;  // body-loop unroll of force_pair (diagnostic knob)
__device__ __forceinline__ int f2(int j, int c, int s) {
    return (j >> 2) * FKS + (c >> 1) * 32 + ((s * 2 + (c & 1)) * 4 + (j & 3));
}

// Optional phase accounting (pswarm_set_option "profile_phases"): MMA-group lane 0 of
// warp 0 stamps slots 0-3 (wait F, DMMA, epilogue, wait b0), FP-group thread 0 slots
// 4-9 (wait Y, staged rows + decisions, retire + claim, warm start, force, b0).
#define WS_PHASE(k)                                  \
    do {                                             \
        if (prof && stamp) {                         \
            const long long now_ = clock64();        \
            s_pc[(k)] += now_ - s_prev[grp_];        \
            s_prev[grp_] = now_;                     \
        }                                            \
    } while (0)

__device__ __forceinline__ void bar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void bar_arrive(int id, int n) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}

struct WsState {
    uint64_t stage_bar;  // mbarrier of the per-launch bulk staging of the ephemeris
    int slot_traj[SLOTS];
    int slot_grp[SLOTS];
    int slot_member[SLOTS];
    int sing_key[SLOTS];
    int nf_key[SLOTS];
    int warm_key[SLOTS];
    int warm_kind[SLOTS];
    unsigned long long slot_err[SLOTS];
    double sing_val[SLOTS];
    double warm_val[SLOTS][2];
    double y0[SLOTS][6];
    double b0h[2][HC];
    int grp_id[SLOTS];
    int grp_size[SLOTS];
    int grp_iter[SLOTS];
    int grp_floor[SLOTS];  // wide-group round: converge only at it >= floor
    int grp_cap[SLOTS];    // stop at it >= cap (max_iterations, or a round's target)
    unsigned long long grp_t0[SLOTS];  // %globaltimer at the claim (per-trajectory budgets only)
    int act_word[2];     // active slots of half h (bits h*HS..h*HS+3); the MMA group reads
                         // act_word[h] while the FP group claims into act_word[h ^ 1]
    int new_mask[2];     // slots claimed at the last refill of each half
    int free_mask[2];    // per half: written by that half's decisions
    int retire_mask[2];
    int half_active[2];  // MMA group skips an empty half
    int queue_done;
    int timeout;
    int exit_flag;
};

struct WsLayout {
    size_t ybuf, fbuf0, fbuf1, xstage, anchor, b0part, eph, state, total;
};

constexpr int B0_PARTS = FP_WARPS;  // one partial sum per FP warp and b0 column

/// Mirror-folded update (fold = 1): U anticommutes with the node reversal
/// (U[N-1-j][N-1-k] = -U[j][k], Chebyshev-Lobatto nodes are mirrored, chebyshev.hpp:33-43),
/// so with s_k = F_k + F_{N-1-k} and a_k = F_k - F_{N-1-k} (k < N/2)
///   Y_j + Y_{N-1-j} = sum_k (U[j][k] - U[j][N-1-k]) a_k,  Y_j - Y_{N-1-j} = sum_k (U[j][k] + U[j][N-1-k]) s_k:
/// two (N/2) x (N/2) contractions instead of one N x N (half the DMMAs).  Fbuf then holds
/// s_k at position k and a_{N-1-p} at position p >= N/2; the extra k-steps past N stay zero.
__host__ __device__ inline int ws_fold_ksteps(int N, int nkp) {
    const int half = N / 2, nkpf = (half + 7) / 8;
    const int need = half / 4 + 2 * nkpf;
    return need > 2 * nkp ? need + (need & 1) : 2 * nkp;
}

__host__ __device__ inline WsLayout ws_layout(int N, int nkp, int xrows, int B, int stage_eph, int fold, bool rel = false) {
    WsLayout L;
    L.ybuf = 0;
    L.fbuf0 = L.ybuf + sizeof(double) * static_cast<size_t>(N) * YS2;
    const size_t fb = sizeof(double) * static_cast<size_t>(fold ? ws_fold_ksteps(N, nkp) : 2 * nkp) * FKS;
    L.fbuf1 = L.fbuf0 + fb;
    L.xstage = L.fbuf1 + fb;  // [2 halves][fold ? lo, hi : 1][xrows][HC]
    L.anchor = L.xstage + sizeof(double) * (fold ? 4 : 2) * static_cast<size_t>(xrows) * HC;
    L.b0part = L.anchor + sizeof(double) * static_cast<size_t>(8 * nkp);
    // staged table (bulk copy target, 16-byte aligned): Newtonian eph_t [3B + 3][eph_ld(N)], or
    // the relativistic node table [N][rel_stride(B)]
    L.eph = (L.b0part + sizeof(double) * 2 * B0_PARTS * HC + 15) & ~static_cast<size_t>(15);  // b0part: [half][part][HC]
    L.state = L.eph + (stage_eph ? sizeof(double) * eph_stage_doubles(N, B, rel) : 0);
    L.total = L.state + sizeof(WsState);
    return L;
}

/// Tile plan of one half (25 m-tiles x 3 n-tiles at N = 200) over the 8 MMA warps:
/// `main` consecutive full-width m-tiles per warp + up to XMW single extra tiles.
struct HalfPlan {
    int main, mb, extras;
};

template <int MAIN, int NX>
struct APairH {
    double2 m[MAIN];
    double2 x[NX > 0 ? NX : 1];
};

/// One warp's share of Y'_h = U F_h over all K (LDG.128 operator pairs, double-buffered;
/// B fragments are LDS.64 of the fragment-native half Fbuf).  NX = this warp's number of
/// single extra tiles, a compile-time constant: a predicated-off DMMA still costs a pipe
/// slot (tools/ws_micro.cu: 16.7 k -> 15.2 k cycles per half without it at N = 192).
template <int MAIN, int NX>
__device__ __forceinline__ void gemm_core(const double2* __restrict__ upack, int nkp, const double* fb,
                                          const HalfPlan& hp, int warp, int lane, double (&acc)[MAIN][3][2],
                                          double (*xacc)[2]) {
#pragma unroll
    for (int i = 0; i < MAIN; ++i)
#pragma unroll
        for (int p = 0; p < 3; ++p) acc[i][p][0] = acc[i][p][1] = 0.0;
    constexpr int XA = NX > 0 ? NX : 1;
    const double2* am[MAIN];
    const double2* ax[XA];
    int xp[XA];
    double xa[XA][2];
#pragma unroll
    for (int i = 0; i < MAIN; ++i) am[i] = upack + static_cast<size_t>(warp * MAIN + i) * nkp * 32 + lane;
#pragma unroll
    for (int x = 0; x < NX; ++x) {
        const int e = warp + x * MMA_WARPS;
        ax[x] = upack + static_cast<size_t>(hp.mb + e / 3) * nkp * 32 + lane;
        xp[x] = e % 3;
        xa[x][0] = xa[x][1] = 0.0;
    }
    auto load = [&](int kp, APairH<MAIN, NX>& p) {
#pragma unroll
        for (int i = 0; i < MAIN; ++i) p.m[i] = __ldg(am[i] + kp * 32);
#pragma unroll
        for (int x = 0; x < NX; ++x) p.x[x] = __ldg(ax[x] + kp * 32);
    };
    auto compute = [&](int kp, const APairH<MAIN, NX>& c) {
#pragma unroll
        for (int s = 0; s < 2; ++s) {
            const int ks = 2 * kp + s;
            const double* fk = fb + ks * FKS + lane;
            const double b0 = fk[0], b1 = fk[32], b2 = fk[64];
            const double bv[3] = {b0, b1, b2};
#pragma unroll
            for (int i = 0; i < MAIN; ++i) {
                const double a = s ? c.m[i].y : c.m[i].x;
#pragma unroll
                for (int p = 0; p < 3; ++p) dmma(acc[i][p][0], acc[i][p][1], a, bv[p]);
            }
#pragma unroll
            for (int x = 0; x < NX; ++x) {
                const double bx = xp[x] == 0 ? b0 : (xp[x] == 1 ? b1 : b2);
                dmma(xa[x][0], xa[x][1], s ? c.x[x].y : c.x[x].x, bx);
            }
        }
    };
    if constexpr (MAIN + NX <= 4) {
        APairH<MAIN, NX> p0, p1, p2;  // two operator pairs in flight (L2 latency under load)
        load(0, p0);
        if (nkp > 1) load(1, p1);
        int kp = 0;
        for (; kp + 2 < nkp; kp += 3) {
            load(kp + 2, p2);
            compute(kp, p0);
            if (kp + 3 < nkp) load(kp + 3, p0);
            compute(kp + 1, p1);
            if (kp + 4 < nkp) load(kp + 4, p1);
            compute(kp + 2, p2);
        }
        if (kp < nkp) compute(kp, p0);
        if (kp + 1 < nkp) compute(kp + 1, p1);
    } else {  // wide warps: one pair in flight keeps the accumulators in registers
        APairH<MAIN, NX> p0, p1;
        load(0, p0);
        int kp = 0;
        for (; kp + 1 < nkp; kp += 2) {
            load(kp + 1, p1);
            compute(kp, p0);
            if (kp + 2 < nkp) load(kp + 2, p0);
            compute(kp + 1, p1);
        }
        if (kp < nkp) compute(kp, p0);
    }
#pragma unroll
    for (int x = 0; x < NX; ++x) {
        xacc[x][0] = xa[x][0];
        xacc[x][1] = xa[x][1];
    }
}

/// gemm_core for this warp's (uniform) number of extra tiles, 0..XMW.
template <int MAIN, int XMW>
__device__ __forceinline__ void gemm_half(const double2* __restrict__ upack, int nkp, const double* fb,
                                          const HalfPlan& hp, int warp, int lane, double (&acc)[MAIN][3][2],
                                          double (&xacc)[XMW][2]) {
    int nx = 0;
#pragma unroll
    for (int x = 0; x < XMW; ++x) {
        xacc[x][0] = xacc[x][1] = 0.0;
        nx += warp + x * MMA_WARPS < hp.extras ? 1 : 0;
    }
    if (nx == 0) {
        gemm_core<MAIN, 0>(upack, nkp, fb, hp, warp, lane, acc, xacc);
    } else if (nx == 1 || XMW == 1) {
        gemm_core<MAIN, 1>(upack, nkp, fb, hp, warp, lane, acc, xacc);
    } else if constexpr (XMW >= 2) {
        if (nx == 2 || XMW == 2)
            gemm_core<MAIN, 2>(upack, nkp, fb, hp, warp, lane, acc, xacc);
        else if constexpr (XMW >= 3)
            gemm_core<MAIN, 3>(upack, nkp, fb, hp, warp, lane, acc, xacc);
    }
}

/// Folded counterpart of gemm_core: each of the warp's NV tiles is a pair tile (rows
/// 8mt..8mt+7 of both half-size operators), mt = warp + i * MMA_WARPS (strided), plus NX
/// (0/1) single-n-tile unit of a leftover pair tile (xt, n-tile xp) that balances the four
/// SMSPs' DMMA streams: acc[.][.][0] = Y_j + Y_{N-1-j} part (upf part 1, Fbuf positions
/// >= N/2), acc[.][.][1] = Y_j - Y_{N-1-j} part (upf part 0, positions < N/2).
/// upf layout: [pair mt][part][k-pair][lane] double2, nkpf k-pairs per part.
template <int NV, int NX, int MAIN>
__device__ __forceinline__ void gemm_core_fold(const double2* __restrict__ upf, int nkpf, int half, const double* fb,
                                               int warp, int lane, int xt, int xp, double (&acc)[MAIN][3][2][2],
                                               double (&xacc)[2][2]) {
    constexpr int NA = NV + NX;
    const double2* am[NA][2];
#pragma unroll
    for (int i = 0; i < NA; ++i) {
        const int t = i < NV ? warp + i * MMA_WARPS : xt;
#pragma unroll
        for (int u = 0; u < 2; ++u) am[i][u] = upf + (static_cast<size_t>(t) * 2 + (1 - u)) * nkpf * 32 + lane;
    }
    const double* fb_lo = fb + lane;                          // part 0: s at positions < N/2
    const double* fb_hi = fb + (half >> 2) * FKS + lane;      // part 1: a at positions >= N/2
    struct Pair {
        double2 m[NA][2];
    };
    auto load = [&](int kp, Pair& c) {
#pragma unroll
        for (int i = 0; i < NA; ++i)
#pragma unroll
            for (int u = 0; u < 2; ++u) c.m[i][u] = __ldg(am[i][u] + (PSWARM_ABLATE == 5 ? 0 : kp * 32));  // 5: L1-hot A
    };
    auto compute = [&](int kp, const Pair& c) {
#pragma unroll
        for (int sub = 0; sub < 2; ++sub) {
            const int ks = PSWARM_ABLATE == 6 ? sub : 2 * kp + sub;  // 6: diagnostic, B from k-steps 0-1 only
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const double* fk = (u ? fb_lo : fb_hi) + ks * FKS;
                const double bv[3] = {fk[0], fk[32], fk[64]};
#pragma unroll
                for (int i = 0; i < NV; ++i) {
                    const double av = sub ? c.m[i][u].y : c.m[i][u].x;
#pragma unroll
                    for (int p = 0; p < 3; ++p) dmma(acc[i][p][u][0], acc[i][p][u][1], av, bv[p]);
                }
                if constexpr (NX > 0) {
                    const double bx = xp == 0 ? bv[0] : (xp == 1 ? bv[1] : bv[2]);
                    dmma(xacc[u][0], xacc[u][1], sub ? c.m[NV][u].y : c.m[NV][u].x, bx);
                }
            }
        }
    };
    Pair p0, p1;  // one k-pair in flight: two operator parts per tile
    load(0, p0);
    int kp = 0;
    for (; kp + 1 < nkpf; kp += 2) {
        load(kp + 1, p1);
        compute(kp, p0);
        if (kp + 2 < nkpf) load(kp + 2, p0);
        compute(kp + 1, p1);
    }
    if (kp < nkpf) compute(kp, p0);
}

/// The warp's folded share of half h: its full pair tiles (0..MAIN of tiles < nfull) and
/// its extra unit (xt >= 0) — compile-time counts (a predicated-off DMMA costs a pipe slot).
template <int MAIN>
__device__ __forceinline__ void gemm_half_fold(const double2* __restrict__ upf, int nkpf, int half, const double* fb,
                                               int nfull, int warp, int lane, int xt, int xp,
                                               double (&acc)[MAIN][3][2][2], double (&xacc)[2][2]) {
#pragma unroll
    for (int i = 0; i < MAIN; ++i)
#pragma unroll
        for (int p = 0; p < 3; ++p)
#pragma unroll
            for (int u = 0; u < 2; ++u) acc[i][p][u][0] = acc[i][p][u][1] = 0.0;
    xacc[0][0] = xacc[0][1] = xacc[1][0] = xacc[1][1] = 0.0;
    if (PSWARM_ABLATE == 3) return;  // diagnostic: no DMMA
    const int nv = warp + (MAIN - 1) * MMA_WARPS < nfull ? MAIN : (warp < nfull ? 1 : 0);
    if (xt >= 0) {  // extra units go to warps with fewer than MAIN full tiles (host plan)
        if (nv >= 1) gemm_core_fold<1, 1, MAIN>(upf, nkpf, half, fb, warp, lane, xt, xp, acc, xacc);
        else gemm_core_fold<0, 1, MAIN>(upf, nkpf, half, fb, warp, lane, xt, xp, acc, xacc);
    } else {
        if (nv == MAIN) gemm_core_fold<MAIN, 0, MAIN>(upf, nkpf, half, fb, warp, lane, xt, xp, acc, xacc);
        else if constexpr (MAIN >= 2) {
            if (nv == 1) gemm_core_fold<1, 0, MAIN>(upf, nkpf, half, fb, warp, lane, xt, xp, acc, xacc);
        }
    }
}

/// Relativistic force of half h for node j (EXTENSION, n_body_1pn): one fused pass over
/// the massive bodies of the node table (Sun row first) per slot pair yields both the
/// Newtonian sum and the EIH 1PN terms from the same d, |d|^-1 (see rel_correction for the
/// factorisation); the reference's singularity guards run exactly on the slow path.
template <int NS, bool GLOBAL_TAB>
__device__ __forceinline__ void force_half_rel(const ForceData& fd, const double* rel_base, const double* ybuf,
                                               double* fb, int* sing_key, int act_h, int h, int j, int s_begin) {
    constexpr int PAIR = NS < 2 ? NS : 2;  // slots per fused pass
    const int B = fd.n_bodies, nb1 = B + 1;
    const double ic2 = fd.ic2;
    const double* rt = rel_base + static_cast<size_t>(j) * rel_stride(B);  // staged (smem) or global
    const double ix = rt[nb1 * REL_W], iy = rt[nb1 * REL_W + 1], iz = rt[nb1 * REL_W + 2];
#pragma unroll 1
    for (int s0 = s_begin; s0 < s_begin + NS; s0 += PAIR) {
        // Per body A (d = r_A - r, rho = |d|, g = mu_A / rho^3):
        //   U += mu_A / rho,  n += g d,  b += g [K_A - (4 v.v_A + 1.5 (d.v_A / rho)^2 - 0.5 d.a_A) / c^2] d,
        //   w_A = -g d.(4v - 3 v_A) = -g (4 d.v - 3 d.v_A),  W += w_A,
        //   sum_A w_A (v - v_A) = v W - sum_A w_A v_A,  q += (mu_A / rho) a_A
        // -- the EIH terms of rel_correction with d.(4v - 3v_A) and the (v - v_A) factor expanded
        // (8 FP64 operations fewer per body).  b, -sum w_A v_A / c^2 and 3.5 q / c^2 share ONE
        // accumulator C (14 doubles of state per chain instead of 20, fewer register spills); the
        // correction is f n + C + v W / c^2.  Both rewrites change only the rounding of the 1/c^2
        // terms, ~1e-8 of the acceleration
        const double k35 = 3.5 * ic2;
        double rx[PAIR], ry[PAIR], rz[PAIR], vx[PAIR], vy[PAIR], vz[PAIR];
        double U[PAIR], nx[PAIR], ny[PAIR], nz[PAIR], cx[PAIR], cy[PAIR], cz[PAIR], W[PAIR];
        bool on[PAIR];
        bool flag = false;
#pragma unroll
        for (int k = 0; k < PAIR; ++k) {
            const int s = s0 + k;
            on[k] = (act_h >> s) & 1;
            rx[k] = on[k] ? ybuf[y2(j, h, 0, s)] : 1.0e8;
            ry[k] = on[k] ? ybuf[y2(j, h, 1, s)] : 0.0;
            rz[k] = on[k] ? ybuf[y2(j, h, 2, s)] : 0.0;
            vx[k] = on[k] ? ybuf[y2(j, h, 3, s)] : 0.0;
            vy[k] = on[k] ? ybuf[y2(j, h, 4, s)] : 0.0;
            vz[k] = on[k] ? ybuf[y2(j, h, 5, s)] : 0.0;
            U[k] = nx[k] = ny[k] = nz[k] = cx[k] = cy[k] = cz[k] = W[k] = 0.0;
            flag |= !(rx[k] * rx[k] + ry[k] * ry[k] + rz[k] * rz[k] > 0.0);
        }
        // single chain (small N): 3 bodies in flight for ILP; slot pairs already give 2 chains
#pragma unroll(PAIR == 1 ? 3 : 1)
        for (int A = 0; A < nb1; ++A) {
            const double* t = rt + A * REL_W;
            // table in global memory (not staged): the single-chain path (3 bodies unrolled) loads
            // with ld.global.ca, which the compiler does not hoist across the unrolled bodies --
            // hoisted, its 33 live table values spilled 116 B per thread in the whole kernel
            auto ld = [t](int i) { return (GLOBAL_TAB && PAIR == 1) ? __ldca(t + i) : t[i]; };
            const double tx = ld(0), ty = ld(1), tz = ld(2), vax = ld(3), vay = ld(4), vaz = ld(5);
            const double aax = ld(6), aay = ld(7), aaz = ld(8), mu = ld(9), K = ld(10);
#pragma unroll
            for (int k = 0; k < PAIR; ++k) {
                const double dx = tx - rx[k], dy = ty - ry[k], dz = tz - rz[k];
                const double d2 = dx * dx + dy * dy + dz * dz;
                if (A > 0) flag |= below_bits(d2, fd.floor2_hi_bits);  // integer pre-test, off the FP64 pipe
                double ir = rsqrt_newton(d2, rsqrt_seed(d2));
                if (A == 0) ir = rsqrt_newton(d2, ir);  // central term: full precision
                const double mi = mu * ir, g = mi * ir * ir;
                U[k] += mi;
                nx[k] = fma(g, dx, nx[k]);
                ny[k] = fma(g, dy, ny[k]);
                nz[k] = fma(g, dz, nz[k]);
                const double vva = vx[k] * vax + vy[k] * vay + vz[k] * vaz;
                const double dva = dx * vax + dy * vay + dz * vaz;
                const double dv = dx * vx[k] + dy * vy[k] + dz * vz[k];
                const double daa = dx * aax + dy * aay + dz * aaz;
                const double di = dva * ir;
                const double br = g * (K - ic2 * fma(4.0, vva, fma(1.5 * di, di, -0.5 * daa)));
                const double w = g * fma(3.0, dva, -4.0 * dv);
                const double wv = -ic2 * w, qa = k35 * mi;
                W[k] += w;
                cx[k] = fma(br, dx, fma(wv, vax, fma(qa, aax, cx[k])));
                cy[k] = fma(br, dy, fma(wv, vay, fma(qa, aay, cy[k])));
                cz[k] = fma(br, dz, fma(wv, vaz, fma(qa, aaz, cz[k])));
            }
        }
        if (flag) {  // rare: exact guard order of table_acceleration (force_model.hpp:57-69)
#pragma unroll
            for (int k = 0; k < PAIR; ++k) {
                if (!on[k]) continue;
                int fail = (rx[k] * rx[k] + ry[k] * ry[k] + rz[k] * rz[k] > 0.0) ? -1 : 0;
                for (int b = 0; b < B && fail < 0; ++b) {
                    const double* q = rt + (b + 1) * REL_W;
                    const double dx = q[0] - rx[k], dy = q[1] - ry[k], dz = q[2] - rz[k];
                    if (sqrt(dx * dx + dy * dy + dz * dz) < fd.floor_km) fail = 1 + b;
                }
                if (fail >= 0) atomicMin(&sing_key[h * HS + s0 + k], j * (B + 1) + fail);
            }
        }
#pragma unroll
        for (int k = 0; k < PAIR; ++k) {
            const int s = s0 + k;
            const double f = ic2 * (vx[k] * vx[k] + vy[k] * vy[k] + vz[k] * vz[k] - 4.0 * U[k]);
            const double iw = ic2 * W[k];
            const double ax = (nx[k] - ix) + fma(f, nx[k], fma(iw, vx[k], cx[k]));
            const double ay = (ny[k] - iy) + fma(f, ny[k], fma(iw, vy[k], cy[k]));
            const double az = (nz[k] - iz) + fma(f, nz[k], fma(iw, vz[k], cz[k]));
            fb[f2(j, 0, s)] = on[k] ? vx[k] : 0.0;
            fb[f2(j, 1, s)] = on[k] ? vy[k] : 0.0;
            fb[f2(j, 2, s)] = on[k] ? vz[k] : 0.0;
            fb[f2(j, 3, s)] = on[k] ? ax : 0.0;
            fb[f2(j, 4, s)] = on[k] ? ay : 0.0;
            fb[f2(j, 5, s)] = on[k] ? az : 0.0;
        }
    }
}

/// Force of half h for node j, slots [s0, s0 + NS) as independent chains (force_model.hpp:93-142).
/// F holds [v, a] unscaled: the segment's omega2 (force_model.hpp:122-127) is applied by the
/// epilogue (Y' = omega2 U F + b0/2 with b0 = omega2 anchor.F + 2 y0), one FMA per entry.
template <int NS>
__device__ __forceinline__ void force_half(const ForceData& fd, const double* ybuf, double* fb, int* sing_key,
                                           const double* pos_base, const double* ind_base, int psj, int psc,
                                           int act_h, int h, int j, int s0) {
    const int B = fd.n_bodies;
    double rx[NS], ry[NS], rz[NS], ax[NS], ay[NS], az[NS], r2[NS], ir[NS];
    bool on[NS];
    bool flag = false;
#pragma unroll
    for (int s = 0; s < NS; ++s) {
        on[s] = (act_h >> (s0 + s)) & 1;
        rx[s] = on[s] ? ybuf[y2(j, h, 0, s0 + s)] : 1.0e8;
        ry[s] = on[s] ? ybuf[y2(j, h, 1, s0 + s)] : 0.0;
        rz[s] = on[s] ? ybuf[y2(j, h, 2, s0 + s)] : 0.0;
        r2[s] = rx[s] * rx[s] + ry[s] * ry[s] + rz[s] * rz[s];
        flag |= !(r2[s] > 0.0);
    }
#pragma unroll
    for (int s = 0; s < NS; ++s) ir[s] = rsqrt_newton(r2[s], rsqrt_newton(r2[s], rsqrt_seed(r2[s])));
#pragma unroll
    for (int s = 0; s < NS; ++s) {
        const double sc = -fd.central_mu * (ir[s] * ir[s] * ir[s]);
        ax[s] = sc * rx[s];
        ay[s] = sc * ry[s];
        az[s] = sc * rz[s];
    }
    const double* bp = pos_base + static_cast<size_t>(j) * psj;  // element (b, c) at bp[(3b + c) * psc]
#pragma unroll 4
    for (int b = 0; b < B; ++b) {
        const double mu8 = 0.125 * __ldg(fd.body_mu + b);
        const double qx = bp[(3 * b) * psc], qy = bp[(3 * b + 1) * psc], qz = bp[(3 * b + 2) * psc];
        double dx[NS], dy[NS], dz[NS], d2[NS], y[NS];
#pragma unroll
        for (int s = 0; s < NS; ++s) {
            dx[s] = qx - rx[s];
            dy[s] = qy - ry[s];
            dz[s] = qz - rz[s];
            d2[s] = dx[s] * dx[s] + dy[s] * dy[s] + dz[s] * dz[s];
            flag |= below_bits(d2[s], fd.floor2_hi_bits);
        }
#pragma unroll
        for (int s = 0; s < NS; ++s) y[s] = body_mu_ir3(d2[s], mu8);
#pragma unroll
        for (int s = 0; s < NS; ++s) {
            const double kk = y[s];
            ax[s] += kk * dx[s];
            ay[s] += kk * dy[s];
            az[s] += kk * dz[s];
        }
    }
    if (B > 0) {
        const int ij = psc == 1 ? 3 * j : j;  // [N][3] in global memory, [3][N] when staged
        const double ix = ind_base[ij], iy = ind_base[ij + psc], iz = ind_base[ij + 2 * psc];
#pragma unroll
        for (int s = 0; s < NS; ++s) {
            ax[s] -= ix;
            ay[s] -= iy;
            az[s] -= iz;
        }
    }
    if (flag) {  // rare: exact guard order of table_acceleration (force_model.hpp:57-69)
#pragma unroll
        for (int s = 0; s < NS; ++s) {
            if (!on[s]) continue;
            int fail = (rx[s] * rx[s] + ry[s] * ry[s] + rz[s] * rz[s] > 0.0) ? -1 : 0;
            for (int b = 0; b < B && fail < 0; ++b) {
                const double dx = bp[(3 * b) * psc] - rx[s], dy = bp[(3 * b + 1) * psc] - ry[s],
                             dz = bp[(3 * b + 2) * psc] - rz[s];
                if (sqrt(dx * dx + dy * dy + dz * dz) < fd.floor_km) fail = 1 + b;
            }
            if (fail >= 0) atomicMin(&sing_key[h * HS + s0 + s], j * (B + 1) + fail);
        }
    }
#pragma unroll
    for (int s = 0; s < NS; ++s) {
        fb[f2(j, 0, s0 + s)] = on[s] ? ybuf[y2(j, h, 3, s0 + s)] : 0.0;
        fb[f2(j, 1, s0 + s)] = on[s] ? ybuf[y2(j, h, 4, s0 + s)] : 0.0;
        fb[f2(j, 2, s0 + s)] = on[s] ? ybuf[y2(j, h, 5, s0 + s)] : 0.0;
        fb[f2(j, 3, s0 + s)] = on[s] ? ax[s] : 0.0;
        fb[f2(j, 4, s0 + s)] = on[s] ? ay[s] : 0.0;
        fb[f2(j, 5, s0 + s)] = on[s] ? az[s] : 0.0;
    }
}

/// Folded force (fold = 1, Newtonian): one thread evaluates the mirrored nodes j and
/// N-1-j (j < N/2) for slots [s0, s0 + NS) — 2 NS independent chains — and writes the
/// folded F directly: s = F_j + F_{N-1-j} at node j, a = F_j - F_{N-1-j} at node N-1-j
/// (no separate fold pass).  Same arithmetic per node as force_half.
template <int NS>
__device__ __forceinline__ void force_pair(const ForceData& fd, const double* ybuf, double* fb, int* sing_key,
                                           const double* pos_base, const double* ind_base, int psj, int psc,
                                           int act_h, int h, int j, int N, int s0) {
    constexpr int C = 2 * NS;  // chain k: node side k / NS (0: j, 1: N-1-j), slot s0 + k % NS
    const int B = fd.n_bodies;
    const int nd[2] = {j, N - 1 - j};
    double rx[C], ry[C], rz[C], ax[C], ay[C], az[C], r2[C], ir[C];
    bool on[C];
    bool flag = false;
#pragma unroll
    for (int k = 0; k < C; ++k) {
        const int n = nd[k / NS], sl = s0 + k % NS;
        on[k] = (act_h >> sl) & 1;
        rx[k] = on[k] ? ybuf[y2(n, h, 0, sl)] : 1.0e8;
        ry[k] = on[k] ? ybuf[y2(n, h, 1, sl)] : 0.0;
        rz[k] = on[k] ? ybuf[y2(n, h, 2, sl)] : 0.0;
        r2[k] = rx[k] * rx[k] + ry[k] * ry[k] + rz[k] * rz[k];
        flag |= !(r2[k] > 0.0);
    }
#pragma unroll
    for (int k = 0; k < C; ++k) ir[k] = rsqrt_newton(r2[k], rsqrt_newton(r2[k], rsqrt_seed(r2[k])));
#pragma unroll
    for (int k = 0; k < C; ++k) {
        const double sc = -fd.central_mu * (ir[k] * ir[k] * ir[k]);
        ax[k] = sc * rx[k];
        ay[k] = sc * ry[k];
        az[k] = sc * rz[k];
    }
    const double* bp0 = pos_base + static_cast<size_t>(nd[0]) * psj;
    const double* bp1 = pos_base + static_cast<size_t>(nd[1]) * psj;
#pragma unroll(kForceUnroll)
    for (int b = 0; b < B; ++b) {
        const double mu8 = 0.125 * __ldg(fd.body_mu + b);
        const double q0x = bp0[(3 * b) * psc], q0y = bp0[(3 * b + 1) * psc], q0z = bp0[(3 * b + 2) * psc];
        const double q1x = bp1[(3 * b) * psc], q1y = bp1[(3 * b + 1) * psc], q1z = bp1[(3 * b + 2) * psc];
        double dx[C], dy[C], dz[C], d2[C], y[C];
#pragma unroll
        for (int k = 0; k < C; ++k) {
            dx[k] = (k < NS ? q0x : q1x) - rx[k];
            dy[k] = (k < NS ? q0y : q1y) - ry[k];
            dz[k] = (k < NS ? q0z : q1z) - rz[k];
            d2[k] = dx[k] * dx[k] + dy[k] * dy[k] + dz[k] * dz[k];
            flag |= below_bits(d2[k], fd.floor2_hi_bits);
        }
#pragma unroll
        for (int k = 0; k < C; ++k) y[k] = body_mu_ir3(d2[k], mu8);
#pragma unroll
        for (int k = 0; k < C; ++k) {
            const double kk = y[k];
            ax[k] += kk * dx[k];
            ay[k] += kk * dy[k];
            az[k] += kk * dz[k];
        }
    }
    if (B > 0) {
#pragma unroll
        for (int side = 0; side < 2; ++side) {
            const int n = nd[side];
            const int ij = psc == 1 ? 3 * n : n;  // [N][3] in global memory, [3][N] when staged
            const double ix = ind_base[ij], iy = ind_base[ij + psc], iz = ind_base[ij + 2 * psc];
#pragma unroll
            for (int k = side * NS; k < (side + 1) * NS; ++k) {
                ax[k] -= ix;
                ay[k] -= iy;
                az[k] -= iz;
            }
        }
    }
    if (flag) {  // rare: exact guard order of table_acceleration (force_model.hpp:57-69)
#pragma unroll
        for (int k = 0; k < C; ++k) {
            if (!on[k]) continue;
            const int n = nd[k / NS], sl = s0 + k % NS;
            const double* bp = k < NS ? bp0 : bp1;
            int fail = (rx[k] * rx[k] + ry[k] * ry[k] + rz[k] * rz[k] > 0.0) ? -1 : 0;
            for (int b = 0; b < B && fail < 0; ++b) {
                const double dx = bp[(3 * b) * psc] - rx[k], dy = bp[(3 * b + 1) * psc] - ry[k],
                             dz = bp[(3 * b + 2) * psc] - rz[k];
                if (sqrt(dx * dx + dy * dy + dz * dz) < fd.floor_km) fail = 1 + b;
            }
            if (fail >= 0) atomicMin(&sing_key[h * HS + sl], n * (B + 1) + fail);
        }
    }
#pragma unroll
    for (int t = 0; t < NS; ++t) {
        const int sl = s0 + t, k0 = t, k1 = NS + t;
        const bool o = on[k0];  // both sides of a slot share its activity
        double lo[6], hi[6];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            lo[c] = o ? ybuf[y2(nd[0], h, 3 + c, sl)] : 0.0;
            hi[c] = o ? ybuf[y2(nd[1], h, 3 + c, sl)] : 0.0;
        }
        lo[3] = o ? ax[k0] : 0.0;
        lo[4] = o ? ay[k0] : 0.0;
        lo[5] = o ? az[k0] : 0.0;
        hi[3] = o ? ax[k1] : 0.0;
        hi[4] = o ? ay[k1] : 0.0;
        hi[5] = o ? az[k1] : 0.0;
#pragma unroll
        for (int c = 0; c < 6; ++c) {
            fb[f2(nd[0], c, sl)] = lo[c] + hi[c];
            fb[f2(nd[1], c, sl)] = lo[c] - hi[c];
        }
    }
}

}  // namespace


/// Group decisions for half h after its epilogue (one warp, lane = slot of the half):
/// pc_solve's stopping rule (err <= tol, it == max_it) and the fault order of the reference
/// (warm-start failure, singularity, divergence); the leader of each group writes its report
/// and frees / retires its slots (free_mask / retire_mask of the half).
/// decide_half for singleton groups (independent mode, gmax == 1): each lane decides its
/// own slot — no cross-lane scan or warp sync (a lane rewrites only its own group record),
/// one combined mask reduction; same stopping rule, fault order and reports.
__device__ __forceinline__ void decide_single(const SegArgs& a, WsState& st, int h, int lane, int B) {
    const int s = lane, t = h * HS + s;
    unsigned bits = 0;  // bit t: slot freed; bit 8 + t: outputs to retire
    if (s < HS && ((st.act_word[h] >> t) & 1)) {
        const int lg = st.slot_grp[t];
        const int gid = st.grp_id[lg];
        const long long e2b = static_cast<long long>(st.slot_err[t]);
        const double gerr2 = __longlong_as_double(e2b);
        const int sk = st.sing_key[t], nk = st.nf_key[t];
        GroupFault* fl = a.faults + gid;
        bool retire = false, ok = false, conv = false;
        int it = st.grp_iter[lg];
        if (((st.new_mask[h] >> t) & 1) && st.warm_key[t] != INT_MAX) {
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
            if (sk != INT_MAX) {
                fl->status = FAULT_SINGULARITY;
                fl->iteration = it;
                fl->node = sk / (B + 1);
                fl->body = sk % (B + 1) - 1;
                fl->trajectory = st.slot_member[t];
                fl->value = st.sing_val[t];
                retire = true;
            } else if (nk != INT_MAX) {
                const long long key = static_cast<long long>(nk >> 3) * 6 + (nk & 7);
                fl->status = FAULT_DIVERGENCE;
                fl->iteration = it;
                fl->node = key / 6;
                fl->column = key % 6;
                retire = true;
            } else {
                if (a.rep_hist) a.rep_hist[static_cast<size_t>(gid) * a.hist_stride + (it - 1)] = sqrt(gerr2);
                const bool le_tol = PSWARM_ABLATE == 0 &&
                    (e2b <= __double_as_longlong(a.tol2_lo)
                         ? true
                         : (e2b > __double_as_longlong(a.tol2_hi) ? false : sqrt(gerr2) <= a.tol));
                if (le_tol && it >= st.grp_floor[lg]) {
                    retire = ok = conv = true;
                } else if (it >= st.grp_cap[lg]) {
                    retire = ok = true;
                }
            }
        }
        if (a.traj_ns && traj_budget_spent(a, st.slot_traj[t], st.grp_t0[lg], retire)) {
            fl->status = FAULT_TIMEOUT;  // own budget spent before the next force evaluation
            fl->iteration = it;
            retire = true;
        }
        if (retire) {
            a.rep_iter[gid] = it;
            a.rep_err[gid] = sqrt(gerr2);
            a.rep_conv[gid] = conv ? 1 : 0;
            bits = (1u << t) | (ok ? (1u << (8 + t)) : 0u);
            st.grp_id[lg] = -1;
        }
    }
    bits = __reduce_or_sync(0xffffffffu, bits);
    if (lane == 0) {
        st.free_mask[h] = static_cast<int>(bits & 0xffu);
        st.retire_mask[h] = static_cast<int>(bits >> 8);
    }
    if (s < HS) {  // reset this half's accumulators for its next iteration
        st.slot_err[t] = 0ull;
        st.sing_key[t] = INT_MAX;
        st.nf_key[t] = INT_MAX;
    }
}

__device__ __forceinline__ void decide_half(const SegArgs& a, WsState& st, int h, int lane, int B) {
    if (a.gmax == 1 && a.fast_decide) {
        decide_single(a, st, h, lane, B);
        return;
    }
    const int am = st.act_word[h];
    const int s = lane, t = h * HS + s;
    const bool act_t = s < HS && ((am >> t) & 1);
    const int my_grp = act_t ? st.slot_grp[t] : -1;
    const int my_mbr = act_t ? st.slot_member[t] : 0;
    const double my_e2 = act_t ? __longlong_as_double(static_cast<long long>(st.slot_err[t])) : 0.0;
    const int my_sk = act_t ? st.sing_key[t] : INT_MAX;
    const int my_nk = act_t ? st.nf_key[t] : INT_MAX;
    const int my_wk = (act_t && ((st.new_mask[h] >> t) & 1)) ? st.warm_key[t] : INT_MAX;
    const int my_tr = act_t ? st.slot_traj[t] : INT_MAX;
    const int lg = my_grp;
    const int gid = act_t ? st.grp_id[lg] : -1;
    const int size = act_t ? st.grp_size[lg] : 1;
    int it = act_t ? st.grp_iter[lg] : 0;
    bool leader = act_t;
    double gerr2 = 0.0;
    long long sing_s = LLONG_MAX, nf_best = LLONG_MAX;
    int sing_t = -1, warm_t = -1, warm_tr = INT_MAX, members = 0;
    if (a.gmax == 1 && act_t) {  // singleton groups (independent mode): no cross-lane scan
        members = 1 << t;
        gerr2 = my_e2;
        if (my_wk != INT_MAX) warm_t = t;
        if (my_sk != INT_MAX) {
            sing_s = my_sk / (B + 1);
            sing_t = t;
        }
        if (my_nk != INT_MAX) nf_best = static_cast<long long>(my_nk >> 3) * 6 + (my_nk & 7);
    }
#pragma unroll
    for (int u = 0; u < (a.gmax == 1 ? 0 : HS); ++u) {
        const int ug = __shfl_sync(0xffffffffu, my_grp, u);
        const int um = __shfl_sync(0xffffffffu, my_mbr, u);
        const double ue = __shfl_sync(0xffffffffu, my_e2, u);
        const int usk = __shfl_sync(0xffffffffu, my_sk, u);
        const int unk = __shfl_sync(0xffffffffu, my_nk, u);
        const int uwk = __shfl_sync(0xffffffffu, my_wk, u);
        const int utr = __shfl_sync(0xffffffffu, my_tr, u);
        if (!act_t || ug != lg) continue;
        const int ut = h * HS + u;
        if (u < s) leader = false;
        members |= 1 << ut;
        gerr2 = fmax(gerr2, ue);
        if (uwk != INT_MAX && utr < warm_tr) {
            warm_tr = utr;
            warm_t = ut;
        }
        if (usk != INT_MAX) {
            const long long smp = static_cast<long long>(usk / (B + 1)) * size + um;
            if (smp < sing_s) {
                sing_s = smp;
                sing_t = ut;
            }
        }
        if (unk != INT_MAX) {
            const long long key = static_cast<long long>(unk >> 3) * (6LL * size) +
                                  static_cast<long long>(unk & 7) * size + um;
            nf_best = min(nf_best, key);
        }
    }
    __syncwarp();  // every lane has read the slot / group records the leader rewrites
    int free_bits = 0, retire_bits = 0;
    if (leader) {
        // sqrt only where the value is needed (history, retire) or the squared test
        // is within rounding of tol^2 (tol2_lo/hi carry a 1e-13 relative margin)
        auto gerr_of = [&] { return sqrt(gerr2); };
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
                if (a.rep_hist) a.rep_hist[static_cast<size_t>(gid) * a.hist_stride + (it - 1)] = gerr_of();
                // squared-error bands as integer compares of the IEEE bits (non-negative doubles
                // order like integers; NaN sorts above every finite band): off the FP64 pipe
                const long long e2b = __double_as_longlong(gerr2);
                const bool le_tol = PSWARM_ABLATE == 0 &&  // ablation builds: fixed max_it work
                    (e2b <= __double_as_longlong(a.tol2_lo)
                         ? true
                         : (e2b > __double_as_longlong(a.tol2_hi) ? false : gerr_of() <= a.tol));
                if (le_tol && it >= st.grp_floor[lg]) {
                    retire = ok = conv = true;
                } else if (it >= st.grp_cap[lg]) {
                    retire = ok = true;
                }
            }
        }
        if (a.traj_ns && traj_budget_spent(a, my_tr, st.grp_t0[lg], retire)) {  // singleton groups only
            fl->status = FAULT_TIMEOUT;
            fl->iteration = it;
            retire = true;
        }
        if (retire) {
            a.rep_iter[gid] = it;
            a.rep_err[gid] = gerr_of();
            a.rep_conv[gid] = conv ? 1 : 0;
            free_bits = members;
            retire_bits = ok ? members : 0;
            st.grp_id[lg] = -1;
        }
    }
    free_bits = __reduce_or_sync(0xffffffffu, static_cast<unsigned>(free_bits));
    retire_bits = __reduce_or_sync(0xffffffffu, static_cast<unsigned>(retire_bits));
    if (lane == 0) {
        st.free_mask[h] = free_bits;
        st.retire_mask[h] = retire_bits;
    }
    if (s < HS) {  // reset this half's accumulators for its next iteration
        st.slot_err[t] = 0ull;
        st.sing_key[t] = INT_MAX;
        st.nf_key[t] = INT_MAX;
    }
}

template <int MAIN, int XMW, bool STAGE, bool REL, bool FOLD>
__global__ void __launch_bounds__(WS_THREADS, PSWARM_MIN_BLOCKS) k_pc_ws(const SegArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int N = a.N, B = a.fd.n_bodies;
    const int xrows = a.xrows;
    const int half = N / 2;
    const WsLayout L = ws_layout(N, a.nkp, xrows, B, STAGE ? 1 : 0, FOLD ? 1 : 0, REL);
    double* ybuf = reinterpret_cast<double*>(smem_raw + L.ybuf);
    const size_t fb_bytes = L.fbuf1 - L.fbuf0;
    double* fb0 = reinterpret_cast<double*>(smem_raw + L.fbuf0);
    double* xstage = reinterpret_cast<double*>(smem_raw + L.xstage);
    double* anc = reinterpret_cast<double*>(smem_raw + L.anchor);
    double* b0part = reinterpret_cast<double*>(smem_raw + L.b0part);
    double* eph = reinterpret_cast<double*>(smem_raw + L.eph);
    WsState& st = *reinterpret_cast<WsState*>(smem_raw + L.state);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int KP = 8 * a.nkp;
    // node rows only (b0 comes from the FP group's anchor GEMV); folded: row pairs
    const int mtiles = FOLD ? (half + 7) / 8 : (N + 7) / 8;
    // folded with a spare pair row (N/2 % 8 != 0): pair row N/2 of the packed operator is the
    // anchor row, so the DMMA stream forms b0 and the FP group's GEMV + B_h barrier drop out
    const bool b0mma = FOLD && (half & 7) != 0 && a.b0_mma;
    const bool prof = a.phase_cycles != nullptr;
    const bool stamp = tid == 0 || tid == MMA_THREADS;
    // phase counters live in shared memory (no registers / local memory on the hot path)
    __shared__ long long s_pc[PHASES], s_prev[2];
    const int grp_ = tid < MMA_THREADS ? 0 : 1;
    if (tid < PHASES) s_pc[tid] = 0;
    if (stamp) s_prev[grp_] = clock64();
    HalfPlan hp;
    hp.main = MAIN;
    hp.mb = MAIN * MMA_WARPS;
    hp.extras = (mtiles - hp.mb) * 3;

    // ---- per-launch staging of the frozen ephemeris through the TMA unit: bulk copies of the
    //      segment's node table (k_ephemeris wrote it in the staged layout) completing on an
    //      mbarrier, overlapped with the rest of the prologue
    constexpr bool kStaged = STAGE;
    if (kStaged && tid == 0) {
        mbar_init(&st.stage_bar, 1);
        bulk_stage(eph, REL ? a.fd.rel_tab : a.fd.eph_t, static_cast<unsigned>(sizeof(double) * eph_stage_doubles(N, B, REL)),
                   &st.stage_bar);
    }
    const int fb_doubles = (FOLD ? ws_fold_ksteps(N, a.nkp) : 2 * a.nkp) * FKS;
    for (int i = tid; i < 2 * fb_doubles; i += WS_THREADS) fb0[i] = 0.0;  // both halves (contiguous)
    if (FOLD) {  // anchor weights of the folded F layout (s at k, a at p >= N/2)
        for (int k = tid; k < KP; k += WS_THREADS) anc[k] = k < N ? a.anc_fold[k] : 0.0;
    } else {  // anchor_op row (pc_matrices.hpp:98-100) = row N of the packed operator
        const double* up = reinterpret_cast<const double*>(a.upack);
        const int amt = N >> 3, ag = N & 7;
        for (int k = tid; k < KP; k += WS_THREADS)
            anc[k] = k < N ? up[2 * ((static_cast<size_t>(amt) * a.nkp + (k >> 3)) * 32 + ag * 4 + (k & 3)) + ((k >> 2) & 1)]
                           : 0.0;
    }
    // element (node j, body b, coordinate c) at pos_base[j * psj + (3b + c) * psc]: staged
    // node-contiguous, so the force threads (one node each) read conflict-free; unstaged, the
    // node-contiguous global copy when the host passes one (coalesced), else [N][B][3]
    const bool nodec = STAGE || a.fd.eph_t != nullptr;
    const double* pos_base = STAGE ? eph : nodec ? a.fd.eph_t : a.fd.body_pos;
    const double* ind_base = STAGE ? eph + 3 * B * eph_ld(N) : nodec ? a.fd.eph_t + 3 * B * eph_ld(N) : a.fd.indirect;
    const int psj = nodec ? 1 : 3 * B, psc = nodec ? eph_ld(N) : 1;
    const double* rel_base = STAGE ? eph : a.fd.rel_tab;  // relativistic node table
    if (tid == 0) {
        for (int t = 0; t < SLOTS; ++t) {
            st.slot_traj[t] = -1;
            st.grp_id[t] = -1;
            st.sing_key[t] = INT_MAX;
            st.nf_key[t] = INT_MAX;
            st.slot_err[t] = 0ull;
        }
        st.act_word[0] = st.act_word[1] = 0;
        st.new_mask[0] = st.new_mask[1] = 0;
        st.half_active[0] = st.half_active[1] = 0;
        st.queue_done = 0;
        st.timeout = 0;
        st.exit_flag = 0;
    }
    __syncthreads();
    if (kStaged) mbar_wait(&st.stage_bar, 0);

    if (warp < MMA_WARPS) {
        // ============================================================ MMA group
        const int g = lane >> 2, q = lane & 3;
        for (int h = 0;; h ^= 1) {
            bar_sync(BAR_F0 + h, WS_THREADS);
            WS_PHASE(0);
            if (st.exit_flag) break;
            if (st.half_active[h]) {
                if constexpr (FOLD) {
                    // full pair tiles < nfull strided over the warps; the leftover tiles' 3 n-tiles
                    // each go to the warps that hold one full tile fewer (rows staged, below)
                    const int nxt = xrows >> 3, nfull = mtiles - nxt;
                    const int xk = (warp - nfull % MMA_WARPS + MMA_WARPS) % MMA_WARPS;
                    const int xt = (XMW > 0 && xk < 3 * nxt) ? nfull + xk / 3 : -1, xp = xk % 3;  // XMW: extras
                    double facc[MAIN][3][2][2], fxacc[2][2];
                    gemm_half_fold<MAIN>(a.upack_fold, a.nkp_fold, half,
                                         reinterpret_cast<const double*>(smem_raw + L.fbuf0 + h * fb_bytes), nfull,
                                         warp, lane, xt, xp, facc, fxacc);
                    WS_PHASE(1);
                    // extra unit -> stage its unfolded raw sums now (both mirrored rows); the light
                    // warps add omega2 / b0 and finalise them after the b0 barrier, concurrently
                    // with the other warps' main epilogue
                    double* xs_lo = xstage + (2 * h) * xrows * HC;
                    double* xs_hi = xs_lo + xrows * HC;
                    if (xt >= 0) {
                        const int j = xt * 8 + g;
                        if (j < half) {
#pragma unroll
                            for (int e = 0; e < 2; ++e) {
                                const int o = (j - nfull * 8) * HC + q * 6 + 2 * xp + e;
                                xs_lo[o] = fxacc[0][e] + fxacc[1][e];
                                xs_hi[o] = fxacc[0][e] - fxacc[1][e];
                            }
                        }
                    }
                    if (b0mma) {  // b0 = (omega2 anchor.F + 2 y0) / 2 from the anchor pair row
                        const int at = half >> 3;
                        if (g == (half & 7)) {
                            const double w2a = a.omega2;
#pragma unroll
                            for (int i = 0; i < MAIN; ++i)
                                if (warp + i * MMA_WARPS == at && at < nfull)
#pragma unroll
                                    for (int p = 0; p < 3; ++p)
#pragma unroll
                                        for (int e = 0; e < 2; ++e)
                                            st.b0h[h][p * 8 + 2 * q + e] =
                                                0.5 * fma(w2a, facc[i][p][0][e] + facc[i][p][1][e],
                                                          2.0 * st.y0[h * HS + q][2 * p + e]);
                            if (xt == at)
#pragma unroll
                                for (int e = 0; e < 2; ++e)
                                    st.b0h[h][xp * 8 + 2 * q + e] = 0.5 * fma(w2a, fxacc[0][e] + fxacc[1][e],
                                                                               2.0 * st.y0[h * HS + q][2 * xp + e]);
                        }
                        bar_sync(BAR_MMA, MMA_THREADS);
                    } else if (nxt > 0) {
                        // the FP group formed b0 before releasing F_h (ordered by the F barrier);
                        // the barrier orders the raw staging writes before the light warps' reads
                        bar_sync(BAR_MMA, MMA_THREADS);
                    }
                    WS_PHASE(3);
                    // unfold: Y_j = acc_sum + acc_diff, Y_{N-1-j} = acc_sum - acc_diff (the 1/2 sits in
                    // the packed operators), then the same epilogue as the dense path for both rows
                    const int act_h = (st.act_word[h] >> (h * HS)) & 0xF;
                    const double* b0 = st.b0h[h];
                    const double w2 = a.omega2;
                    double bn = 0.0, bd = 1.0;
                    int nf = INT_MAX;
#pragma unroll
                    for (int i = 0; i < MAIN; ++i) {
                        const int j = (warp + i * MMA_WARPS) * 8 + g, jm = N - 1 - j;
                        if (warp + i * MMA_WARPS >= nfull || j >= half || !((act_h >> q) & 1)) continue;
                        double ylo[6], yhi[6], olo[6], ohi[6];
#pragma unroll
                        for (int p = 0; p < 3; ++p)
#pragma unroll
                            for (int e = 0; e < 2; ++e) {
                                const int c = 2 * p + e;
                                const double bb = b0[p * 8 + 2 * q + e];
                                ylo[c] = fma(w2, facc[i][p][0][e] + facc[i][p][1][e], bb);
                                yhi[c] = fma(w2, facc[i][p][0][e] - facc[i][p][1][e], bb);
                                olo[c] = ybuf[y2(j, h, c, q)];
                                ohi[c] = ybuf[y2(jm, h, c, q)];
                            }
                        update_sample(ylo, olo, j, a.error_mode, bn, bd, nf);
                        update_sample(yhi, ohi, jm, a.error_mode, bn, bd, nf);
#pragma unroll
                        for (int c = 0; c < 6; ++c) {
                            ybuf[y2(j, h, c, q)] = ylo[c];
                            ybuf[y2(jm, h, c, q)] = yhi[c];
                        }
                    }
                    double e2 = bn / bd;
#pragma unroll
                    for (int off = 4; off < 32; off <<= 1) {
                        e2 = fmax(e2, __shfl_xor_sync(0xffffffffu, e2, off));
                        nf = min(nf, __shfl_xor_sync(0xffffffffu, nf, off));
                    }
                    if (g == 0 && ((act_h >> q) & 1)) {
                        atomicMax(&st.slot_err[h * HS + q], static_cast<unsigned long long>(__double_as_longlong(e2)));
                        if (nf != INT_MAX) atomicMin(&st.nf_key[h * HS + q], nf);
                    }
                    if (nxt > 0) {  // staged rows (pair rows of the leftover tiles and mirrors): light warps
                        const int light = MMA_WARPS - (nfull % MMA_WARPS + 3 * nxt);  // warps without extras
                        const int lt = tid - (MMA_WARPS - light) * 32;
                        if (lt >= 0) {
                            const int xv = min(xrows, half - nfull * 8);  // valid pair rows
                            for (int i = lt; i < xv * HS * 2; i += light * 32) {
                                const int mir = i / (xv * HS), ii = i - mir * xv * HS;
                                const int r = ii >> 2, s = ii & 3;
                                const int jp = nfull * 8 + r, j = mir ? N - 1 - jp : jp;
                                if (!((act_h >> s) & 1)) continue;
                                const double* xs = mir ? xs_hi : xs_lo;
                                double yn[6], yo[6];
#pragma unroll
                                for (int c = 0; c < 6; ++c) {
                                    yn[c] = fma(w2, xs[r * HC + s * 6 + c], b0[(c >> 1) * 8 + 2 * s + (c & 1)]);
                                    yo[c] = ybuf[y2(j, h, c, s)];
                                }
                                double sbn = 0.0, sbd = 1.0;
                                int snf = INT_MAX;
                                update_sample(yn, yo, j, a.error_mode, sbn, sbd, snf);
#pragma unroll
                                for (int c = 0; c < 6; ++c) ybuf[y2(j, h, c, s)] = yn[c];
                                atomicMax(&st.slot_err[h * HS + s],
                                          static_cast<unsigned long long>(__double_as_longlong(sbn / sbd)));
                                if (snf != INT_MAX) atomicMin(&st.nf_key[h * HS + s], snf);
                            }
                        }
                    }
                    // decisions of half h here, not in the FP group: the MMA group has slack once
                    // its DMMA stream is halved, and the FP group's warps issue ~3x slower while
                    // DMMAs stream (the decisions sat on the FP group's critical chain)
                    WS_PHASE(2);
                    bar_sync(BAR_MMA, MMA_THREADS);  // every warp's slot_err / nf_key update is in
                    WS_PHASE(11);
                    WS_PHASE(12);
                    if (warp == 0) decide_half(a, st, h, lane, B);
                    WS_PHASE(13);
                } else {
                double acc[MAIN][3][2], xacc[XMW][2];
#if PSWARM_ABLATE == 3  // diagnostic: no DMMA
                for (int i = 0; i < MAIN; ++i)
                    for (int p = 0; p < 3; ++p) acc[i][p][0] = acc[i][p][1] = 0.0;
                for (int x = 0; x < XMW; ++x) xacc[x][0] = xacc[x][1] = 0.0;
                if (false)
#endif
                gemm_half<MAIN, XMW>(a.upack, a.nkp, reinterpret_cast<const double*>(smem_raw + L.fbuf0 + h * fb_bytes),
                                     hp, warp, lane, acc, xacc);
                WS_PHASE(1);
                bar_sync(BAR_B0 + h, WS_THREADS);  // b0 of half h (FP group)
                WS_PHASE(3);
                // epilogue of this warp's rows: + b0/2 (pc_matrices.hpp:145; b0 was formed by
                // the FP group with the force), finite check, error vs the previous iterate.
                // No barrier inside the MMA group: a warp that finishes early runs its
                // epilogue while its SMSP partner still issues DMMAs.
                const int act_h = (st.act_word[h] >> (h * HS)) & 0xF;
                const double* b0 = st.b0h[h];
                const double w2 = a.omega2;  // F holds [v, a]; the segment's step scale applies here
                double bn = 0.0, bd = 1.0;
                int nf = INT_MAX;
#pragma unroll
                for (int i = 0; i < MAIN; ++i) {
                    const int j = (warp * MAIN + i) * 8 + g;
                    if (j >= N || !((act_h >> q) & 1) || PSWARM_ABLATE == 1) continue;  // 1: diagnostic
                    double yn[6], yo[6];
#pragma unroll
                    for (int p = 0; p < 3; ++p)
#pragma unroll
                        for (int e = 0; e < 2; ++e) {
                            const int c = 2 * p + e;
                            yo[c] = ybuf[y2(j, h, c, q)];
                            yn[c] = fma(w2, acc[i][p][e], b0[p * 8 + 2 * q + e]);
                        }
                    update_sample(yn, yo, j, a.error_mode, bn, bd, nf);
#pragma unroll
                    for (int c = 0; c < 6; ++c) ybuf[y2(j, h, c, q)] = yn[c];
                }
#if PSWARM_ABLATE == 1  // keep the skipped rows' DMMAs live
                {
                    double t = 0.0;
#pragma unroll
                    for (int i = 0; i < MAIN; ++i)
#pragma unroll
                        for (int p = 0; p < 3; ++p) t += acc[i][p][0] + acc[i][p][1];
                    if (t == 12345.678) ybuf[0] = t;
                }
#endif
                double* xs = xstage + h * xrows * HC;
#pragma unroll
                for (int x = 0; x < XMW; ++x) {  // extra tiles -> stage (components spread over warps)
                    const int ex = warp + x * MMA_WARPS;
                    if (ex >= hp.extras) continue;
                    const int j = (hp.mb + ex / 3) * 8 + g, p = ex % 3;
                    if (j >= N) continue;
#pragma unroll
                    for (int e = 0; e < 2; ++e)
                        xs[(j - hp.mb * 8) * HC + q * 6 + 2 * p + e] = fma(w2, xacc[x][e], b0[p * 8 + 2 * q + e]);
                }
                double e2 = bn / bd;
#pragma unroll
                for (int off = 4; off < 32; off <<= 1) {
                    e2 = fmax(e2, __shfl_xor_sync(0xffffffffu, e2, off));
                    nf = min(nf, __shfl_xor_sync(0xffffffffu, nf, off));
                }
                if (g == 0 && ((act_h >> q) & 1)) {
                    atomicMax(&st.slot_err[h * HS + q], static_cast<unsigned long long>(__double_as_longlong(e2)));
                    if (nf != INT_MAX) atomicMin(&st.nf_key[h * HS + q], nf);
                }
                }
                WS_PHASE(2);
            } else {
                if (FOLD && tid == 0) st.free_mask[h] = st.retire_mask[h] = 0;  // no decisions ran
                if (!FOLD) bar_sync(BAR_B0 + h, WS_THREADS);  // keep the B_h generations paired
            }
            bar_arrive(BAR_Y0 + h, WS_THREADS);  // bar.arrive/bar.sync order smem among participants
        }
    } else {
        // ============================================================= FP group
        const int ft = tid - MMA_THREADS;  // 0..255
        const int fw = ft >> 5;
        bool first[2] = {true, true};
        for (int h = 0;; h ^= 1) {
            if (!first[h]) bar_sync(BAR_Y0 + h, WS_THREADS);  // epilogue of half h done
            WS_PHASE(4);
            // ---- staged rows of half h (node rows whose components sit in several MMA warps)
            if (!FOLD && !first[h] && xrows > 0 && st.half_active[h]) {  // (folded: the MMA group's)
                const int act_h = (st.act_word[h] >> (h * HS)) & 0xF;
                const double* xs = xstage + h * xrows * HC;
                for (int i = ft; i < xrows * HS; i += FP_THREADS) {
                    const int r = i >> 2, s = i & 3, j = MAIN * MMA_WARPS * 8 + r;
                    if (!((act_h >> s) & 1)) continue;
                    double yn[6], yo[6];
#pragma unroll
                    for (int c = 0; c < 6; ++c) {
                        yn[c] = xs[r * HC + s * 6 + c];
                        yo[c] = ybuf[y2(j, h, c, s)];
                    }
                    double sbn = 0.0, sbd = 1.0;
                    int snf = INT_MAX;
                    update_sample(yn, yo, j, a.error_mode, sbn, sbd, snf);
#pragma unroll
                    for (int c = 0; c < 6; ++c) ybuf[y2(j, h, c, s)] = yn[c];
                    atomicMax(&st.slot_err[h * HS + s], static_cast<unsigned long long>(__double_as_longlong(sbn / sbd)));
                    if (snf != INT_MAX) atomicMin(&st.nf_key[h * HS + s], snf);
                }
                if (xrows * HS > 32)
                    bar_sync(BAR_FP, FP_THREADS);
                else
                    __syncwarp();  // warp 0 staged every row and also takes the decisions
            }
            WS_PHASE(10);
            // ---- decisions for half h (warp 0 of the FP group; folded: done by the MMA group)
            if (!FOLD && !first[h] && fw == 0) decide_half(a, st, h, lane, B);
            bar_sync(BAR_FP, FP_THREADS);
            WS_PHASE(5);
            // ---- retire outputs of half h
            if (!first[h] && st.retire_mask[h]) {
                const int retire = st.retire_mask[h];
                const int j_begin = a.seg == 0 ? 0 : 1;
                for (int i = ft; i < N * HS; i += FP_THREADS) {
                    const int j = i >> 2, s = i & 3, t = h * HS + s;
                    if (!((retire >> t) & 1)) continue;
                    const size_t tr = static_cast<size_t>(st.slot_traj[t]);
                    if (a.samples && j >= j_begin) {
                        double* o = a.samples + (tr * a.R + a.row0 + j) * 6;
#pragma unroll
                        for (int c = 0; c < 6; ++c) o[c] = ybuf[y2(j, h, c, s)];
                    }
                    if (a.hot)
                        for (int c = 0; c < 6; ++c) hot_retire_node(a.hot + (tr * N + j) * 6, c, ybuf[y2(j, h, c, s)]);
                    if (a.blk)  // wide-group round: the full iterate (resume source)
                        for (int c = 0; c < 6; ++c) a.blk[(tr * N + j) * 6 + c] = ybuf[y2(j, h, c, s)];
                    if (j == N - 1) {
#pragma unroll
                        for (int c = 0; c < 6; ++c) a.state_out[tr * 6 + c] = ybuf[y2(j, h, c, s)];
                    }
                }
                bar_sync(BAR_FP, FP_THREADS);  // slot_traj is rewritten by the claim below
            }
            // ---- free + claim into half h (thread 0 of the FP group)
            if (ft == 0) {
                int am = st.act_word[0] | st.act_word[1];
                if (!first[h]) {
                    const int fm = st.free_mask[h];
                    am &= ~fm;
                    for (int t = 0; t < SLOTS; ++t)
                        if ((fm >> t) & 1) st.slot_traj[t] = -1;
                }
                int new_mask = 0;
                const int hmask = 0xF << (h * HS);
                const int free_h = HS - __popc(static_cast<unsigned>(am & hmask));
                if (!st.queue_done && free_h >= a.gmax) {
                    const int k = free_h / a.gmax;
                    const int g0 = atomicAdd(a.queue, k);
                    const int g1 = min(g0 + k, a.P);
                    if (g0 + k >= a.P) st.queue_done = 1;
                    for (int gi = g0; gi < g1; ++gi) {
                        int lg = h * HS;  // group records of half h (a group never spans halves)
                        while (st.grp_id[lg] >= 0) ++lg;
                        int off, size, gid;
                        claim_group(a, gi, off, size, gid);
                        st.grp_id[lg] = gid;
                        st.grp_size[lg] = size;
                        st.grp_iter[lg] = start_iteration(a, off);
                        st.grp_floor[lg] = claim_floor(a, gid);
                        st.grp_cap[lg] = claim_cap(a, gid);
                        if (a.traj_ns) st.grp_t0[lg] = globaltimer_ns();
                        int t = h * HS;
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
                if (a.deadline_ns != 0ull && globaltimer_ns() > a.deadline_ns) st.timeout = 1;
                st.act_word[h] = am & (0xF << (h * HS));
                st.new_mask[h] = new_mask;
                st.half_active[h] = (am & hmask) != 0;
            }
            bar_sync(BAR_FP, FP_THREADS);
            WS_PHASE(6);
            const int am = st.act_word[0] | st.act_word[1];
            if (st.timeout || (am == 0 && st.queue_done)) {  // done: release the MMA group and leave
                if (ft == 0) {
                    if (st.timeout)
                        for (int lg = 0; lg < SLOTS; ++lg) {
                            const int gi = st.grp_id[lg];
                            if (gi < 0) continue;
                            a.faults[gi].status = FAULT_TIMEOUT;
                            a.faults[gi].iteration = st.grp_iter[lg];
                            a.rep_iter[gi] = st.grp_iter[lg];
                            a.rep_conv[gi] = 0;
                        }
                    st.exit_flag = 1;
                }
                bar_sync(BAR_FP, FP_THREADS);
                bar_arrive(BAR_F0 + h, WS_THREADS);
                // the MMA group still finishes the other half it was released for:
                // consume its Y arrive so no named barrier is left half-open
                if (!first[h ^ 1]) bar_sync(BAR_Y0 + (h ^ 1), WS_THREADS);
                break;
            }
            // ---- load + warm start of new slots in half h
            const int new_mask = st.new_mask[h];
            if (new_mask) {
                for (int i = ft; i < SLOTS * 6; i += FP_THREADS) {
                    const int s = i / 6, c = i % 6;
                    if ((new_mask >> s) & 1) st.y0[s][c] = a.state_in[static_cast<size_t>(st.slot_traj[s]) * 6 + c];
                }
                bar_sync(BAR_FP, FP_THREADS);
                for (int i = ft; i < N * HS; i += FP_THREADS) {
                    const int j = i >> 2, s = i & 3, t = h * HS + s;
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
                            hot_start_node(a.hot + (static_cast<size_t>(st.slot_traj[t]) * N + j) * 6, a.hot_apply,
                                           ro, vo);
                    }
#pragma unroll
                    for (int c = 0; c < 3; ++c) {
                        ybuf[y2(j, h, c, s)] = ro[c];
                        ybuf[y2(j, h, c + 3, s)] = vo[c];
                    }
                }
                bar_sync(BAR_FP, FP_THREADS);
                if (ft < SLOTS && ((new_mask >> ft) & 1) && st.warm_key[ft] != INT_MAX) {
                    const int t = ft, j = st.warm_key[t] / 4;
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
            WS_PHASE(7);
            // ---- force of half h
            const int act_h = (am >> (h * HS)) & 0xF;
#if PSWARM_ABLATE == 2  // diagnostic: no force
            if (false) {
#else
            if (act_h) {
#endif
                // slots per force thread: all FP warps stay busy down to N = 64 (the FP warps only
                // issue in the DMMA stream's gaps, so their count sets the force throughput)
                double* fbh = reinterpret_cast<double*>(smem_raw + L.fbuf0 + h * fb_bytes);
                if constexpr (FOLD && !REL) {  // mirrored node pairs, F folded as it is written
                    if (a.force_ns == 2 || (a.force_ns == 0 && half > FP_THREADS / 4)) {
                        for (int w = ft; w < 2 * half; w += FP_THREADS)
                            force_pair<2>(a.fd, ybuf, fbh, st.sing_key, pos_base, ind_base, psj, psc, act_h, h,
                                          w % half, N, (w / half) * 2);
                    } else {
                        for (int w = ft; w < 4 * half; w += FP_THREADS)
                            force_pair<1>(a.fd, ybuf, fbh, st.sing_key, pos_base, ind_base, psj, psc, act_h, h,
                                          w % half, N, w / half);
                    }
                } else if (N > FP_THREADS / 2) {
                    for (int j = ft; j < N; j += FP_THREADS) {
                        if constexpr (REL)
                            force_half_rel<4, !STAGE>(a.fd, rel_base, ybuf, fbh, st.sing_key, act_h, h, j, 0);
                        else
                            force_half<4>(a.fd, ybuf, fbh, st.sing_key, pos_base, ind_base, psj, psc, act_h, h, j, 0);
                    }
                } else if (N > FP_THREADS / 4) {
                    for (int w = ft; w < 2 * N; w += FP_THREADS) {
                        // relativistic: the slot pairs of a node in adjacent lanes (one table row
                        // read per node, broadcast)
                        const int j = REL ? w >> 1 : w % N, s0 = REL ? (w & 1) * 2 : (w / N) * 2;
                        if constexpr (REL)
                            force_half_rel<2, !STAGE>(a.fd, rel_base, ybuf, fbh, st.sing_key, act_h, h, j, s0);
                        else
                            force_half<2>(a.fd, ybuf, fbh, st.sing_key, pos_base, ind_base, psj, psc, act_h, h, j, s0);
                    }
                } else {
                    for (int w = ft; w < 4 * N; w += FP_THREADS) {
                        const int j = REL ? w >> 2 : w % N, s0 = REL ? w & 3 : w / N;
                        if constexpr (REL)
                            force_half_rel<1, !STAGE>(a.fd, rel_base, ybuf, fbh, st.sing_key, act_h, h, j, s0);
                        else
                            force_half<1>(a.fd, ybuf, fbh, st.sing_key, pos_base, ind_base, psj, psc, act_h, h, j, s0);
                    }
                }
            }
            bar_sync(BAR_FP, FP_THREADS);
            WS_PHASE(8);
            if constexpr (FOLD && REL) {  // fold F in place: s_k at position k, a_k = F_k - F_{N-1-k} at N-1-k
                if (act_h) {
                    double* fbh = reinterpret_cast<double*>(smem_raw + L.fbuf0 + h * fb_bytes);
                    for (int col = fw; col < HC; col += FP_WARPS) {  // warp per column, lane per node
                        const int c = 2 * (col >> 3) + (col & 1), sl = (col & 7) >> 1;
                        for (int k = lane; k < half; k += 32) {
                            const int lo = f2(k, c, sl), hi = f2(N - 1 - k, c, sl);
                            const double flo = fbh[lo], fhi = fbh[hi];
                            fbh[lo] = flo + fhi;
                            fbh[hi] = flo - fhi;
                        }
                    }
                }
                bar_sync(BAR_FP, FP_THREADS);
            }
            if (ft < HS && st.sing_key[h * HS + ft] != INT_MAX) {
                const int t = h * HS + ft, key = st.sing_key[t], j = key / (B + 1), chk = key % (B + 1);
                st.sing_val[t] =
                    check_distance(ybuf[y2(j, h, 0, ft)], ybuf[y2(j, h, 1, ft)], ybuf[y2(j, h, 2, ft)], j, chk, a.fd);
            }
            first[h] = false;
            WS_PHASE(10);  // (diagnostic split: fold pass)
            // dense: F_h released before b0, which then overlaps the DMMAs of half h.  Folded:
            // the halved DMMA stream leaves the MMA group slack, so b0 is formed first, while
            // the FP64 pipe is free of DMMAs (it is ~3x slower issued into their gaps)
            if constexpr (!FOLD) bar_arrive(BAR_F0 + h, WS_THREADS);  // F_h ready: the MMA group starts
            // ---- b0 = anchor_op.F + 2 y0 of half h (pc_matrices.hpp:138), overlapped with the
            //      DMMAs of half h: B0_PARTS strided partial dot products per column, summed in a
            //      fixed order; the MMA group waits for it (B_h) only before its epilogue
            if (act_h && !b0mma && PSWARM_ABLATE != 4) {  // 4: diagnostic, no b0
                const double* fbh = reinterpret_cast<const double*>(smem_raw + L.fbuf0 + h * fb_bytes);
                {  // warp fw reads whole 32-double fragments (conflict-free): lane = (col & 7) * 4 + (j & 3)
                    double s0 = 0.0, s1 = 0.0, s2 = 0.0;
                    const int jl = lane & 3;
                    for (int kq = fw; kq < a.nkp * 2; kq += FP_WARPS) {
                        const double w = anc[4 * kq + jl];  // zero past N
                        const double* fq = fbh + kq * FKS + lane;
                        s0 = fma(w, fq[0], s0);
                        s1 = fma(w, fq[32], s1);
                        s2 = fma(w, fq[64], s2);
                    }
#pragma unroll
                    for (int off = 1; off < 4; off <<= 1) {  // sum the 4 nodes of a k-step (lanes ^1, ^2)
                        s0 += __shfl_xor_sync(0xffffffffu, s0, off);
                        s1 += __shfl_xor_sync(0xffffffffu, s1, off);
                        s2 += __shfl_xor_sync(0xffffffffu, s2, off);
                    }
                    if (jl == 0) {
                        const int c8 = lane >> 2;
                        b0part[fw * HC + c8] = s0;
                        b0part[fw * HC + 8 + c8] = s1;
                        b0part[fw * HC + 16 + c8] = s2;
                    }
                }
                bar_sync(BAR_FP, FP_THREADS);
                if (ft < HC) {
                    const int c = 2 * (ft >> 3) + (ft & 1), s = (ft & 7) >> 1;
                    double sum = 0.0;
#pragma unroll
                    for (int part = 0; part < FP_WARPS; ++part) sum += b0part[part * HC + ft];
                    st.b0h[h][ft] = 0.5 * fma(a.omega2, sum, 2.0 * st.y0[h * HS + s][c]);
                }
            }
            WS_PHASE(9);
            if constexpr (FOLD) bar_arrive(BAR_F0 + h, WS_THREADS);
            if (!FOLD) bar_arrive(BAR_B0 + h, WS_THREADS);  // folded: b0 precedes F_h
        }
    }
    if (prof) {
        __syncthreads();
        if (tid == 0) {
            s_pc[PHASES - 1] = 1;
            for (int k = 0; k < PHASES; ++k)
                if (s_pc[k]) atomicAdd(a.phase_cycles + k, static_cast<unsigned long long>(s_pc[k]));
        }
    }
}

// =====================================================================================
// k_pc_uni — unified (non-specialised) folded slot kernel, Newtonian forces.
//
// Same slots, state layout, operators and arithmetic as k_pc_ws<..., FOLD>, but every phase
// runs on all 16 warps over both halves at once: decisions -> retire -> claim -> warm start
// -> force -> b0 -> DMMA + epilogue.  Rationale: DMMA and DFMA share one FP64
// pipe and the FP warps barely issue while a DMMA stream runs, so k_pc_ws's two groups do
// not overlap their FP64 work; the tick is the DMMA phase plus the FP group's latency-bound
// chain.  Here the force runs with twice the warps on an idle pipe, and the DMMA phase
// spreads 2 x 13 pair tiles (N = 200) over 16 warps.
// =====================================================================================

/// The warp's NV pair-tile units (tile[i] of half hh[i]): folded GEMM of gemm_core_fold with
/// a per-unit B-fragment buffer (the two halves have separate F buffers).
template <int NV>
__device__ __forceinline__ void gemm_units_fold(const double2* __restrict__ upf, int nkpf, int half,
                                                const double* const (&fb)[NV], const int (&tile)[NV], int lane,
                                                double (&acc)[NV][3][2][2]) {
#pragma unroll
    for (int i = 0; i < NV; ++i)
#pragma unroll
        for (int p = 0; p < 3; ++p)
#pragma unroll
            for (int u = 0; u < 2; ++u) acc[i][p][u][0] = acc[i][p][u][1] = 0.0;
    const double2* am[NV][2];
#pragma unroll
    for (int i = 0; i < NV; ++i)
#pragma unroll
        for (int u = 0; u < 2; ++u) am[i][u] = upf + (static_cast<size_t>(tile[i]) * 2 + (1 - u)) * nkpf * 32 + lane;
    const int hi_off = (half >> 2) * FKS;  // part 1 (a) sits at positions >= N/2
    struct Pair {
        double2 m[NV][2];
    };
    auto load = [&](int kp, Pair& c) {
#pragma unroll
        for (int i = 0; i < NV; ++i)
#pragma unroll
            for (int u = 0; u < 2; ++u) c.m[i][u] = __ldg(am[i][u] + kp * 32);
    };
    auto compute = [&](int kp, const Pair& c) {
#pragma unroll
        for (int sub = 0; sub < 2; ++sub) {
            const int ks = 2 * kp + sub;
#pragma unroll
            for (int u = 0; u < 2; ++u) {
#pragma unroll
                for (int i = 0; i < NV; ++i) {
                    const double* fk = fb[i] + lane + (u ? 0 : hi_off) + ks * FKS;
                    const double bv[3] = {fk[0], fk[32], fk[64]};
                    const double av = sub ? c.m[i][u].y : c.m[i][u].x;
#pragma unroll
                    for (int p = 0; p < 3; ++p) dmma(acc[i][p][u][0], acc[i][p][u][1], av, bv[p]);
                }
            }
        }
    };
    Pair p0, p1;
    load(0, p0);
    int kp = 0;
    for (; kp + 1 < nkpf; kp += 2) {
        load(kp + 1, p1);
        compute(kp, p0);
        if (kp + 2 < nkpf) load(kp + 2, p0);
        compute(kp + 1, p1);
    }
    if (kp < nkpf) compute(kp, p0);
}

/// Unfold + epilogue of one pair-tile unit of half h (rows j = 8 tile + g and N-1-j):
/// identical arithmetic to k_pc_ws's folded epilogue.
__device__ __forceinline__ void epilogue_unit_fold(const SegArgs& a, WsState& st, double* ybuf,
                                                   const double (&acc)[3][2][2], int h, int tile, int half, int lane) {
    const int g = lane >> 2, q = lane & 3, N = a.N;
    const int act_h = (st.act_word[h] >> (h * HS)) & 0xF;
    const double* b0 = st.b0h[h];
    const double w2 = a.omega2;
    double bn = 0.0, bd = 1.0;
    int nf = INT_MAX;
    const int j = tile * 8 + g, jm = N - 1 - j;
    if (j < half && ((act_h >> q) & 1)) {
        double ylo[6], yhi[6], olo[6], ohi[6];
#pragma unroll
        for (int p = 0; p < 3; ++p)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int c = 2 * p + e;
                const double bb = b0[p * 8 + 2 * q + e];
                ylo[c] = fma(w2, acc[p][0][e] + acc[p][1][e], bb);
                yhi[c] = fma(w2, acc[p][0][e] - acc[p][1][e], bb);
                olo[c] = ybuf[y2(j, h, c, q)];
                ohi[c] = ybuf[y2(jm, h, c, q)];
            }
        update_sample(ylo, olo, j, a.error_mode, bn, bd, nf);
        update_sample(yhi, ohi, jm, a.error_mode, bn, bd, nf);
#pragma unroll
        for (int c = 0; c < 6; ++c) {
            ybuf[y2(j, h, c, q)] = ylo[c];
            ybuf[y2(jm, h, c, q)] = yhi[c];
        }
    }
    double e2 = bn / bd;
#pragma unroll
    for (int off = 4; off < 32; off <<= 1) {
        e2 = fmax(e2, __shfl_xor_sync(0xffffffffu, e2, off));
        nf = min(nf, __shfl_xor_sync(0xffffffffu, nf, off));
    }
    if (g == 0 && ((act_h >> q) & 1)) {
        atomicMax(&st.slot_err[h * HS + q], static_cast<unsigned long long>(__double_as_longlong(e2)));
        if (nf != INT_MAX) atomicMin(&st.nf_key[h * HS + q], nf);
    }
}

#define UNI_PHASE(k)                                  \
    do {                                              \
        if (prof && tid == 0) {                       \
            const long long now_ = clock64();         \
            s_pc[(k)] += now_ - s_prev;               \
            s_prev = now_;                            \
        }                                             \
    } while (0)

template <int NV, bool STAGE, bool REL>
__global__ void __launch_bounds__(WS_THREADS, PSWARM_MIN_BLOCKS) k_pc_uni(const SegArgs a) {
    constexpr int T = WS_THREADS, NW = WS_THREADS / 32;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int N = a.N, B = a.fd.n_bodies;
    const int half = N / 2;
    const WsLayout L = ws_layout(N, a.nkp, 0, B, STAGE ? 1 : 0, 1, REL);
    double* ybuf = reinterpret_cast<double*>(smem_raw + L.ybuf);
    const size_t fb_bytes = L.fbuf1 - L.fbuf0;
    double* fb0 = reinterpret_cast<double*>(smem_raw + L.fbuf0);
    double* anc = reinterpret_cast<double*>(smem_raw + L.anchor);
    double* b0part = reinterpret_cast<double*>(smem_raw + L.b0part);
    double* eph = reinterpret_cast<double*>(smem_raw + L.eph);
    WsState& st = *reinterpret_cast<WsState*>(smem_raw + L.state);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int KP = 8 * a.nkp;
    const int mtiles = (half + 7) / 8;
    const bool prof = a.phase_cycles != nullptr;
    __shared__ long long s_pc[PHASES];
    long long s_prev = 0;
    if (tid < PHASES) s_pc[tid] = 0;
    if (tid == 0) s_prev = clock64();

    // ---- TMA bulk staging of the segment's node table (as k_pc_ws), overlapped with the prologue
    if (STAGE && tid == 0) {
        mbar_init(&st.stage_bar, 1);
        bulk_stage(eph, REL ? a.fd.rel_tab : a.fd.eph_t, static_cast<unsigned>(sizeof(double) * eph_stage_doubles(N, B, REL)),
                   &st.stage_bar);
    }
    const int fb_doubles = ws_fold_ksteps(N, a.nkp) * FKS;
    for (int i = tid; i < 2 * fb_doubles; i += T) fb0[i] = 0.0;
    for (int k = tid; k < KP; k += T) anc[k] = k < N ? a.anc_fold[k] : 0.0;
    const bool nodec = STAGE || a.fd.eph_t != nullptr;  // (as k_pc_ws)
    const double* pos_base = STAGE ? eph : nodec ? a.fd.eph_t : a.fd.body_pos;
    const double* ind_base = STAGE ? eph + 3 * B * eph_ld(N) : nodec ? a.fd.eph_t + 3 * B * eph_ld(N) : a.fd.indirect;
    const int psj = nodec ? 1 : 3 * B, psc = nodec ? eph_ld(N) : 1;
    const double* rel_base = STAGE ? eph : a.fd.rel_tab;
    if (tid == 0) {
        for (int t = 0; t < SLOTS; ++t) {
            st.slot_traj[t] = -1;
            st.grp_id[t] = -1;
            st.sing_key[t] = INT_MAX;
            st.nf_key[t] = INT_MAX;
            st.slot_err[t] = 0ull;
        }
        st.act_word[0] = st.act_word[1] = 0;
        st.new_mask[0] = st.new_mask[1] = 0;
        st.half_active[0] = st.half_active[1] = 0;
        st.free_mask[0] = st.free_mask[1] = st.retire_mask[0] = st.retire_mask[1] = 0;
        st.queue_done = 0;
        st.timeout = 0;
        st.exit_flag = 0;
    }
    __syncthreads();
    if (STAGE) mbar_wait(&st.stage_bar, 0);
    bool first = true;
    for (;;) {
        // ---- decisions of both halves (warp h), after the previous iteration's epilogue
        if (!first && warp < 2) decide_half(a, st, warp, lane, B);
        __syncthreads();
        UNI_PHASE(0);
        // ---- retire outputs (both halves)
        const int rm = st.retire_mask[0] | st.retire_mask[1];
        if (!first && rm) {
            const int j_begin = a.seg == 0 ? 0 : 1;
            for (int i = tid; i < N * SLOTS; i += T) {
                const int j = i >> 3, t = i & 7, h = t / HS, s = t % HS;
                if (!((rm >> t) & 1)) continue;
                const size_t tr = static_cast<size_t>(st.slot_traj[t]);
                if (a.samples && j >= j_begin) {
                    double* o = a.samples + (tr * a.R + a.row0 + j) * 6;
#pragma unroll
                    for (int c = 0; c < 6; ++c) o[c] = ybuf[y2(j, h, c, s)];
                }
                if (a.hot)
                    for (int c = 0; c < 6; ++c) hot_retire_node(a.hot + (tr * N + j) * 6, c, ybuf[y2(j, h, c, s)]);
                if (a.blk)  // wide-group round: the full iterate (resume source)
                    for (int c = 0; c < 6; ++c) a.blk[(tr * N + j) * 6 + c] = ybuf[y2(j, h, c, s)];
                if (j == N - 1) {
#pragma unroll
                    for (int c = 0; c < 6; ++c) a.state_out[tr * 6 + c] = ybuf[y2(j, h, c, s)];
                }
            }
            __syncthreads();  // slot_traj is rewritten by the claim below
        }
        // ---- free + claim into both halves (thread 0): ONE queue atomic for both halves (half 0's
        //      groups first, as k_pc_ws claims them), so a tick pays one global round trip
        if (tid == 0) {
            int am = st.act_word[0] | st.act_word[1];
            if (!first) {
                const int fm = st.free_mask[0] | st.free_mask[1];
                am &= ~fm;
                for (int t = 0; t < SLOTS; ++t)
                    if ((fm >> t) & 1) st.slot_traj[t] = -1;
            }
            int want[2] = {0, 0}, gq = 0, gend = 0;
            for (int h = 0; h < 2; ++h) {
                const int free_h = HS - __popc(static_cast<unsigned>(am & (0xF << (h * HS))));
                want[h] = !st.queue_done && free_h >= a.gmax ? free_h / a.gmax : 0;
            }
            if (want[0] + want[1] > 0) {
                gq = atomicAdd(a.queue, want[0] + want[1]);
                gend = min(gq + want[0] + want[1], a.P);
                if (gq + want[0] + want[1] >= a.P) st.queue_done = 1;
            }
            for (int h = 0; h < 2; ++h) {
                int new_mask = 0;
                const int g0 = gq + (h ? want[0] : 0), g1 = min(g0 + want[h], gend);
                for (int gi = g0; gi < g1; ++gi) {
                    int lg = h * HS;
                    while (st.grp_id[lg] >= 0) ++lg;
                    int off, size, gid;
                    claim_group(a, gi, off, size, gid);
                    st.grp_id[lg] = gid;
                    st.grp_size[lg] = size;
                    st.grp_iter[lg] = start_iteration(a, off);
                    st.grp_floor[lg] = claim_floor(a, gid);
                    st.grp_cap[lg] = claim_cap(a, gid);
                    if (a.traj_ns) st.grp_t0[lg] = globaltimer_ns();
                    int t = h * HS;
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
                st.new_mask[h] = new_mask;
            }
            for (int h = 0; h < 2; ++h) {
                const int hmask = 0xF << (h * HS);
                st.act_word[h] = am & hmask;
                st.half_active[h] = (am & hmask) != 0;
            }
            // (free / retire masks: rewritten by decide_half every iteration; every thread read
            //  retire_mask above without a barrier when nothing retired)
            if (a.deadline_ns != 0ull && globaltimer_ns() > a.deadline_ns) st.timeout = 1;
        }
        __syncthreads();
        UNI_PHASE(1);
        const int am = st.act_word[0] | st.act_word[1];
        if (st.timeout || (am == 0 && st.queue_done)) {
            if (tid == 0 && st.timeout)
                for (int lg = 0; lg < SLOTS; ++lg) {
                    const int gi = st.grp_id[lg];
                    if (gi < 0) continue;
                    a.faults[gi].status = FAULT_TIMEOUT;
                    a.faults[gi].iteration = st.grp_iter[lg];
                    a.rep_iter[gi] = st.grp_iter[lg];
                    a.rep_conv[gi] = 0;
                }
            break;
        }
        // ---- load + warm start of new slots (both halves)
        const int new_mask = st.new_mask[0] | st.new_mask[1];
        if (new_mask) {
            for (int i = tid; i < SLOTS * 6; i += T) {
                const int s = i / 6, c = i % 6;
                if ((new_mask >> s) & 1) st.y0[s][c] = a.state_in[static_cast<size_t>(st.slot_traj[s]) * 6 + c];
            }
            __syncthreads();
            for (int i = tid; i < N * SLOTS; i += T) {
                const int j = i >> 3, t = i & 7, h = t / HS, s = t % HS;
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
                            if (kepler_propagate(r, v, a.fd.central_mu, a.times[j] - a.epoch, ro, vo, &mf, &ef) != CONIC_OK)
                                atomicMin(&st.warm_key[t], j * 4 + CONIC_SOLVER);
                        }
                        if (j == 0 && a.cold_fallback) a.cold_fallback[st.slot_traj[t]] = (chk == CONIC_NON_ELLIPTIC) ? 1 : 0;
                    }
                    if (a.hot)
                        hot_start_node(a.hot + (static_cast<size_t>(st.slot_traj[t]) * N + j) * 6, a.hot_apply, ro, vo);
                }
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    ybuf[y2(j, h, c, s)] = ro[c];
                    ybuf[y2(j, h, c + 3, s)] = vo[c];
                }
            }
            __syncthreads();
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
        UNI_PHASE(2);
        // ---- force of both halves, folded as written (mirrored node pairs); relativistic: per
        //      node with the fused 1PN pass, then folded in place
        if constexpr (REL) {
            const int ns = a.force_ns ? a.force_ns : (N > 64 ? 2 : 1);  // slots per item (2 fused chains; N = 200: 800 items)
            // items node-major: the 8 / ns (half, slot group) items of a node sit in adjacent lanes,
            // so a warp reads 32 ns / 8 distinct table rows per load (shared-memory broadcast)
            const int per_node = 2 * (4 / ns);
            for (int w = tid; w < N * per_node; w += T) {
                const int j = w / per_node, r = w % per_node, h = r / (4 / ns);
                const int act_h = (am >> (h * HS)) & 0xF;
                if (!act_h) continue;
                double* fbh = fb0 + h * (fb_bytes / sizeof(double));
                const int s0 = (r % (4 / ns)) * ns;
                if (ns == 4) force_half_rel<4, !STAGE>(a.fd, rel_base, ybuf, fbh, st.sing_key, act_h, h, j, s0);
                else if (ns == 2) force_half_rel<2, !STAGE>(a.fd, rel_base, ybuf, fbh, st.sing_key, act_h, h, j, s0);
                else force_half_rel<1, !STAGE>(a.fd, rel_base, ybuf, fbh, st.sing_key, act_h, h, j, s0);
            }
            __syncthreads();
            UNI_PHASE(3);
            // fold: s_k at k, a_k = F_k - F_{N-1-k} at N-1-k (warp per (half, column), lane per node),
            // with b0 = (omega2 anchor.F + 2 y0) / 2 of the column formed in the same pass
            for (int hc = warp; hc < 2 * HC; hc += NW) {
                const int h = hc / HC, col = hc % HC;
                if (!((am >> (h * HS)) & 0xF)) continue;
                double* fbh = fb0 + h * (fb_bytes / sizeof(double));
                const int c = 2 * (col >> 3) + (col & 1), sl = (col & 7) >> 1;
                double part = 0.0;
                for (int k = lane; k < half; k += 32) {
                    const int lo = f2(k, c, sl), hi = f2(N - 1 - k, c, sl);
                    const double flo = fbh[lo], fhi = fbh[hi];
                    const double sk = flo + fhi, ak = flo - fhi;
                    fbh[lo] = sk;
                    fbh[hi] = ak;
                    part = fma(anc[k], sk, fma(anc[N - 1 - k], ak, part));
                }
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) part += __shfl_xor_sync(0xffffffffu, part, off);
                if (lane == 0) st.b0h[h][col] = 0.5 * fma(a.omega2, part, 2.0 * st.y0[h * HS + sl][c]);
            }
        } else {
            const int npw = half > T / 8 ? 2 : 4;  // work items per (half, node pair): slot pairs or slots
            for (int w = tid; w < 2 * npw * half; w += T) {
                const int h = w / (npw * half), r = w % (npw * half);
                const int act_h = (am >> (h * HS)) & 0xF;
                if (!act_h) continue;
                double* fbh = fb0 + h * (fb_bytes / sizeof(double));
                if (npw == 2)
                    force_pair<2>(a.fd, ybuf, fbh, st.sing_key, pos_base, ind_base, psj, psc, act_h, h, r % half, N,
                                  (r / half) * 2);
                else
                    force_pair<1>(a.fd, ybuf, fbh, st.sing_key, pos_base, ind_base, psj, psc, act_h, h, r % half, N,
                                  r / half);
            }
        }
        __syncthreads();
        UNI_PHASE(REL ? 7 : 3);  // relativistic: the fold + b0 pass
        if (tid < SLOTS && st.sing_key[tid] != INT_MAX) {
            const int t = tid, h = t / HS, s = t % HS, key = st.sing_key[t], j = key / (B + 1), chk = key % (B + 1);
            st.sing_val[t] = check_distance(ybuf[y2(j, h, 0, s)], ybuf[y2(j, h, 1, s)], ybuf[y2(j, h, 2, s)], j, chk, a.fd);
        }
        // ---- b0 = anchor.F + 2 y0 of both halves (warps 0-7: half 0, 8-15: half 1; fixed order);
        //      relativistic: formed by the fold pass above
        if constexpr (!REL) {
            const int h = warp / (NW / 2), fw = warp % (NW / 2);  // (NW / 2 == B0_PARTS)
            if ((am >> (h * HS)) & 0xF) {
                const double* fbh = fb0 + h * (fb_bytes / sizeof(double));
                double s0 = 0.0, s1 = 0.0, s2 = 0.0;
                const int jl = lane & 3;
                for (int kq = fw; kq < a.nkp * 2; kq += NW / 2) {
                    const double w = anc[4 * kq + jl];
                    const double* fq = fbh + kq * FKS + lane;
                    s0 = fma(w, fq[0], s0);
                    s1 = fma(w, fq[32], s1);
                    s2 = fma(w, fq[64], s2);
                }
#pragma unroll
                for (int off = 1; off < 4; off <<= 1) {
                    s0 += __shfl_xor_sync(0xffffffffu, s0, off);
                    s1 += __shfl_xor_sync(0xffffffffu, s1, off);
                    s2 += __shfl_xor_sync(0xffffffffu, s2, off);
                }
                if (jl == 0) {
                    double* bp = b0part + (h * B0_PARTS + fw) * HC;
                    const int c8 = lane >> 2;
                    bp[c8] = s0;
                    bp[8 + c8] = s1;
                    bp[16 + c8] = s2;
                }
            }
        }
        if constexpr (!REL) __syncthreads();
        if (!REL && tid < 2 * HC) {
            const int h = tid / HC, ft = tid % HC;
            if ((am >> (h * HS)) & 0xF) {
                const int c = 2 * (ft >> 3) + (ft & 1), s = (ft & 7) >> 1;
                double sum = 0.0;
#pragma unroll
                for (int part = 0; part < B0_PARTS; ++part) sum += b0part[(h * B0_PARTS + part) * HC + ft];
                st.b0h[h][ft] = 0.5 * fma(a.omega2, sum, 2.0 * st.y0[h * HS + s][c]);
            }
        }
        __syncthreads();
        UNI_PHASE(4);
        // ---- DMMA + epilogue: units (pair tile, half), unit u = warp + 16 i
        {
            const int nunits = 2 * mtiles;
            int tl[NV], hh[NV];
            const double* fbu[NV];
            int nv = 0;
#pragma unroll
            for (int i = 0; i < NV; ++i) {
                const int u = warp + i * NW;
                hh[i] = u < nunits ? u / mtiles : 0;
                tl[i] = u < nunits ? u % mtiles : 0;
                fbu[i] = fb0 + hh[i] * (fb_bytes / sizeof(double));
                if (u < nunits && st.half_active[hh[i]]) nv = i + 1;
            }
            double acc[NV][3][2][2];
            if (nv == NV) {
                gemm_units_fold<NV>(a.upack_fold, a.nkp_fold, half, fbu, tl, lane, acc);
                UNI_PHASE(5);
#pragma unroll
                for (int i = 0; i < NV; ++i)
                    if (st.half_active[hh[i]]) epilogue_unit_fold(a, st, ybuf, acc[i], hh[i], tl[i], half, lane);
            } else if (nv > 0) {  // NV == 2, the warp's second unit is out of range or idle
                if constexpr (NV == 2) {
                    const double* f1[1] = {fbu[0]};
                    const int t1[1] = {tl[0]};
                    double a1[1][3][2][2];
                    if (st.half_active[hh[0]]) {
                        gemm_units_fold<1>(a.upack_fold, a.nkp_fold, half, f1, t1, lane, a1);
                        epilogue_unit_fold(a, st, ybuf, a1[0], hh[0], tl[0], half, lane);
                    }
                }
            }
        }
        __syncthreads();
        UNI_PHASE(6);
        first = false;
    }
    if (prof) {
        __syncthreads();
        if (tid == 0) {
            s_pc[PHASES - 1] = 1;
            for (int k = 0; k < PHASES; ++k)
                if (s_pc[k]) atomicAdd(a.phase_cycles + k, static_cast<unsigned long long>(s_pc[k]));
        }
    }
}

template <int NV, bool STAGE, bool REL = false>
static cudaError_t launch_uni_t(const SegArgs& a, int grid, size_t smem, cudaStream_t s) {
    auto kern = k_pc_uni<NV, STAGE, REL>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    kern<<<grid, WS_THREADS, smem, s>>>(a);
    return cudaGetLastError();
}

template <int MAIN, int XMW, bool FOLD = false>
static cudaError_t launch_ws_t(const SegArgs& a, int grid, size_t smem, cudaStream_t s) {
    // relativistic launches of this kernel never stage the node table (the host clears stage_eph)
    auto kern = a.fd.rel ? k_pc_ws<MAIN, XMW, false, true, FOLD>
                         : (a.stage_eph ? k_pc_ws<MAIN, XMW, true, false, FOLD> : k_pc_ws<MAIN, XMW, false, false, FOLD>);
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    kern<<<grid, WS_THREADS, smem, s>>>(a);
    return cudaGetLastError();
}

/// Tiles of one half: m-tiles of node rows, or (folded) of row pairs.
static int ws_mtiles(int N, bool fold) { return fold ? (N / 2 + 7) / 8 : (N + 7) / 8; }
/// Folded: pair tiles beyond the largest multiple of 4 (one per SMSP) when 1 or 2 are left
/// over become single-n-tile units on the warps with one full tile fewer (3 or 6 units; with
/// 3 left over the strided plan is already as balanced; below 9 pair tiles the staged rows
/// cost more than the balance gains).  N = 200: 13 pair tiles -> 12 full
/// + 3 units, the busiest SMSP issues 10 instead of 12 n-tile streams per half.
static int ws_fold_extra_tiles(int N) {
    const int mt = ws_mtiles(N, true), r = mt % 4, nfull = mt - r;
    if (!(r == 1 || r == 2) || mt <= 8) return 0;  // N = 96: staging costs more (measured)
    // every extra unit must land on a warp with fewer than MAIN full tiles (gemm_half_fold runs
    // one full tile + the unit there): with MAIN = 2 only 16 - nfull warps qualify
    const int main = (nfull + MMA_WARPS - 1) / MMA_WARPS;
    if (main > 1 && 3 * r > 2 * MMA_WARPS - nfull) return 0;  // N = 216: 6 units, 4 such warps
    return r;
}
/// Dense: MAIN = floor(m-tiles / 8) full-width m-tiles per warp + extras.  Folded: full pair
/// tiles strided over the warps (ceil) + the extra units above.
int ws_main_tiles(int N, bool fold) {
    return fold ? (ws_mtiles(N, true) - ws_fold_extra_tiles(N) + MMA_WARPS - 1) / MMA_WARPS
                : ws_mtiles(N, false) / MMA_WARPS;
}
/// Extra (m-tile, n-tile) tiles beyond the MAIN full-width m-tiles of every MMA warp.
static int ws_extras(int N, bool fold) {
    return fold ? 0 : (ws_mtiles(N, false) - ws_main_tiles(N, false) * MMA_WARPS) * 3;
}

int ws_extra_rows(int N, bool fold) {
    if (fold) return 8 * ws_fold_extra_tiles(N);  // staged pair rows
    const int r = N - ws_main_tiles(N, false) * MMA_WARPS * 8;
    return r > 0 ? r : 0;
}

bool ws_supported(int N, bool fold) {
    const int main = ws_main_tiles(N, fold);
    if (fold)  // whole k-quads per part, 1-2 pair tiles per warp
        return N % 8 == 0 && main >= 1 && main <= 2;
    // <3, 3> (N = 233..247: 18-21 extra tiles on 3 full m-tiles per warp) spills and loses to
    // k_pc_segment (profiles/dense_plans_r02.json); every other dense plan beats it
    return main >= 1 && main <= 4 && ws_extras(N, false) <= 3 * MMA_WARPS && (main < 4 || ws_extras(N, false) <= MMA_WARPS) &&
           !(main == 3 && ws_extras(N, false) > 2 * MMA_WARPS);
}

size_t ws_smem_bytes(int N, int nkp, int xrows, int B, int stage_eph, bool fold, bool rel) {
    return ws_layout(N, nkp, xrows, B, stage_eph, fold ? 1 : 0, rel).total;
}

/// Unified folded kernel (N % 8 == 0): units of 2 x ceil(N/16) pair tiles over all warps.
constexpr int UNI_WARPS = WS_THREADS / 32;
bool uni_supported(int N) { return N % 8 == 0 && (2 * ws_mtiles(N, true) + UNI_WARPS - 1) / UNI_WARPS <= 2; }

cudaError_t launch_segment_uni(const SegArgs& a, int grid, cudaStream_t s) {
    if (!uni_supported(a.N) || a.upack_fold == nullptr) return cudaErrorNotSupported;
    const int nv = (2 * ws_mtiles(a.N, true) + UNI_WARPS - 1) / UNI_WARPS;
    const size_t smem = ws_smem_bytes(a.N, a.nkp, 0, a.fd.n_bodies, a.stage_eph, true, a.fd.rel != 0);
    if (a.fd.rel) {  // relativistic: the node table is staged when it fits (host: stage_eph)
        if (a.stage_eph)
            return nv == 1 ? launch_uni_t<1, true, true>(a, grid, smem, s) : launch_uni_t<2, true, true>(a, grid, smem, s);
        return nv == 1 ? launch_uni_t<1, false, true>(a, grid, smem, s) : launch_uni_t<2, false, true>(a, grid, smem, s);
    }
    if (a.stage_eph)
        return nv == 1 ? launch_uni_t<1, true>(a, grid, smem, s) : launch_uni_t<2, true>(a, grid, smem, s);
    return nv == 1 ? launch_uni_t<1, false>(a, grid, smem, s) : launch_uni_t<2, false>(a, grid, smem, s);
}

cudaError_t launch_segment_ws(const SegArgs& a, int grid, cudaStream_t s) {
    const bool fold = a.upack_fold != nullptr;
    if (!ws_supported(a.N, fold)) return cudaErrorNotSupported;
    const int main = ws_main_tiles(a.N, fold);
    const int xmw = std::max(1, (ws_extras(a.N, fold) + MMA_WARPS - 1) / MMA_WARPS);
    const size_t smem = ws_smem_bytes(a.N, a.nkp, a.xrows, a.fd.n_bodies, a.stage_eph, fold);
    if (fold) {
        if (ws_fold_extra_tiles(a.N) > 0)  // XMW = 1: leftover pair tiles as single-n-tile units
            return main == 1 ? launch_ws_t<1, 1, true>(a, grid, smem, s) : launch_ws_t<2, 1, true>(a, grid, smem, s);
        return main == 1 ? launch_ws_t<1, 0, true>(a, grid, smem, s) : launch_ws_t<2, 0, true>(a, grid, smem, s);
    }
    switch (main * 4 + xmw) {
    case 5: return launch_ws_t<1, 1>(a, grid, smem, s);
    case 6: return launch_ws_t<1, 2>(a, grid, smem, s);
    case 7: return launch_ws_t<1, 3>(a, grid, smem, s);
    case 9: return launch_ws_t<2, 1>(a, grid, smem, s);
    case 10: return launch_ws_t<2, 2>(a, grid, smem, s);
    case 11: return launch_ws_t<2, 3>(a, grid, smem, s);
    case 13: return launch_ws_t<3, 1>(a, grid, smem, s);
    case 14: return launch_ws_t<3, 2>(a, grid, smem, s);
    case 17: return launch_ws_t<4, 1>(a, grid, smem, s);
    default: return cudaErrorNotSupported;
    }
}

#ifdef PSWARM_SLOTS_SMALL
}  // namespace small
#endif
}  // namespace pswarm_dev
