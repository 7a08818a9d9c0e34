// Kernel interfaces of the B200 PC path (host-visible structs + launchers).
// Implemented in pc_kernels.cu; called by the C-ABI layer (pswarm_capi.cu).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "pc_device.cuh"

namespace pswarm_dev {

/// Per-group failure record of one segment solve.  status codes below; coordinates
/// follow the reference exceptions (errors.hpp:40-62).
enum FaultStatus : int {
    FAULT_NONE = 0,
    FAULT_DIVERGENCE = 1,     // picard.hpp:26-36 first non-finite (node, column)
    FAULT_SINGULARITY = 2,    // force_model.hpp:115-120 (node, trajectory-in-group, body)
    FAULT_WARM_ZERO_RADIUS = 3,  // kepler.hpp:61-62 thrown out of warm_start
    FAULT_WARM_SOLVER = 4,    // kepler.hpp:40-41 thrown out of warm_start
    FAULT_TIMEOUT = 5,        // augment.hpp:117-121
};

struct GroupFault {
    int32_t status;
    int32_t iteration;   // iteration at which it happened (0 = warm start)
    int32_t body;        // -1 central / none
    int32_t pad;
    int64_t node;
    int64_t column;      // block column (divergence)
    int64_t trajectory;  // slot within the group (singularity) / batch index (warm start)
    double value;        // distance (singularity), mean anomaly (solver)
    double value2;       // eccentricity (solver)
};

/// Phase accounting slots (generic kernel): 0 claim, 1 warm start, 2 force, 3 DMMA,
/// 4 anchor/b0 barrier, 5 epilogue (main rows), 6 epilogue (staged rows), 7 decisions,
/// 8 retire; warp-specialised kernel: see pc_slots2.cu.  Slot PHASES-1 = CTA count.
constexpr int PHASES = 16;

/// Arguments of one segment launch of the persistent slot kernel.
struct SegArgs {
    int N;          // nodes
    int nkp;        // k-step pairs: K padded to 8*nkp
    GemmPlan gp;    // warp plan of the DMMA tiles (warps per CTA = gp.warps)
    int xrows;      // node rows covered by extra tiles (staged epilogue)
    int stage_eph;  // 1: per-segment ephemeris staged in shared memory
    int M;          // trajectories
    int P;          // groups
    int gmax;       // largest group (<= SLOTS)
    int seg;
    int cold_start;     // segment 0 with StartMode::cold
    int error_mode;     // 0 relative, 1 absolute
    int max_it;
    int record_history;
    int pad0;
    double tol;
    double tol2_lo, tol2_hi;  // tol^2 (1 -+ 1e-13): squared pre-test of err <= tol (picard.hpp:77)
    double omega2;
    double epoch;       // segment start time == times[0]
    unsigned long long deadline_ns;  // %globaltimer deadline, 0 = none
    ForceData fd;
    const double2* upack;       // packed [U; anchor] operator
    const double* times;        // [N]
    const int64_t* group_off;   // [P+1], nullptr for singleton groups
    const double* state_in;     // [M][6] segment initial states
    double* state_out;          // [M][6] terminal rows (chained)
    double* samples;            // [M][R][6] or nullptr
    int64_t R;
    int64_t row0;               // seg*(N-1)
    int* queue;                 // group work counter (zeroed per launch)
    int32_t* rep_iter;          // [P]
    double* rep_err;            // [P]
    uint8_t* rep_conv;          // [P]
    double* rep_hist;           // [P][max_it] or nullptr
    GroupFault* faults;         // [P]
    uint8_t* cold_fallback;     // [M] or nullptr
    unsigned long long* phase_cycles;  // [PHASES] diagnostics or nullptr
    double* hot;                // [M][N][6] hot-start corrections (EXTENSION) or nullptr
    int hot_apply;              // 1: this segment starts from base + correction
    const double2* upack_fold;  // mirror-folded operator pairs [pair][part][k-pair][lane] or nullptr
    int nkp_fold;               // k-pairs per folded part
    int b0_mma;                 // 1: folded b0 from the anchor pair row when N/2 % 8 != 0
    int fast_decide;            // 1: singleton-group decisions fast path (gmax == 1)
    int force_ns;               // force items: slots per item (0 auto, 1, 2; diagnostics)
    const double* anc_fold;     // [8 nkp] anchor weights of the folded F layout
    // ---- wide groups (groups larger than one CTA): member-level rounds (pswarm_capi.cu
    //      solve_wide_rounds).  All nullptr for ordinary launches.
    const int32_t* traj_list;   // [P] virtual singleton group gi -> trajectory; reports indexed by trajectory
    const int32_t* it_start;    // [M] > 0: resume from blk at this iteration count (no warm start)
    const int32_t* it_floor;    // [M] converge only at it >= floor
    const int32_t* it_cap;      // [M] stop at min(max_it, cap)
    double* blk;                // [M][N][6] full iterate of every retired trajectory (resume source)
    int hist_stride;            // row stride of rep_hist (the configured max_iterations)
    int pad1;
    // ---- independent mode with a timeout: each trajectory's OWN wall-clock budget, as the
    //      reference's run_independent gives every trajectory a propagate call (and a deadline)
    //      of its own (runner.hpp:63-80, propagator.hpp:233-236).  Device time a trajectory has
    //      spent in its slots, summed over segments; nullptr when the batch deadline applies.
    unsigned long long* traj_ns;     // [M]
    unsigned long long traj_budget_ns;
};

/// Per-trajectory budget (independent mode, traj_ns != nullptr): called by a group's decision
/// after iteration `it` with t0 = the %globaltimer of the group's claim.  Charges the slot time
/// when the group stops; otherwise returns true when the budget is spent -- the reference
/// checks its deadline before every force evaluation (augment.hpp:116-120), so a group that
/// has not stopped after an iteration times out before the next one.
__device__ __forceinline__ bool traj_budget_spent(const SegArgs& a, int traj, unsigned long long t0, bool stopping) {
    const unsigned long long used = a.traj_ns[traj] + (globaltimer_ns() - t0);
    if (stopping) {
        a.traj_ns[traj] = used;
        return false;
    }
    if (used <= a.traj_budget_ns) return false;
    a.traj_ns[traj] = used;
    return true;
}

/// Group claimed from the queue: offset of its first trajectory, size and the report index
/// (the group, or for a member-level round the trajectory itself).
__device__ __forceinline__ void claim_group(const SegArgs& a, int gi, int& off, int& size, int& gid) {
    if (a.traj_list) {
        off = a.traj_list[gi];
        size = 1;
        gid = off;
    } else if (a.group_off) {
        off = static_cast<int>(a.group_off[gi]);
        size = static_cast<int>(a.group_off[gi + 1]) - off;
        gid = gi;
    } else {  // singleton groups (no offsets uploaded): group gi is trajectory gi
        off = gi;
        size = 1;
        gid = gi;
    }
}
/// Iteration count a claimed trajectory starts from (> 0: resumed from a.blk).
__device__ __forceinline__ int start_iteration(const SegArgs& a, int traj) { return a.it_start ? a.it_start[traj] : 0; }
/// pc_solve's stopping rule with the member-level floor / cap of a wide-group round, fixed
/// at claim time into the CTA's group record: the decisions (on the kernel's critical
/// chain) compare against shared memory only.
__device__ __forceinline__ int claim_floor(const SegArgs& a, int gid) { return a.it_floor ? a.it_floor[gid] : 0; }
__device__ __forceinline__ int claim_cap(const SegArgs& a, int gid) {
    return a.it_cap ? min(a.max_it, a.it_cap[gid]) : a.max_it;
}
/// Resumed slot (wide-group round): node row j of the saved iterate; the hot-start record
/// (the previous retire's correction) is turned back into this segment's base.
__device__ __forceinline__ void resume_node(const SegArgs& a, int traj, int j, double ro[3], double vo[3]) {
    const double* b = a.blk + (static_cast<size_t>(traj) * a.N + j) * 6;
    for (int c = 0; c < 3; ++c) {
        ro[c] = b[c];
        vo[c] = b[3 + c];
    }
    if (a.hot) {
        double* hb = a.hot + (static_cast<size_t>(traj) * a.N + j) * 6;
        for (int c = 0; c < 6; ++c) hb[c] = b[c] - hb[c];
    }
}

/// Perturbing bodies on the device (ephemeris.hpp:44-73): analytic elements or
/// tabulated Chebyshev segments, flattened.
struct BodyTable {
    int B;
    const int* kind;          // [B] 0 analytic, 1 tabulated
    const double* elements;   // [B][7]
    const double* mu;         // [B]
    const int* seg_off;       // [B+1] first segment of each body
    const double* seg_bounds; // [S][2]
    const long long* coeff_off;  // [S] offset of the segment's [3][nc] block in coeffs
    const int* ncoef;         // [B]
    const double* coeffs;
};

/// Frozen per-segment ephemeris on the device: body positions [N][B][3] at the node
/// times and the indirect term [N][3] (ephemeris.hpp:89-107, force_model.hpp:50-51).
/// fault_key = min over (body, node) of (b*N + j)*4 + kind (1 coverage, 3 solver).
/// Relativistic model (EXTENSION, rel_tab != nullptr): also body velocities vel [N][B][3]
/// and the node table rel_tab [N][rel_stride(B)] (Sun row first, the indirect term last).
/// eph_t (optional): positions and indirect term node-contiguous, [3B + 3][eph_ld(N)].
cudaError_t launch_repack_states(const double* s7, double* s6, long long M, cudaStream_t s);
cudaError_t launch_pack_states7(const double* s6, double epoch, double* s7, long long M, cudaStream_t s);
cudaError_t launch_ephemeris(int N, const double* times, double central_mu, const BodyTable& bt, double* pos,
                             double* indirect, unsigned long long* fault_key, double* vel, double* rel_tab, double ic2,
                             double* eph_t, cudaStream_t s);

/// Wide-group path (member-level rounds): trajectory list 0..n-1 and the group error history
/// gh[P][stride] = max over members of mh[M][stride] for k < K[g], NaN beyond (gh zeroed first).
cudaError_t launch_iota(int32_t* out, int n, cudaStream_t s);
cudaError_t launch_group_hist(const double* mh, int stride, const int64_t* group_off, int P, const int32_t* gK, int M,
                              double* gh, cudaStream_t s);


/// Batched RKF7(8) verifier (pc_rk.cu; oracle.hpp:63-183): one thread per trajectory.
struct RkArgs {
    int M, R;
    int rel;                     // 1: n_body_1pn derivative (EXTENSION)
    int pad;
    long long max_steps;
    double rel_tol, abs_tol, central_mu, floor_km, c_light;
    BodyTable bt;
    const double* states;        // [M][7]
    const double* times;         // [R], times[0] == epoch
    const double* candidate;     // [M][R][6] samples to compare, or nullptr
    double* samples_out;         // [M][R][6] RK samples, or nullptr
    double* node_err;            // [M][R] max(position, velocity) relative discrepancy, or nullptr
    double* max_err;             // [M], or nullptr
    unsigned long long* fault_key;  // min of trajectory << 24 | code << 16 | node
    double* fault_t;             // [M] epoch reached at a fault
};
cudaError_t launch_rk_check(const RkArgs& a, cudaStream_t s);

/// Warp-specialised slot kernel (pc_slots2.cu) for groups of <= 4 trajectories.
/// fold: mirror-folded update (two half-size contractions, pc_slots2.cu ws_layout notes).
size_t ws_smem_bytes(int N, int nkp, int xrows, int B, int stage_eph, bool fold, bool rel = false);
int ws_main_tiles(int N, bool fold);
int ws_extra_rows(int N, bool fold);
bool ws_supported(int N, bool fold);
bool uni_supported(int N);
cudaError_t launch_segment_uni(const SegArgs& a, int grid, cudaStream_t s);
cudaError_t launch_segment_ws(const SegArgs& a, int grid, cudaStream_t s);
/// The same kernels with 4 MMA + 4 FP warps (256 threads) and two CTAs per SM, for small N
/// (pc_slots2.cu compiled with -DPSWARM_SLOTS_SMALL).
namespace small {
size_t ws_smem_bytes(int N, int nkp, int xrows, int B, int stage_eph, bool fold, bool rel = false);
int ws_extra_rows(int N, bool fold);
bool ws_supported(int N, bool fold);
bool uni_supported(int N);
cudaError_t launch_segment_uni(const SegArgs& a, int grid, cudaStream_t s);
cudaError_t launch_segment_ws(const SegArgs& a, int grid, cudaStream_t s);
}  // namespace small

GemmPlan make_gemm_plan(int N);
int extra_rows(int N, const GemmPlan& gp);
size_t segment_smem_bytes(int N, int nkp, int xrows, int B, int stage_eph);
cudaError_t launch_segment(const SegArgs& a, int grid, cudaStream_t s);

cudaError_t launch_picard_update(int N, int nkp, int C, const double* F, const double* y0, double* out,
                                 const double2* upack, cudaStream_t s);
cudaError_t launch_force_block(int N, int m, const double* y, double omega2, const ForceData& fd, int kind_nbody,
                               double* force, unsigned long long* fault_key, cudaStream_t s);
cudaError_t launch_block_error(int N, int m, const double* cur, const double* prev, int mode,
                               unsigned long long* per_state_bits, cudaStream_t s);
cudaError_t launch_warm_start(int M, const double* states, int N, const double* times, double mu, double* guesses,
                              uint8_t* fallback, unsigned long long* fault_key, double* fault_vals, cudaStream_t s);

}  // namespace pswarm_dev
