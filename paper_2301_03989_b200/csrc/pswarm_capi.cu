// C-ABI implementation (include/pswarm_gpu.h): device context, host
// orchestration of the segment loop (propagator.hpp:192-347), and the
// operator-level entry points.  All numerics of the hot loop run in the CUDA
// kernels of pc_kernels.cu; the host only prepares per-segment constants (grid,
// frozen ephemeris, packed operators) and turns device fault records into the
// reference's exceptions.  There is no CPU fallback anywhere in this file.
#include <algorithm>
#include <iterator>
#include <chrono>
#include <climits>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>  // types only: libnccl is opened at run time (multi-device gather)
#include <thread>

#include "pc_kernels.cuh"
#include "pswarm/block.hpp"
#include "pswarm/chebyshev.hpp"
#include "pswarm/ephemeris.hpp"
#include "pswarm/errors.hpp"
#include "pswarm/kepler.hpp"
#include "pswarm/pc_matrices.hpp"
#include "pswarm/propagator.hpp"
#include "pswarm/synthetic.hpp"
#include "pswarm_gpu.h"

using pswarm::Index;
using namespace pswarm_dev;

namespace {

// ------------------------------------------------------------ error plumbing
struct CapiFault {
    pswarm_error e{};
};

std::string fmtf(const char* f, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, f);
    std::vsnprintf(buf, sizeof buf, f, ap);
    va_end(ap);
    return buf;
}

void init_err(pswarm_error* e, int32_t status, const std::string& msg) {
    std::memset(e, 0, sizeof(*e));
    e->status = status;
    e->body = -1;
    e->segment = e->group = e->node = e->column = e->trajectory = -1;
    std::snprintf(e->message, sizeof(e->message), "%s", msg.c_str());
}

[[noreturn]] void raise(int32_t status, const std::string& msg) {
    CapiFault f;
    init_err(&f.e, status, msg);
    throw f;
}

void cuda_check(cudaError_t e, const char* what) {
    if (e == cudaSuccess) return;
    raise(e == cudaErrorMemoryAllocation ? PSWARM_ERR_OOM : PSWARM_ERR_CUDA,
          std::string("CUDA failure in ") + what + ": " + cudaGetErrorString(e));
}

template <typename Fn>
pswarm_status guarded(pswarm_error* err, Fn&& fn) {
    pswarm_error local;
    pswarm_error* e = err ? err : &local;
    init_err(e, PSWARM_OK, "");
    try {
        fn();
        return PSWARM_OK;
    } catch (const CapiFault& f) {
        *e = f.e;
    } catch (const pswarm::DivergenceError& x) {
        init_err(e, PSWARM_ERR_DIVERGENCE, x.what());
        e->node = x.node();
        e->column = x.column();
    } catch (const pswarm::SingularityError& x) {
        init_err(e, PSWARM_ERR_SINGULARITY, x.what());
        std::snprintf(e->body_name, sizeof(e->body_name), "%s", x.body().c_str());
    } catch (const pswarm::CoverageError& x) {
        init_err(e, PSWARM_ERR_COVERAGE, x.what());
        e->value = x.epoch();
    } catch (const pswarm::InvalidSpanError& x) {
        init_err(e, PSWARM_ERR_INVALID_SPAN, x.what());
    } catch (const pswarm::InvalidSizeError& x) {
        init_err(e, PSWARM_ERR_INVALID_SIZE, x.what());
    } catch (const pswarm::ShapeError& x) {
        init_err(e, PSWARM_ERR_SHAPE, x.what());
    } catch (const pswarm::AlignmentError& x) {
        init_err(e, PSWARM_ERR_ALIGNMENT, x.what());
    } catch (const pswarm::NonEllipticError& x) {
        init_err(e, PSWARM_ERR_NON_ELLIPTIC, x.what());
    } catch (const pswarm::SolverError& x) {
        init_err(e, PSWARM_ERR_SOLVER, x.what());
    } catch (const pswarm::InvalidPlanError& x) {
        init_err(e, PSWARM_ERR_INVALID_PLAN, x.what());
    } catch (const pswarm::TimeoutError& x) {
        init_err(e, PSWARM_ERR_TIMEOUT, x.what());
    } catch (const pswarm::OracleError& x) {
        init_err(e, PSWARM_ERR_ORACLE, x.what());
    } catch (const std::bad_alloc&) {
        init_err(e, PSWARM_ERR_OOM, "host allocation failed");
    } catch (const std::exception& x) {
        init_err(e, PSWARM_ERR_GENERIC, x.what());
    }
    return static_cast<pswarm_status>(e->status);
}

// ------------------------------------------------------------ device memory
struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
    template <typename T>
    T* get(size_t count) {
        const size_t bytes = std::max<size_t>(count * sizeof(T), 16);
        if (bytes > cap) {
            if (p) cudaFree(p);
            p = nullptr;
            cap = 0;
            cuda_check(cudaMalloc(&p, bytes), "cudaMalloc");
            cap = bytes;
        }
        return static_cast<T*>(p);
    }
    ~DevBuf() {
        if (p) cudaFree(p);
    }
};

struct OpPack {
    DevBuf buf;
    int nkp = 0;
    GemmPlan gp{};
    // mirror-folded operators (even N, N % 8 == 0): [pair][part][k-pair][lane] double2 + the
    // anchor weights of the folded F layout (pc_slots2.cu ws_layout notes)
    DevBuf fold, anc_fold;
    int nkp_fold = 0;
};

enum BufId {
    B_STATE_A, B_STATE_B, B_GROUP_OFF, B_TIMES, B_BODY_POS, B_BODY_MU, B_INDIRECT, B_QUEUE,
    B_REP_ITER, B_REP_ERR, B_REP_CONV, B_REP_HIST, B_FAULTS, B_FALLBACK, B_SAMPLES, B_DEAD,
    B_OP_IN, B_OP_IN2, B_OP_OUT, B_OP_AUX, B_OP_KEY,
    B_BT_KIND, B_BT_SOFF, B_BT_NC, B_BT_EL, B_BT_BND, B_BT_COFF, B_BT_CF, B_PHASES,
    B_W_REP, B_W_LIST, B_W_CTL, B_W_HIST, B_W_BLK, B_W_GK,
    B_IN_PACK, B_REPORT, B_BODY_VEL, B_REL_TAB, B_HOT, B_STATES7, B_EPH_T, B_TRAJ_NS, B_COUNT
};

/// Page-locked host staging (grow-only): every host<->device transfer of a solve goes
/// through one of these so the copies are true async DMA, one per direction and segment.
struct PinnedBuf {
    void* p = nullptr;
    size_t cap = 0;
    template <typename T>
    T* get(size_t bytes) {
        bytes = std::max<size_t>(bytes, 64);
        if (bytes > cap) {
            if (p) cudaFreeHost(p);
            p = nullptr;
            cap = 0;
            cuda_check(cudaHostAlloc(&p, bytes, cudaHostAllocDefault), "cudaHostAlloc");
            cap = bytes;
        }
        return static_cast<T*>(p);
    }
    ~PinnedBuf() {
        if (p) cudaFreeHost(p);
    }
};

/// Byte layout of a packed transfer: 16-byte aligned sub-arrays.
struct Pack {
    size_t total = 0;
    size_t add(size_t bytes) {
        const size_t o = total;
        total += (bytes + 15) & ~static_cast<size_t>(15);
        return o;
    }
};

}  // namespace

struct pswarm_ctx {
    // host copies of the per-segment reports when the caller asks for none (grow-only: no fresh
    // pages per call); otherwise the caller's [S][P] / [S][M] output arrays are written directly
    std::vector<int32_t> host_iter;
    std::vector<double> host_err;
    std::vector<uint8_t> host_conv, host_fb;
    int device = 0;
    int sm_count = 0;
    cudaStream_t stream = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr, evk0 = nullptr, evk1 = nullptr;
    cudaStream_t copy_stream = nullptr;  // per-segment sample D2H overlapped with the next segment
    cudaEvent_t ev_seg = nullptr;
    std::map<Index, std::unique_ptr<OpPack>> ops;
    DevBuf buf[B_COUNT];
    int64_t launches = 0;
    int ctas_per_sm = 1;
    int max_ctas = 0;  // 0 = SM count * ctas_per_sm
    int profile_phases = 0;
    const char* last_kernel = "";
    int slot_kernel = 0;  // 0 auto, 1 generic k_pc_segment, 2 warp-specialised k_pc_ws
    int poison_outputs = 0;  // 1: NaN-fill device outputs before each solve (tests)
    int fold = 1;            // 1: mirror-folded update when N % 8 == 0 (k_pc_ws_fold)
    int fast_decide = 1;     // singleton-group decisions fast path
    int force_ns = 0;        // force items: slots per item (0 auto; diagnostics)
    int small_ctas = 1;      // small N: 256-thread slot kernels, two CTAs per SM
    int small_max_n = 0;     // largest N for them (0: by force model, measured)
    int stage = 1;           // stage the per-segment node table in shared memory when it fits (0: never)
    int eph_nc = 1;          // unstaged ephemeris read node-contiguous from global (eph_t): coalesced
                             // (-14 % kernel time at N = 256, tools/probe_ab_opt.py eph_nc)
    int b0_mma = 2;          // folded: b0 from the anchor pair row (spare row, N/2 % 8 != 0): 1 on, 0 off, 2 auto
    int unified = 2;         // folded solves: 1 k_pc_uni (all warps per phase), 0 k_pc_ws_fold, 2 auto =
                             // k_pc_uni for the force-bound 1PN model (N <= 200), else k_pc_ws_fold
                             // (measured, tools/probe_uni.py)
    unsigned long long phase_host[pswarm_dev::PHASES] = {};
    PinnedBuf pin_in, pin_rep, pin_term, pin_wide;
    int wide_rounds = 0;  // member-level rounds of the last wide-group segment (diagnostics)
};

namespace {

void bind(pswarm_ctx* ctx) { cuda_check(cudaSetDevice(ctx->device), "cudaSetDevice"); }

/// [update_op; anchor_op] packed in mma.m8n8k4 A-fragment order (pc_device.cuh).
/// [update_op; anchor_op] (row-major N x N and N) in the DMMA A-fragment order
/// [m-tile][k-pair][lane] double2, rows padded to the plan's m-tiles, K to 8.
std::vector<double> pack_dense_operator(Index n, const GemmPlan& gp, const double* U, const double* anchor) {
    const int nkp = static_cast<int>((n + 7) / 8);
    const int rows = 8 * gp.mtiles;
    auto A = [&](int r, int k) -> double {
        if (k >= n) return 0.0;
        if (r < n) return U[static_cast<size_t>(r) * n + k];
        if (r == n) return anchor[k];
        return 0.0;
    };
    std::vector<double> host(static_cast<size_t>(rows / 8) * nkp * 32 * 2);
    for (int m = 0; m < rows / 8; ++m)
        for (int kp = 0; kp < nkp; ++kp)
            for (int lane = 0; lane < 32; ++lane) {
                const int g = lane >> 2, q = lane & 3;
                const size_t idx = (static_cast<size_t>(m) * nkp + kp) * 32 + lane;
                host[2 * idx] = A(m * 8 + g, kp * 8 + q);
                host[2 * idx + 1] = A(m * 8 + g, kp * 8 + 4 + q);
            }
    return host;
}

const OpPack& operators(pswarm_ctx* ctx, Index n) {
    auto it = ctx->ops.find(n);
    if (it != ctx->ops.end()) return *it->second;
    if (n > 264) raise(PSWARM_ERR_INVALID_SIZE, fmtf("device operators support up to 264 nodes, got %lld", (long long)n));
    const auto mats = pswarm::cached_matrices(n);  // InvalidSizeError for n < 3
    const GemmPlan gp = make_gemm_plan(static_cast<int>(n));
    const int nkp = static_cast<int>((n + 7) / 8);
    const std::vector<double> host = pack_dense_operator(n, gp, mats->update_op.data(), mats->anchor_op.data());
    auto p = std::make_unique<OpPack>();
    p->nkp = nkp;
    p->gp = gp;
    double* d = p->buf.get<double>(host.size());
    cuda_check(cudaMemcpy(d, host.data(), host.size() * sizeof(double), cudaMemcpyHostToDevice), "upload operators");
    if (n % 8 == 0) {  // U anticommutes with the node reversal: two half-size operators
        const int half = static_cast<int>(n / 2), np = (half + 7) / 8, nkpf = (half + 7) / 8;
        std::vector<double> af(static_cast<size_t>(8 * nkp), 0.0);
        for (int k = 0; k < n; ++k)
            af[k] = k < half ? 0.5 * (mats->anchor_op[k] + mats->anchor_op[n - 1 - k])
                             : 0.5 * (mats->anchor_op[n - 1 - k] - mats->anchor_op[k]);
        auto G = [&](int part, int r, int k) -> double {  // 1/2 folded into the operator
            // pair row N/2 (a spare row of the last pair tile when N/2 % 8 != 0) carries the
            // anchor row: its unfolded sum is anchor_op.F (the DMMA stream forms b0)
            if (r == half && k < half) return part == 0 ? af[k] : af[half + k];
            if (r >= half || k >= half) return 0.0;
            if (part == 0) return 0.5 * (mats->update_op(r, k) + mats->update_op(r, n - 1 - k));  // -> Y_r - Y_{N-1-r}
            const int pos = half + k;                                                           // a at pos >= N/2
            return 0.5 * (mats->update_op(r, n - 1 - pos) - mats->update_op(r, pos));          // -> Y_r + Y_{N-1-r}
        };
        std::vector<double> hf(static_cast<size_t>(np) * 2 * nkpf * 32 * 2);
        for (int m = 0; m < np; ++m)
            for (int part = 0; part < 2; ++part)
                for (int kp = 0; kp < nkpf; ++kp)
                    for (int lane = 0; lane < 32; ++lane) {
                        const int g = lane >> 2, q = lane & 3;
                        const size_t idx = ((static_cast<size_t>(m) * 2 + part) * nkpf + kp) * 32 + lane;
                        hf[2 * idx] = G(part, m * 8 + g, kp * 8 + q);
                        hf[2 * idx + 1] = G(part, m * 8 + g, kp * 8 + 4 + q);
                    }
        p->nkp_fold = nkpf;
        cuda_check(cudaMemcpy(p->fold.get<double>(hf.size()), hf.data(), hf.size() * sizeof(double),
                              cudaMemcpyHostToDevice),
                   "upload folded operators");
        cuda_check(cudaMemcpy(p->anc_fold.get<double>(af.size()), af.data(), af.size() * sizeof(double),
                              cudaMemcpyHostToDevice),
                   "upload folded anchor");
    }
    return *ctx->ops.emplace(n, std::move(p)).first->second;
}

/// Device body table of one call: flattened analytic elements / tabulated Chebyshev
/// segments (ephemeris.hpp:44-73) plus the names used in error messages.
struct BodyUpload {
    std::vector<int> kind, seg_off, ncoef;
    std::vector<double> elements, mu, bounds, coeffs;
    std::vector<long long> coeff_off;
    std::vector<std::string> names;
    int first_invalid = -1;  // first analytic body that elements_to_state rejects (kepler.hpp:103-106)
    std::string invalid_msg;
};

BodyUpload flatten_bodies(const pswarm_config& cfg, int nb) {
    BodyUpload u;
    u.seg_off.push_back(0);
    for (int b = 0; b < nb; ++b) {
        const pswarm_body& pb = cfg.bodies[b];
        u.names.push_back(pb.name ? pb.name : "");
        u.mu.push_back(pb.mu);
        u.kind.push_back(pb.kind == 0 ? 0 : 1);
        for (int k = 0; k < 7; ++k) u.elements.push_back(pb.kind == 0 ? pb.elements[k] : 0.0);
        u.ncoef.push_back(pb.kind == 0 ? 0 : pb.n_coeffs);
        if (pb.kind == 0) {
            const double ae = pb.elements[0], ee = pb.elements[1];
            if (u.first_invalid < 0 && (!(ae > 0.0) || ee < 0.0 || ee >= 1.0 - 1e-8)) {
                u.first_invalid = b;
                u.invalid_msg = "elements_to_state: elements do not define a bound conic (a = " + std::to_string(ae) +
                                ", e = " + std::to_string(ee) + ")";
            }
        } else {
            for (int sg = 0; sg < pb.n_segments; ++sg) {
                u.bounds.push_back(pb.seg_bounds[2 * sg]);
                u.bounds.push_back(pb.seg_bounds[2 * sg + 1]);
                u.coeff_off.push_back(static_cast<long long>(u.coeffs.size()));
                const double* c = pb.coeffs + static_cast<size_t>(sg) * 3 * pb.n_coeffs;
                u.coeffs.insert(u.coeffs.end(), c, c + 3 * pb.n_coeffs);
            }
        }
        u.seg_off.push_back(static_cast<int>(u.coeff_off.size()));
    }
    return u;
}

ForceData make_force_data(const double* pos, const double* mus, const double* indirect, double central_mu,
                          double floor_km, int n_bodies) {
    ForceData fd{};
    fd.body_pos = pos;
    fd.body_mu = mus;
    fd.indirect = indirect;
    fd.central_mu = central_mu;
    fd.floor_km = floor_km;
    fd.floor2_hi = floor_km * floor_km * (1.0 + 1e-9);
    std::memcpy(&fd.floor2_hi_bits, &fd.floor2_hi, sizeof(double));
    fd.n_bodies = n_bodies;
    return fd;
}

__global__ void k_read_timer(unsigned long long* out) { *out = globaltimer_ns(); }

template <typename T>
void upload(pswarm_ctx* ctx, BufId id, const T* host, size_t count, T** dev) {
    *dev = ctx->buf[id].get<T>(count);
    if (count) cuda_check(cudaMemcpyAsync(*dev, host, count * sizeof(T), cudaMemcpyHostToDevice, ctx->stream), "H2D");
}

// ------------------------------------------------------------- wide groups
/// One segment of groups larger than a CTA's slots (augmented / big grouped modes), solved on
/// the same persistent slot kernels as singleton groups.
///
/// A group's Picard iterates are column-separable: every member's update, force and error
/// depend on that member alone (augment.hpp:32-104); only the stopping rule couples them --
/// the group stops at the first iteration K where the max of its members' errors is <= tol
/// (pc_solve, picard.hpp:46-83), or at max_iterations, or at the first fault.  So the members
/// run as independent slots in rounds, each retiring with its full iterate saved in HBM:
///   round 0: every member stops at its own first crossing k_m (err <= tol);
///   round r: per group K_cand = max over members of their stop; members that stopped earlier
///            resume from the saved iterate and stop at the first k >= K_cand with err <= tol.
/// K_cand never passes K (below K_cand some member's error is above tol), so the rounds end
/// when every member of a group stops at the same K -- exactly the reference's K, with the
/// reference's arithmetic per member.  A member that hits max_iterations makes the others run
/// to max_iterations; a fault at iteration f makes every member that stopped before f run to f
/// so an earlier fault of another member is not missed.  The group's report, fault
/// coordinates (sample / column order of the whole group block) and error history are then
/// formed from the member records.  One round is the common case (a clone cloud converges in
/// step); each further round is one more launch over the lagging members only.
void solve_wide_rounds(pswarm_ctx* ctx, SegArgs a, const std::function<cudaError_t(const SegArgs&, int)>& launch,
                       int cta_cap, const std::vector<int64_t>& h_off, int64_t P, int max_it,
                       std::chrono::steady_clock::time_point deadline, int32_t* d_iter, double* d_err, uint8_t* d_conv,
                       GroupFault* d_faults, double* d_hist_seg, const int64_t* d_off, double& kernel_ms) {
    cudaStream_t st = ctx->stream;
    const int64_t M = a.M, N = a.N;
    // member reports: [M] iterations | converged | error, then [M] fault records
    Pack mp;
    const size_t o_it = mp.add(sizeof(int32_t) * M), o_cv = mp.add(M), o_er = mp.add(sizeof(double) * M),
                 o_head = mp.total, o_fl = mp.add(sizeof(GroupFault) * M);
    char* dm = ctx->buf[B_W_REP].get<char>(mp.total);
    char* hm = ctx->pin_wide.get<char>(mp.total);
    int32_t* d_list = ctx->buf[B_W_LIST].get<int32_t>(M);
    int32_t* d_ctl = ctx->buf[B_W_CTL].get<int32_t>(3 * M);  // it_start | floor | cap
    a.blk = ctx->buf[B_W_BLK].get<double>(static_cast<size_t>(M) * N * 6);
    a.rep_iter = reinterpret_cast<int32_t*>(dm + o_it);
    a.rep_conv = reinterpret_cast<uint8_t*>(dm + o_cv);
    a.rep_err = reinterpret_cast<double*>(dm + o_er);
    a.faults = reinterpret_cast<GroupFault*>(dm + o_fl);
    double* m_hist = d_hist_seg ? ctx->buf[B_W_HIST].get<double>(static_cast<size_t>(M) * max_it) : nullptr;
    a.rep_hist = m_hist;
    a.hist_stride = max_it;
    a.traj_list = d_list;
    a.gmax = 1;
    cuda_check(cudaMemsetAsync(dm, 0, mp.total, st), "memset member reports");
    cuda_check(launch_iota(d_list, static_cast<int>(M), st), "k_iota");
    ++ctx->launches;

    std::vector<int32_t> h_list, ctl(static_cast<size_t>(3 * M), 0);
    int32_t *c_start = ctl.data(), *c_floor = ctl.data() + M, *c_cap = ctl.data() + 2 * M;
    std::vector<uint8_t> decided(static_cast<size_t>(P), 0);
    std::vector<int32_t> g_iter(static_cast<size_t>(P), 0);
    std::vector<double> g_err(static_cast<size_t>(P), 0.0);
    std::vector<uint8_t> g_conv(static_cast<size_t>(P), 0);
    std::vector<GroupFault> g_fault(static_cast<size_t>(P));
    const int32_t* m_it = reinterpret_cast<const int32_t*>(hm + o_it);
    const uint8_t* m_cv = reinterpret_cast<const uint8_t*>(hm + o_cv);
    const double* m_er = reinterpret_cast<const double*>(hm + o_er);
    const GroupFault* m_fl = reinterpret_cast<const GroupFault*>(hm + o_fl);
    int64_t listed = M;
    ctx->wide_rounds = 0;
    for (int round = 0;; ++round) {
        // ---- launch the listed members
        a.P = static_cast<int>(listed);
        const bool ctl_on = round > 0;
        a.it_start = ctl_on ? d_ctl : nullptr;
        a.it_floor = ctl_on ? d_ctl + M : nullptr;
        a.it_cap = ctl_on ? d_ctl + 2 * M : nullptr;
        cuda_check(cudaMemsetAsync(a.queue, 0, sizeof(int), st), "memset queue");
        const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((listed + SLOTS - 1) / SLOTS, cta_cap)));
        cuda_check(cudaEventRecord(ctx->evk0, st), "event");
        cuda_check(launch(a, grid), "slot kernel launch (wide-group round)");
        cuda_check(cudaEventRecord(ctx->evk1, st), "event");
        ++ctx->launches;
        ++ctx->wide_rounds;
        cuda_check(cudaMemcpyAsync(hm, dm, o_head, cudaMemcpyDeviceToHost, st), "D2H member reports");
        cuda_check(cudaStreamSynchronize(st), "wide-group round");
        float kms = 0.f;
        cudaEventElapsedTime(&kms, ctx->evk0, ctx->evk1);
        kernel_ms += kms;
        bool any_fault = false;
        for (int64_t m = 0; m < M && !any_fault; ++m) any_fault = !m_cv[m];
        if (any_fault) {  // fault records only when some member stopped unconverged
            cuda_check(cudaMemcpyAsync(hm + o_fl, dm + o_fl, sizeof(GroupFault) * M, cudaMemcpyDeviceToHost, st), "D2H");
            cuda_check(cudaStreamSynchronize(st), "wide-group faults");
        }
        auto faulted = [&](int64_t m) { return any_fault && !m_cv[m] && m_fl[m].status != FAULT_NONE; };
        // ---- warm-start faults stop the batch before any solve (propagator.hpp:252-270)
        bool warm = false, timeout = std::chrono::steady_clock::now() > deadline;
        for (int64_t m = 0; m < M; ++m)
            if (faulted(m)) {
                warm |= m_fl[m].status == FAULT_WARM_ZERO_RADIUS || m_fl[m].status == FAULT_WARM_SOLVER;
                timeout |= m_fl[m].status == FAULT_TIMEOUT;
            }
        h_list.clear();
        for (int64_t g = 0; g < P; ++g) {
            if (decided[g]) continue;
            const int64_t lo = h_off[g], hi = h_off[g + 1], G = hi - lo;
            GroupFault& gf = g_fault[g];
            auto decide = [&](int32_t it, double err, bool conv) {
                decided[g] = 1;
                g_iter[g] = it;
                g_err[g] = err;
                g_conv[g] = conv ? 1 : 0;
            };
            if (warm) {  // the batch fails with the lowest warm-start fault (the caller picks it)
                gf = GroupFault{};
                for (int64_t m = lo; m < hi; ++m)
                    if (faulted(m) && (m_fl[m].status == FAULT_WARM_ZERO_RADIUS || m_fl[m].status == FAULT_WARM_SOLVER) &&
                        (gf.status == FAULT_NONE || m_fl[m].trajectory < gf.trajectory))
                        gf = m_fl[m];
                decide(0, 0.0, false);
                continue;
            }
            if (timeout) {  // a member cut by the device deadline, or never reached: the group timed out
                bool hit = false;
                int32_t itg = 0;
                for (int64_t m = lo; m < hi; ++m) {
                    hit |= (faulted(m) && m_fl[m].status == FAULT_TIMEOUT) || (!m_cv[m] && !faulted(m) && m_it[m] < max_it);
                    itg = std::max(itg, m_it[m]);
                }
                if (hit) {
                    gf = GroupFault{};
                    gf.status = FAULT_TIMEOUT;
                    gf.iteration = itg;
                    decide(itg, 0.0, false);
                    continue;
                }
                // every member stopped before the deadline: the group's outcome stands (below);
                // a further round would meet the device deadline and report the timeout there
            }
            // ---- earliest solve fault of the group (singularity / divergence)
            int32_t fmin = INT32_MAX;
            for (int64_t m = lo; m < hi; ++m)
                if (faulted(m)) fmin = std::min(fmin, m_fl[m].iteration);
            auto resume = [&](int64_t m, int32_t floor, int32_t cap) {
                c_start[m] = m_it[m];
                c_floor[m] = floor;
                c_cap[m] = cap;
                h_list.push_back(static_cast<int32_t>(m));
            };
            if (fmin != INT32_MAX) {
                bool pending = false;
                for (int64_t m = lo; m < hi; ++m)
                    if (!faulted(m) && m_it[m] < fmin) {
                        resume(m, fmin, fmin);
                        pending = true;
                    }
                if (pending) continue;
                // the group block's order at iteration fmin: singularity (sample = node * G + member,
                // force_model.hpp:93-142) before divergence ((node, column), column = comp * G + member)
                gf = GroupFault{};
                long long best_s = LLONG_MAX, best_d = LLONG_MAX;
                for (int64_t m = lo; m < hi; ++m) {
                    if (!faulted(m) || m_fl[m].iteration != fmin) continue;
                    const GroupFault& f = m_fl[m];
                    const int64_t mbr = m - lo;
                    if (f.status == FAULT_SINGULARITY) {
                        const long long key = f.node * G + mbr;
                        if (key < best_s) {
                            best_s = key;
                            gf = f;
                            gf.trajectory = mbr;
                        }
                    }
                }
                if (best_s == LLONG_MAX)
                    for (int64_t m = lo; m < hi; ++m) {
                        if (!faulted(m) || m_fl[m].iteration != fmin || m_fl[m].status != FAULT_DIVERGENCE) continue;
                        const long long key = m_fl[m].node * 6 * G + m_fl[m].column * G + (m - lo);
                        if (key < best_d) {
                            best_d = key;
                            gf = m_fl[m];
                            gf.column = m_fl[m].column * G + (m - lo);
                        }
                    }
                decide(fmin, 0.0, false);
                continue;
            }
            // ---- a member out of iterations: the whole group runs to max_iterations
            bool capped = false;
            for (int64_t m = lo; m < hi; ++m) capped |= !m_cv[m];
            if (capped) {
                bool pending = false;
                for (int64_t m = lo; m < hi; ++m)
                    if (m_it[m] < max_it) {
                        resume(m, max_it, max_it);
                        pending = true;
                    }
                if (pending) continue;
                double e = 0.0;
                for (int64_t m = lo; m < hi; ++m) e = std::max(e, m_er[m]);
                decide(max_it, e, false);
                continue;
            }
            // ---- every member below tol at its stop: the group stops at the latest one if all agree
            int32_t K = 0;
            for (int64_t m = lo; m < hi; ++m) K = std::max(K, m_it[m]);
            bool pending = false;
            for (int64_t m = lo; m < hi; ++m)
                if (m_it[m] < K) {
                    resume(m, K, max_it);
                    pending = true;
                }
            if (pending) continue;
            double e = 0.0;
            for (int64_t m = lo; m < hi; ++m) e = std::max(e, m_er[m]);
            decide(K, e, true);
        }
        if (h_list.empty()) break;
        // ---- next round: the lagging members only
        listed = static_cast<int64_t>(h_list.size());
        cuda_check(cudaMemcpyAsync(d_list, h_list.data(), sizeof(int32_t) * listed, cudaMemcpyHostToDevice, st), "H2D");
        cuda_check(cudaMemcpyAsync(d_ctl, ctl.data(), sizeof(int32_t) * 3 * M, cudaMemcpyHostToDevice, st), "H2D");
        a.cold_fallback = nullptr;  // written by round 0 (resumed members skip the warm start)
    }
    // ---- group reports into the segment's report block (the caller reads them back as usual)
    cuda_check(cudaMemcpyAsync(d_iter, g_iter.data(), sizeof(int32_t) * P, cudaMemcpyHostToDevice, st), "H2D");
    cuda_check(cudaMemcpyAsync(d_err, g_err.data(), sizeof(double) * P, cudaMemcpyHostToDevice, st), "H2D");
    cuda_check(cudaMemcpyAsync(d_conv, g_conv.data(), P, cudaMemcpyHostToDevice, st), "H2D");
    cuda_check(cudaMemcpyAsync(d_faults, g_fault.data(), sizeof(GroupFault) * P, cudaMemcpyHostToDevice, st), "H2D");
    if (d_hist_seg) {
        int32_t* d_gk = ctx->buf[B_W_GK].get<int32_t>(P);
        cuda_check(cudaMemcpyAsync(d_gk, g_iter.data(), sizeof(int32_t) * P, cudaMemcpyHostToDevice, st), "H2D");
        cuda_check(cudaMemsetAsync(d_hist_seg, 0, sizeof(double) * P * max_it, st), "memset");
        cuda_check(launch_group_hist(m_hist, max_it, d_off, static_cast<int>(P), d_gk, static_cast<int>(M), d_hist_seg, st),
                   "k_group_hist");
        ctx->launches += 2;
    }
    cuda_check(cudaStreamSynchronize(st), "wide-group reports");  // host vectors go out of scope
}

// ----------------------------------------------------------------- propagate
/// Lowest i with states[i].epoch != states[0].epoch (propagator.hpp:205-212), -1 if none.
/// The scan touches every cache line of the [M][7] batch; large batches are split over host
/// threads (56 MB at 10^6 states: ~4 ms on one core).
int64_t first_epoch_mismatch(const double* states, int64_t M) {
    auto scan = [&](int64_t lo, int64_t hi) {
        for (int64_t i = std::max<int64_t>(lo, 1); i < hi; ++i)
            if (states[7 * i] != states[0]) return i;
        return int64_t{-1};
    };
    const int64_t W = M >= (int64_t{1} << 17) ? std::min<int64_t>(8, std::max(1u, std::thread::hardware_concurrency())) : 1;
    if (W == 1) return scan(0, M);
    std::vector<int64_t> hit(static_cast<size_t>(W), -1);
    std::vector<std::thread> pool;
    for (int64_t w = 1; w < W; ++w) pool.emplace_back([&, w] { hit[w] = scan(M * w / W, M * (w + 1) / W); });
    hit[0] = scan(0, M / W);
    for (auto& t : pool) t.join();
    for (int64_t h : hit)
        if (h >= 0) return h;
    return -1;
}

struct RunSpec {
    bool independent = false;  // run_batch independent mode: reference error order is per trajectory
    // multi-device shards: leave the terminal states on the device and return their address
    // ([M][6] f64 in a context buffer, valid until the context's next call)
    const double** term_dev = nullptr;
    // independent mode: batch index of the trajectory whose error is raised (-1: none)
    int64_t* fail_index = nullptr;
};

/// PSWARM_TRACE=1: host-side stage times of propagate (diagnostics, stderr).
struct StageTrace {
    bool on = std::getenv("PSWARM_TRACE") != nullptr;
    std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
    void mark(const char* what) {
        if (!on) return;
        const auto now = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[pswarm] %-22s %8.3f ms\n", what, std::chrono::duration<double, std::milli>(now - t).count());
        t = now;
    }
};

void propagate_impl(pswarm_ctx* ctx, int64_t M, const double* states, int64_t P, const int64_t* group_sizes,
                    int64_t n_boundaries, const double* boundaries, int64_t N, const pswarm_config* cfg,
                    pswarm_outputs* out, const RunSpec& spec) {
    const auto wall0 = std::chrono::steady_clock::now();
    StageTrace trace;
    if (!cfg) raise(PSWARM_ERR_GENERIC, "propagate: null config");
    // ---- validation, same order and wording as propagator.hpp:196-216
    if (M <= 0) throw pswarm::InvalidPlanError("propagate: empty batch");
    int64_t total = 0, gmax = 0;
    for (int64_t g = 0; g < P; ++g) {
        if (group_sizes[g] < 1) throw pswarm::InvalidPlanError("plan_from_sizes: group sizes must be positive");
        total += group_sizes[g];
        gmax = std::max(gmax, group_sizes[g]);
    }
    if (total != M)
        throw pswarm::InvalidPlanError("propagate: grouping plan covers " + std::to_string(total) +
                                       " states, batch has " + std::to_string(M));
    const int64_t S = n_boundaries - 1;
    if (S < 1) throw pswarm::InvalidSpanError("propagate: empty segment plan");
    if (const int64_t i = first_epoch_mismatch(states, M); i >= 0)
        throw pswarm::AlignmentError("propagate: state " + std::to_string(i) + " epoch " +
                                     std::to_string(states[7 * i]) + " differs from shared epoch " +
                                     std::to_string(states[0]));
    if (states[0] != boundaries[0])
        throw pswarm::AlignmentError("propagate: batch epoch does not match the first segment boundary");
    if (cfg->tolerance <= 0.0) throw pswarm::Error("pc_solve: tolerance must be positive");
    if (N < 3) throw pswarm::InvalidSizeError("build_matrices: need at least 3 nodes, got " + std::to_string(N));
    if (!ctx) raise(PSWARM_ERR_NO_DEVICE, "propagate: no device context (the B200 path has no CPU fallback)");
    bind(ctx);
    const OpPack& op = operators(ctx, N);
    const int max_it = std::max(cfg->max_iterations, 0);
    if (cfg->force_kind < 0 || cfg->force_kind > 2)
        raise(PSWARM_ERR_INVALID_PLAN, "propagate: unknown force kind " + std::to_string(cfg->force_kind));
    if (cfg->start_mode < 0 || cfg->start_mode > 2)
        raise(PSWARM_ERR_INVALID_PLAN, "propagate: unknown start mode " + std::to_string(cfg->start_mode));
    const bool rel = cfg->force_kind == 2;  // EXTENSION: n_body + EIH 1PN
    const double c_light = cfg->c_light > 0.0 ? cfg->c_light : 299792.458;
    const int nb = cfg->force_kind >= 1 ? cfg->n_bodies : 0;
    if (nb > 63) raise(PSWARM_ERR_INVALID_SIZE, "propagate: at most 63 perturbing bodies are supported");
    const BodyUpload bu = flatten_bodies(*cfg, nb);

    // independent mode: every trajectory has a budget of its own (run_independent calls propagate
    // per trajectory, runner.hpp:63-80), charged on the device with the time it spends in its slots;
    // grouped / augmented: one propagate call, one deadline for the batch (propagator.hpp:233-236)
    const bool traj_budget = spec.independent && cfg->timeout_s > 0.0;
    const auto deadline = cfg->timeout_s > 0.0 && !traj_budget
                              ? std::chrono::steady_clock::now() +
                                    std::chrono::duration_cast<std::chrono::steady_clock::duration>(
                                        std::chrono::duration<double>(cfg->timeout_s))
                              : std::chrono::steady_clock::time_point::max();

    cudaStream_t st = ctx->stream;
    const int64_t R = 1 + S * (N - 1);
    // ---- Chebyshev-Gauss-Lobatto grids of every segment (host, exact reference arithmetic)
    std::vector<double> h_times(static_cast<size_t>(R), 0.0), seg_omega2(static_cast<size_t>(S));
    std::vector<double> grid_times(static_cast<size_t>(S * N));
    for (int64_t seg = 0; seg < S; ++seg) {
        const auto g = pswarm::build_grid(N, boundaries[seg], boundaries[seg + 1]);
        seg_omega2[seg] = g.omega2;
        std::memcpy(grid_times.data() + seg * N, g.times.data(), sizeof(double) * N);
        for (Index j = (seg == 0 ? 0 : 1); j < N; ++j) h_times[seg * (N - 1) + j] = g.times[j];
    }
    // ---- one packed host->device transfer: states, group offsets, grids, body table
    Pack in;
    // group offsets: not uploaded for singleton groups (independent mode), group gi = trajectory gi
    const bool unit_groups = gmax == 1;
    const size_t o_off = in.add(unit_groups ? 0 : sizeof(int64_t) * (P + 1)),
                 o_times = in.add(sizeof(double) * S * N), o_kind = in.add(sizeof(int) * bu.kind.size()),
                 o_soff = in.add(sizeof(int) * bu.seg_off.size()), o_nc = in.add(sizeof(int) * bu.ncoef.size()),
                 o_el = in.add(sizeof(double) * bu.elements.size()), o_mu = in.add(sizeof(double) * bu.mu.size()),
                 o_bnd = in.add(sizeof(double) * bu.bounds.size()),
                 o_coff = in.add(sizeof(long long) * bu.coeff_off.size()),
                 o_cf = in.add(sizeof(double) * bu.coeffs.size());
    const size_t o_s6 = in.add(sizeof(double) * M * 6);  // filled on the device (k_repack_states)
    char* hin = ctx->pin_in.get<char>(o_s6);
    {
        if (!unit_groups) {
            int64_t* off = reinterpret_cast<int64_t*>(hin + o_off);
            off[0] = 0;
            for (int64_t g = 0; g < P; ++g) off[g + 1] = off[g] + group_sizes[g];
        }
        auto put = [&](size_t o, const auto& v) {
            if (!v.empty()) std::memcpy(hin + o, v.data(), v.size() * sizeof(v[0]));
        };
        put(o_times, grid_times);
        put(o_kind, bu.kind);
        put(o_soff, bu.seg_off);
        put(o_nc, bu.ncoef);
        put(o_el, bu.elements);
        put(o_mu, bu.mu);
        put(o_bnd, bu.bounds);
        put(o_coff, bu.coeff_off);
        put(o_cf, bu.coeffs);
    }
    trace.mark("validate+grids+pack");
    char* din = ctx->buf[B_IN_PACK].get<char>(in.total);
    cuda_check(cudaMemcpyAsync(din, hin, o_s6, cudaMemcpyHostToDevice, st), "H2D inputs");
    {  // the caller's [M][7] states as they are; repacked to [M][6] on the device
        double* d7 = ctx->buf[B_STATES7].get<double>(static_cast<size_t>(M) * 7);
        cuda_check(cudaMemcpyAsync(d7, states, sizeof(double) * M * 7, cudaMemcpyHostToDevice, st), "H2D states");
        cuda_check(launch_repack_states(d7, reinterpret_cast<double*>(din + o_s6), M, st), "k_repack_states");
        ++ctx->launches;
    }
    double* d_in = reinterpret_cast<double*>(din + o_s6);
    const int64_t* d_off = unit_groups ? nullptr : reinterpret_cast<const int64_t*>(din + o_off);
    double* d_out = ctx->buf[B_STATE_B].get<double>(static_cast<size_t>(M) * 6);
    if (d_in == d_out) raise(PSWARM_ERR_GENERIC, "propagate: state buffers alias");
    double* d_samples = out && out->samples ? ctx->buf[B_SAMPLES].get<double>(static_cast<size_t>(M) * R * 6) : nullptr;
    if (ctx->poison_outputs) {  // test aid: unwritten outputs read back as NaN instead of stale values
        cuda_check(cudaMemsetAsync(d_out, 0xff, sizeof(double) * M * 6, ctx->stream), "poison");
        if (d_samples) cuda_check(cudaMemsetAsync(d_samples, 0xff, sizeof(double) * M * R * 6, ctx->stream), "poison");
    }
    const bool want_hist = out && out->error_history && max_it > 0;
    double* d_hist = want_hist ? ctx->buf[B_REP_HIST].get<double>(static_cast<size_t>(S) * P * max_it) : nullptr;
    if (d_hist) cuda_check(cudaMemsetAsync(d_hist, 0xff, sizeof(double) * S * P * max_it, st), "memset");
    // ---- per-segment report block: zeroed with one memset, read back with one copy
    Pack rp;
    // fault records last: they are read back only when some group did not converge
    const size_t r_queue = rp.add(16), r_iter = rp.add(sizeof(int32_t) * P), r_conv = rp.add(P), r_fb = rp.add(M),
                 r_err = rp.add(sizeof(double) * P), r_zero = rp.total, r_ekey = rp.add(sizeof(unsigned long long)),
                 r_faults = rp.add(sizeof(GroupFault) * P);
    char* drep = ctx->buf[B_REPORT].get<char>(rp.total);
    char* hrep = ctx->pin_rep.get<char>(rp.total);
    int* d_queue = reinterpret_cast<int*>(drep + r_queue);
    int32_t* d_iter = reinterpret_cast<int32_t*>(drep + r_iter);
    double* d_err = reinterpret_cast<double*>(drep + r_err);
    uint8_t* d_conv = reinterpret_cast<uint8_t*>(drep + r_conv);
    GroupFault* d_faults = reinterpret_cast<GroupFault*>(drep + r_faults);
    uint8_t* d_fb = reinterpret_cast<uint8_t*>(drep + r_fb);
    unsigned long long* d_ekey = reinterpret_cast<unsigned long long*>(drep + r_ekey);
    // terminal states: straight into a page-locked caller buffer as [M][7] (one DMA after a
    // device-side pack), else through the context's pinned staging
    bool term_direct = false;
    if (out && out->terminal_states) {
        cudaPointerAttributes pa{};
        term_direct = cudaPointerGetAttributes(&pa, out->terminal_states) == cudaSuccess && pa.type == cudaMemoryTypeHost;
        cudaGetLastError();
    }
    double* h_term =
        out && out->terminal_states && !term_direct ? ctx->pin_term.get<double>(sizeof(double) * M * 6) : nullptr;
    bool term_ready = false;

    // per-segment reports land straight in the caller's output arrays ([S][P], [S][M]) -- no
    // intermediate copy, and no fresh pages to fault in per call (C4: -2 x 14 MB of page faults)
    auto host_rows = [](auto* user, auto& buf, size_t n) {
        if (user) return user;
        if (buf.size() < n) buf.resize(n);
        return buf.data();
    };
    int32_t* h_iter = host_rows(out ? out->iterations : nullptr, ctx->host_iter, static_cast<size_t>(S * P));
    double* h_err = host_rows(out ? out->final_error : nullptr, ctx->host_err, static_cast<size_t>(S * P));
    uint8_t* h_conv = host_rows(out ? out->converged : nullptr, ctx->host_conv, static_cast<size_t>(S * P));
    uint8_t* h_fb = host_rows(out ? out->cold_fallback : nullptr, ctx->host_fb, static_cast<size_t>(S * M));
    std::vector<GroupFault> h_faults;  // sized on the first segment that needs fault records

    // device deadline in %globaltimer units
    unsigned long long gpu_deadline = 0;
    unsigned long long* d_tns = nullptr;
    if (traj_budget) {
        d_tns = ctx->buf[B_TRAJ_NS].get<unsigned long long>(static_cast<size_t>(M));
        cuda_check(cudaMemsetAsync(d_tns, 0, sizeof(unsigned long long) * M, st), "memset budgets");
    } else if (cfg->timeout_s > 0.0) {
        unsigned long long* d_t = reinterpret_cast<unsigned long long*>(ctx->buf[B_OP_KEY].get<double>(1));
        k_read_timer<<<1, 1, 0, st>>>(d_t);
        ++ctx->launches;
        unsigned long long t0 = 0;
        cuda_check(cudaMemcpyAsync(&t0, d_t, sizeof t0, cudaMemcpyDeviceToHost, st), "timer");
        cuda_check(cudaStreamSynchronize(st), "timer sync");
        const auto left = std::chrono::duration_cast<std::chrono::nanoseconds>(deadline - std::chrono::steady_clock::now());
        gpu_deadline = t0 + static_cast<unsigned long long>(std::max<int64_t>(left.count(), 1));
    }

    // kernel choice -- by N, the force model and the options only, never by the grouping, so
    // every grouping (and every multi-device shard) runs the same per-trajectory arithmetic:
    // the warp-specialised slot kernel when N is in its tile range, else the generic one.
    // Groups up to the kernel's in-CTA limit (4 / 8 members) take their decisions in the
    // kernel; larger ones run as member-level rounds on the same kernel (solve_wide_rounds).
    constexpr size_t SMEM_MAX = 227 * 1024 - 1024;  // opt-in limit minus the kernels' static __shared__ (< 1 KB)
    const int Ni = static_cast<int>(N);
    // mirror-folded update when N allows it (half the DMMAs); "fold" option 0 forces the dense one
    const bool fold = ctx->fold && op.nkp_fold > 0 && ws_supported(Ni, true) && ctx->slot_kernel != 1 &&
                      ws_smem_bytes(Ni, op.nkp, ws_extra_rows(Ni, true), nb, 0, true) <= SMEM_MAX;
    const bool use_ws = fold || (ws_supported(Ni, false) && ctx->slot_kernel != 1 &&
                                 ws_smem_bytes(Ni, op.nkp, ws_extra_rows(Ni, false), nb, 0, false) <= SMEM_MAX);
    const bool wide = gmax > (use_ws ? SLOTS / 2 : SLOTS);
    const int64_t gk = wide ? 1 : gmax;  // group size the slot kernel sees
    const int xrows = use_ws ? ws_extra_rows(Ni, fold) : extra_rows(Ni, op.gp);
    // auto: the unified kernel for the force-bound 1PN model (node-major force items: 1PN kernel
    // time 15.0 vs 19.2 ms at N = 200, 17.8 vs 27.0 ms at N = 256 against k_pc_ws_fold,
    // profiles/sanitizer_r02.json run); Newtonian forces stay on the warp-specialised kernel, except
    // N = 80...96 and 112...128: the unified kernel's two-CTA variant beats k_pc_ws_fold.x2 by 2 / 10 / 12 %
    // at N = 80 / 88 / 96, 1 / 0.4 % at 112 / 120, and the 512-thread k_pc_ws_fold by 3.7 % at 128 (+7 % at
    // 72, +1 % at 104; tools/probe_ab_opt.py unified, tools/probe_ab_uni_small.py)
    const bool uni_newton = ctx->small_ctas && ((Ni >= 80 && Ni <= 96) || (Ni >= 112 && Ni <= 128));
    const bool uni = fold && (ctx->unified == 1 || (ctx->unified == 2 && (rel || uni_newton))) && uni_supported(Ni);
    // small N: the 256-thread variants of the same kernels (4 + 4 warps, pswarm_dev::small) run two
    // CTAs per SM, so one CTA's barrier / decision / claim latencies overlap the other's work;
    // each CTA's shared memory must leave room for the second
    constexpr size_t SMEM_PAIR = 228 * 1024 / 2 - 2 * 1024;
    bool small_k = false;
    int small_stage = 0, small_xrows = 0;
    // measured (tools/probe_ab_opt.py small_ctas / small_max_n): Newtonian -32 % kernel time at N = 64,
    // -10 % at 96, -13 / -6 / -4 % at 104 / 112 / 120, +1 % at 128; 1PN -16 % at 64, +1 % at 96, -6 % at 128
    const int small_max = ctx->small_max_n > 0 ? ctx->small_max_n : (rel || uni ? 128 : 120);
    if (ctx->small_ctas && fold && Ni <= small_max && small::ws_supported(Ni, true) &&
        (!uni || small::uni_supported(Ni))) {
        small_xrows = uni ? 0 : small::ws_extra_rows(Ni, true);
        auto bytes = [&](int stg) { return small::ws_smem_bytes(Ni, op.nkp, small_xrows, nb, stg, true, rel && uni); };
        if (bytes(0) <= SMEM_PAIR) {
            small_k = true;
            // (1PN: the two CTAs read the node table from L1 at least as fast as from their own
            // staged copies: -4 % kernel time unstaged at N = 64, tie at 128)
            small_stage = !rel && nb > 0 && bytes(1) <= SMEM_PAIR ? 1 : 0;
        }
    }
    ctx->last_kernel = small_k ? (uni ? "k_pc_uni.x2" : "k_pc_ws_fold.x2")
                       : uni   ? "k_pc_uni"
                       : fold  ? "k_pc_ws_fold"
                       : use_ws ? "k_pc_ws"
                                : "k_pc_segment";
    // stage the frozen ephemeris in shared memory when it fits next to the state blocks (the
    // slot kernels copy it with the TMA unit); relativistic: the node table, k_pc_uni only
    const int stage_eph = !ctx->stage ? 0
                          : small_k ? small_stage
                          : rel   ? (uni && ws_smem_bytes(Ni, op.nkp, 0, nb, 1, true, true) <= SMEM_MAX ? 1 : 0)
                                  : (nb > 0 && (use_ws ? ws_smem_bytes(Ni, op.nkp, xrows, nb, 1, fold)
                                                       : segment_smem_bytes(Ni, op.nkp, xrows, nb, 1)) <= SMEM_MAX
                                         ? 1
                                         : 0);
    if (!use_ws && segment_smem_bytes(Ni, op.nkp, xrows, nb, stage_eph) > SMEM_MAX)
        raise(PSWARM_ERR_INVALID_SIZE, fmtf("propagate: %lld nodes exceed the per-SM shared memory of the slot kernel",
                                            (long long)N));
    const int per_cta = static_cast<int>(SLOTS / gk);
    const int cap = ctx->max_ctas > 0 ? ctx->max_ctas : ctx->sm_count * (small_k ? 2 : ctx->ctas_per_sm);
    auto grid_for = [&](int64_t groups) {
        const int64_t want_ctas = (groups + per_cta - 1) / per_cta;
        return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(want_ctas, cap)));
    };

    BodyTable bt{};
    double *d_pos = nullptr, *d_ind = nullptr, *d_mu = nullptr, *d_eph_t = nullptr;
    if (nb > 0) {
        d_mu = reinterpret_cast<double*>(din + o_mu);
        bt = BodyTable{nb,
                       reinterpret_cast<int*>(din + o_kind),
                       reinterpret_cast<double*>(din + o_el),
                       d_mu,
                       reinterpret_cast<int*>(din + o_soff),
                       reinterpret_cast<double*>(din + o_bnd),
                       reinterpret_cast<long long*>(din + o_coff),
                       reinterpret_cast<int*>(din + o_nc),
                       reinterpret_cast<double*>(din + o_cf)};
        d_pos = ctx->buf[B_BODY_POS].get<double>(static_cast<size_t>(N) * nb * 3);
        d_ind = ctx->buf[B_INDIRECT].get<double>(static_cast<size_t>(N) * 3);
        // node-contiguous copy: the bulk-staging source, or (option eph_nc) read from global
        if (use_ws && !rel && (stage_eph || ctx->eph_nc))
            d_eph_t = ctx->buf[B_EPH_T].get<double>(eph_stage_doubles(Ni, nb, false));
    }
    double* d_hot = cfg->start_mode == 2 ? ctx->buf[B_HOT].get<double>(static_cast<size_t>(M) * N * 6) : nullptr;
    double *d_vel = nullptr, *d_rel = nullptr;
    if (rel) {  // EXTENSION: body velocities + per-node relativistic table (Sun row first)
        bt.B = nb;
        d_vel = ctx->buf[B_BODY_VEL].get<double>(static_cast<size_t>(N) * std::max(nb, 1) * 3);
        d_rel = ctx->buf[B_REL_TAB].get<double>(eph_stage_doubles(Ni, nb, true));
        if (!d_pos) d_pos = ctx->buf[B_BODY_POS].get<double>(static_cast<size_t>(N) * 3);
        if (!d_ind) d_ind = ctx->buf[B_INDIRECT].get<double>(static_cast<size_t>(N) * 3);
    }
    unsigned long long* d_phase = nullptr;
    if (ctx->profile_phases) {
        d_phase = ctx->buf[B_PHASES].get<unsigned long long>(PHASES);
        cuda_check(cudaMemsetAsync(d_phase, 0, sizeof(unsigned long long) * PHASES, st), "memset");
    }
    cuda_check(cudaEventRecord(ctx->ev0, st), "event");
    int64_t seg_done = 0;
    // ---- samples into a pinned host buffer: copy each segment's rows as soon as its kernel
    //      finishes, on a second stream, overlapping the next segment
    bool overlap_samples = false;
    if (out && out->samples && S > 1) {
        cudaPointerAttributes pa{};
        overlap_samples = cudaPointerGetAttributes(&pa, out->samples) == cudaSuccess && pa.type == cudaMemoryTypeHost;
        cudaGetLastError();
        if (overlap_samples && !ctx->copy_stream) {
            cuda_check(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking), "cudaStreamCreate");
            cuda_check(cudaEventCreateWithFlags(&ctx->ev_seg, cudaEventDisableTiming), "cudaEventCreate");
        }
    }
    struct CopySync {  // the copy stream never outlives the call (also on error paths)
        cudaStream_t s;
        ~CopySync() {
            if (s) cudaStreamSynchronize(s);
        }
    } copy_sync{overlap_samples ? ctx->copy_stream : nullptr};
    double kernel_ms = 0.0;
    int64_t traj_iters = 0;
    std::string fail_msg;
    int32_t fail_status = PSWARM_OK;
    pswarm_error fail{};
    init_err(&fail, PSWARM_OK, "");
    // run_independent (runner.hpp:63-80) solves trajectory after trajectory, so the error the
    // caller sees is the one of the LOWEST failing trajectory, whichever segment it fails in.
    // Segment-synchronous processing meets the failures segment by segment: on the first one
    // the lowest failing index c becomes pending and only trajectories [0, c) keep going; a
    // failure among them in a later segment replaces it.  The partial outputs stay those of
    // the first failing segment (every trajectory has rows up to there).
    int64_t P_act = P, M_act = M;
    bool pend = false;
    pswarm_error pend_err{};
    int64_t pend_rep = 0, pend_done = 0;

    for (int64_t seg = 0; seg < S; ++seg) {
        const double* seg_times = grid_times.data() + seg * N;
        if (std::chrono::steady_clock::now() > deadline) {
            init_err(&fail, PSWARM_ERR_TIMEOUT, "solve_group: wall-clock budget exhausted in group 0");
            fail.segment = seg;
            fail.group = 0;
            fail_status = PSWARM_ERR_TIMEOUT;
            break;
        }
        const double* d_times = reinterpret_cast<const double*>(din + o_times) + seg * N;
        cuda_check(cudaMemsetAsync(drep, 0, r_zero, st), "memset reports");
        cuda_check(cudaMemsetAsync(d_ekey, 0xff, sizeof(unsigned long long), st), "memset");
        cuda_check(cudaMemsetAsync(d_faults, 0, sizeof(GroupFault) * P, st), "memset faults");
        if (nb > 0 || rel) {  // frozen per-node ephemeris of this segment, evaluated on the device
            cuda_check(launch_ephemeris(static_cast<int>(N), d_times, cfg->central_mu, bt, d_pos, d_ind, d_ekey, d_vel,
                                        d_rel, 1.0 / (c_light * c_light), d_eph_t, st),
                       "k_ephemeris");
            ++ctx->launches;
        }

        SegArgs a{};
        a.N = static_cast<int>(N);
        a.nkp = op.nkp;
        a.gp = op.gp;
        a.xrows = small_k ? small_xrows : xrows;
        a.stage_eph = stage_eph;
        a.M = static_cast<int>(M_act);
        a.P = static_cast<int>(P_act);
        a.gmax = static_cast<int>(gk);
        a.seg = static_cast<int>(seg);
        a.cold_start = (seg == 0 && cfg->start_mode == 1) ? 1 : 0;
        a.error_mode = cfg->error_mode;
        a.max_it = max_it;
        a.record_history = d_hist ? 1 : 0;
        a.tol = cfg->tolerance;
        a.tol2_lo = cfg->tolerance * cfg->tolerance * (1.0 - 1e-13);
        a.tol2_hi = cfg->tolerance * cfg->tolerance * (1.0 + 1e-13);
        a.omega2 = seg_omega2[seg];
        a.epoch = boundaries[seg];
        a.deadline_ns = gpu_deadline;
        a.fd = make_force_data(d_pos, d_mu, d_ind, cfg->central_mu, cfg->proximity_floor_km, nb);
        if (rel) {
            a.fd.rel = 1;
            a.fd.ic2 = 1.0 / (c_light * c_light);
            a.fd.rel_tab = d_rel;
        }
        a.fd.eph_t = d_eph_t;
        a.upack = reinterpret_cast<const double2*>(op.buf.p);
        a.times = d_times;
        a.group_off = d_off;
        a.state_in = d_in;
        a.state_out = d_out;
        a.samples = d_samples;
        a.R = R;
        a.row0 = seg * (N - 1);
        a.queue = d_queue;
        a.rep_iter = d_iter;
        a.rep_err = d_err;
        a.rep_conv = d_conv;
        a.rep_hist = d_hist ? d_hist + static_cast<size_t>(seg) * P * max_it : nullptr;
        a.faults = d_faults;
        a.cold_fallback = d_fb;
        a.hot = d_hot;  // EXTENSION: hot start corrections, persistent across segments
        a.hot_apply = d_hot && seg >= 1 &&
                      std::abs((boundaries[seg + 1] - boundaries[seg]) - (boundaries[seg] - boundaries[seg - 1])) <=
                          1e-9 * std::abs(boundaries[seg] - boundaries[seg - 1]);
        a.phase_cycles = d_phase;
        a.upack_fold = fold ? reinterpret_cast<const double2*>(op.fold.p) : nullptr;
        a.nkp_fold = op.nkp_fold;
        // auto: the FP group forms b0 itself at N = 168...200 -- k_pc_ws_fold kernel time -1.3 % on C4
        // (1M ICs, N = 200), -1.8 % on C2, -1.1 / -1.5 % at N = 168 / 184; the anchor pair row of the
        // DMMA stream everywhere else (+4...7 % without it at N = 120...152 and 216...248;
        // tools/probe_ab_c4.py, tools/probe_ab_opt.py b0_mma)
        a.b0_mma = ctx->b0_mma == 2 ? !(Ni >= 168 && Ni <= 200) : ctx->b0_mma;
        a.fast_decide = ctx->fast_decide;
        a.force_ns = ctx->force_ns;
        if (a.force_ns == 0 && uni && rel) {
            // relativistic k_pc_uni force items: 1 slot (one chain) or 2 (two fused chains) per item,
            // whichever needs fewer rounds of the block's threads weighted by the item cost (a
            // 2-chain item ~1.8x a 1-chain one) -- fits every 1PN N measured from 64 to 256
            // (tools/probe_ab_opt.py force_ns): e.g. N = 160, 640 two-chain items = 2 rounds of 512
            // threads vs 1280 one-chain items = 3 rounds -> one chain, -4.5 % kernel time.  Chosen
            // here, not in the kernel: ptxas' register allocation of the whole kernel moved (+1 %
            // elsewhere) when the kernel computed it.
            const int T = small_k ? 256 : 512;
            const int r1 = (8 * Ni + T - 1) / T, r2 = (4 * Ni + T - 1) / T;
            a.force_ns = 10 * r1 <= 18 * r2 ? 1 : 2;
        } else if (a.force_ns == 0 && small_k && !uni) {
            // k_pc_ws_fold.x2 (128 FP threads): single-slot items up to N = 80 (the kernel's own
            // threshold is N = 64): -6.6 % / -9.7 % kernel time at N = 72 / 80, two-slot items
            // from N = 88 (tools/probe_ab_opt.py force_ns)
            a.force_ns = Ni / 2 > 40 ? 2 : 1;
        }
        a.anc_fold = fold ? reinterpret_cast<const double*>(op.anc_fold.p) : nullptr;
        a.hist_stride = max_it;
        a.traj_ns = d_tns;
        a.traj_budget_ns = traj_budget ? static_cast<unsigned long long>(std::min(cfg->timeout_s * 1e9, 1.8e19)) : 0ull;
        auto launch = [&](const SegArgs& x, int grid) {
            if (small_k) return uni ? small::launch_segment_uni(x, grid, st) : small::launch_segment_ws(x, grid, st);
            return uni ? launch_segment_uni(x, grid, st) : use_ws ? launch_segment_ws(x, grid, st) : launch_segment(x, grid, st);
        };
        if (max_it > 0 && !wide) {
            cuda_check(cudaEventRecord(ctx->evk0, st), "event");
            cuda_check(launch(a, grid_for(P_act)), "slot kernel launch");
            cuda_check(cudaEventRecord(ctx->evk1, st), "event");
            ++ctx->launches;
        } else if (max_it > 0) {
            std::vector<int64_t> h_off(static_cast<size_t>(P) + 1, 0);
            for (int64_t g = 0; g < P; ++g) h_off[g + 1] = h_off[g] + group_sizes[g];
            solve_wide_rounds(ctx, a, launch, cap, h_off, P, max_it, deadline, d_iter, d_err, d_conv, d_faults,
                              a.rep_hist, d_off, kernel_ms);
        }
        if (overlap_samples) {  // rows [row0 + jb, row0 + N - 1] of every trajectory, pitch R rows
            const int64_t jb = seg == 0 ? 0 : 1, row = seg * (N - 1) + jb, nrows = N - jb;
            const size_t pitch = sizeof(double) * 6 * R;
            cuda_check(cudaEventRecord(ctx->ev_seg, st), "event");
            cuda_check(cudaStreamWaitEvent(ctx->copy_stream, ctx->ev_seg, 0), "wait");
            cuda_check(cudaMemcpy2DAsync(out->samples + row * 6, pitch, d_samples + row * 6, pitch,
                                         sizeof(double) * 6 * nrows, M, cudaMemcpyDeviceToHost, ctx->copy_stream),
                       "D2H segment samples");
        }
        cuda_check(cudaMemcpyAsync(hrep, drep, r_faults, cudaMemcpyDeviceToHost, st), "D2H reports");
        if (h_term && seg == S - 1) {  // terminal states ride along with the last segment's reports
            cuda_check(cudaMemcpyAsync(h_term, d_out, sizeof(double) * M * 6, cudaMemcpyDeviceToHost, st), "D2H terminal");
            term_ready = true;
        }
        if (term_direct && seg == S - 1) {
            double* d7 = ctx->buf[B_STATES7].get<double>(static_cast<size_t>(M) * 7);  // input copy: consumed
            cuda_check(launch_pack_states7(d_out, boundaries[S], d7, M, st), "k_pack_states7");
            ++ctx->launches;
            cuda_check(cudaMemcpyAsync(out->terminal_states, d7, sizeof(double) * M * 7, cudaMemcpyDeviceToHost, st),
                       "D2H terminal");
            term_ready = true;
        }
        cuda_check(cudaStreamSynchronize(st), "segment solve");
        trace.mark("segment sync");
        std::memcpy(h_iter + seg * P, hrep + r_iter, sizeof(int32_t) * P);
        std::memcpy(h_err + seg * P, hrep + r_err, sizeof(double) * P);
        std::memcpy(h_conv + seg * P, hrep + r_conv, P);
        std::memcpy(h_fb + seg * M, hrep + r_fb, M);
        // fault records (48 B per group) only when some group stopped unconverged: every fault
        // retires its group with converged = 0 (the wide rounds write their group records so too)
        bool any_unconverged = false;
        for (int64_t gi = 0; gi < P_act && !any_unconverged; ++gi) any_unconverged = !h_conv[seg * P + gi];
        const bool need_faults = any_unconverged;
        if (need_faults) {
            h_faults.resize(static_cast<size_t>(P));
            cuda_check(cudaMemcpyAsync(h_faults.data(), drep + r_faults, sizeof(GroupFault) * P, cudaMemcpyDeviceToHost,
                                       st),
                       "D2H faults");
            cuda_check(cudaStreamSynchronize(st), "faults");
        }
        unsigned long long ekey;
        std::memcpy(&ekey, hrep + r_ekey, sizeof ekey);
        // ---- ephemeris faults come first: build_ephemeris_cache precedes the solve
        //      (propagator.hpp:252); body-major order (ephemeris.hpp:96-105)
        {
            const long long eb = ekey == ~0ull ? LLONG_MAX : static_cast<long long>((ekey / 4) / N);
            if (seg == 0 && bu.first_invalid >= 0 && bu.first_invalid < eb) {
                init_err(&fail, PSWARM_ERR_NON_ELLIPTIC, bu.invalid_msg);
                fail.segment = seg;
                fail_status = fail.status;
                break;
            }
            if (ekey != ~0ull) {
                const int kind = static_cast<int>(ekey % 4);
                const int b = static_cast<int>((ekey / 4) / N), j = static_cast<int>((ekey / 4) % N);
                if (kind == 1) {
                    init_err(&fail, PSWARM_ERR_COVERAGE,
                             "ephemeris for body '" + bu.names[b] + "' does not cover epoch " +
                                 std::to_string(seg_times[j]));
                    fail.value = seg_times[j];
                } else {
                    init_err(&fail, PSWARM_ERR_SOLVER, "solve_kepler: Newton iteration did not converge for body '" +
                                                           bu.names[b] + "'");
                }
                fail.segment = seg;
                fail.body = b;
                fail_status = fail.status;
                break;
            }
        }
        if (max_it > 0 && !wide) {  // (the wide rounds add their own launches)
            float kms = 0.f;
            cudaEventElapsedTime(&kms, ctx->evk0, ctx->evk1);
            kernel_ms += kms;
        }
        for (int64_t gi = 0; gi < P_act; ++gi) traj_iters += static_cast<int64_t>(h_iter[seg * P + gi]) * group_sizes[gi];

        // ---- the reference exception of one group's record (warm start, solve faults, timeout)
        auto fault_error = [&](const GroupFault& f, int64_t gi, int64_t report_g, pswarm_error& e) {
            if (f.status == FAULT_WARM_ZERO_RADIUS) {
                init_err(&e, PSWARM_ERR_SINGULARITY, "kepler_propagate: zero-radius state");
                e.trajectory = f.trajectory;
            } else if (f.status == FAULT_WARM_SOLVER) {
                init_err(&e, PSWARM_ERR_SOLVER,
                         "solve_kepler: Newton iteration did not converge for M = " + std::to_string(f.value) +
                             ", e = " + std::to_string(f.value2));
                e.trajectory = f.trajectory;
            } else if (f.status == FAULT_DIVERGENCE) {
                init_err(&e, PSWARM_ERR_DIVERGENCE,
                         "group " + std::to_string(report_g) + ": picard iteration produced a non-finite value at node " +
                             std::to_string(f.node) + ", column " + std::to_string(f.column));
                e.node = f.node;
                e.column = f.column;
            } else if (f.status == FAULT_SINGULARITY) {
                std::string what, body;
                if (f.body < 0) {
                    what = "central-body acceleration at zero radius";
                } else {
                    body = bu.names[f.body];
                    what = "close approach to body '" + body + "': distance " + std::to_string(f.value) +
                           " km below floor " + std::to_string(cfg->proximity_floor_km) + " km";
                }
                init_err(&e, PSWARM_ERR_SINGULARITY,
                         "node " + std::to_string(f.node) + ", trajectory " + std::to_string(f.trajectory) + ": " + what);
                std::snprintf(e.body_name, sizeof e.body_name, "%s", body.c_str());
                e.body = f.body;
                e.node = f.node;
                e.trajectory = f.trajectory;
                e.value = f.value;
            } else {
                init_err(&e, PSWARM_ERR_TIMEOUT,
                         "solve_group: wall-clock budget exhausted in group " + std::to_string(report_g));
            }
            if (f.status != FAULT_WARM_ZERO_RADIUS && f.status != FAULT_WARM_SOLVER) {
                e.group = spec.independent ? 0 : gi;
                e.iterations = f.iteration;
            }
            e.segment = seg;
        };
        // ---- non-convergence (propagator.hpp:300-312)
        auto incomplete_error = [&](int64_t gi, pswarm_error& e) {
            const int64_t report_g = spec.independent ? 0 : gi;
            init_err(&e, PSWARM_ERR_INCOMPLETE,
                     "propagate: group " + std::to_string(report_g) + " did not converge in segment " +
                         std::to_string(seg) + " (error " + std::to_string(h_err[seg * P + gi]) + " after " +
                         std::to_string(h_iter[seg * P + gi]) + " iterations)");
            e.segment = seg;
            e.group = report_g;
            e.trajectory = spec.independent ? gi : -1;
            e.iterations = h_iter[seg * P + gi];
            e.value = h_err[seg * P + gi];
        };
        const auto solve_fault = [&](int64_t gi) {
            return need_faults && h_faults[gi].status != FAULT_NONE &&
                   (max_it > 0 || h_faults[gi].status == FAULT_WARM_ZERO_RADIUS ||
                    h_faults[gi].status == FAULT_WARM_SOLVER);
        };

        if (spec.independent) {
            // run_independent (runner.hpp:63-80): the lowest trajectory that fails in ANY way --
            // warm start, solve fault or plain non-convergence (every fault retires its group
            // with converged = 0) -- is the one the serial reference raises for
            int64_t c = -1;
            for (int64_t gi = 0; gi < P_act; ++gi)
                if (!h_conv[seg * P + gi]) {
                    c = gi;
                    break;
                }
            if (c >= 0) {
                if (solve_fault(c))
                    fault_error(h_faults[c], c, 0, pend_err);
                else
                    incomplete_error(c, pend_err);
                if (!pend) {  // partial outputs: every trajectory up to the first failing segment
                    pend_rep = pend_err.status == PSWARM_ERR_INCOMPLETE ? seg + 1 : seg;
                    pend_done = seg;
                }
                pend = true;
                if (spec.fail_index) *spec.fail_index = c;
                if (c == 0 || seg == S - 1) break;  // no lower trajectory is left to fail later
                P_act = M_act = c;                  // only trajectories [0, c) continue
            }
            std::swap(d_in, d_out);
            if (!pend) {
                seg_done = seg + 1;
                if (out) out->segments_reported = seg + 1;
            }
            continue;
        }

        // ---- grouped / augmented: propagate's order -- warm start of the whole batch first
        //      (lowest trajectory), then the groups' solves in group order
        int64_t warm_traj = -1, warm_g = -1, first_g = -1;
        for (int64_t gi = 0; gi < (need_faults ? P : 0); ++gi) {
            const GroupFault& f = h_faults[gi];
            if (f.status == FAULT_WARM_ZERO_RADIUS || f.status == FAULT_WARM_SOLVER) {
                if (warm_traj < 0 || f.trajectory < warm_traj) {
                    warm_traj = f.trajectory;
                    warm_g = gi;
                }
            } else if (f.status != FAULT_NONE && first_g < 0) {
                first_g = gi;
            }
        }
        if (max_it == 0 && P > 0) first_g = -1;
        if (warm_g >= 0 || first_g >= 0) {
            fault_error(h_faults[warm_g >= 0 ? warm_g : first_g], warm_g >= 0 ? warm_g : first_g,
                        warm_g >= 0 ? warm_g : first_g, fail);
            fail_status = fail.status;
            break;
        }
        int64_t nc = -1;
        for (int64_t gi = 0; gi < P; ++gi)
            if (!h_conv[seg * P + gi]) {
                nc = gi;
                break;
            }
        if (nc >= 0) {
            incomplete_error(nc, fail);
            fail_status = PSWARM_ERR_INCOMPLETE;
            seg_done = seg;
            if (out) out->segments_reported = seg + 1;
            break;
        }
        std::swap(d_in, d_out);
        seg_done = seg + 1;
        if (out) out->segments_reported = seg + 1;
    }
    if (pend && fail_status == PSWARM_OK) {  // independent mode: the lowest failing trajectory
        fail = pend_err;
        fail_status = pend_err.status;
    }
    if (pend) {
        seg_done = std::min(seg_done, pend_done);
        if (out) out->segments_reported = pend_rep;
    }
    cuda_check(cudaEventRecord(ctx->ev1, st), "event");
    trace.mark("segments (device+host)");
    if (spec.term_dev) *spec.term_dev = fail_status == PSWARM_OK ? d_in : nullptr;

    // ---- outputs
    if (out) {
        out->segments_completed = seg_done;
        if (fail_status != PSWARM_OK && fail_status != PSWARM_ERR_INCOMPLETE) out->segments_reported = seg_done;
        if (out->times) std::memcpy(out->times, h_times.data(), sizeof(double) * R);
        const int64_t rep = out->segments_reported;
        (void)rep;  // iterations / final_error / converged / cold_fallback were written per segment
        if (out->error_history && max_it > 0 && rep > 0)
            cuda_check(cudaMemcpyAsync(out->error_history, d_hist, sizeof(double) * rep * P * max_it,
                                       cudaMemcpyDeviceToHost, st),
                       "D2H history");
        if (out->samples && !overlap_samples)
            cuda_check(cudaMemcpyAsync(out->samples, d_samples, sizeof(double) * M * R * 6, cudaMemcpyDeviceToHost, st),
                       "D2H samples");
        if (overlap_samples) cuda_check(cudaStreamSynchronize(ctx->copy_stream), "segment samples");
        if (h_term && fail_status == PSWARM_OK && !term_ready) {
            cuda_check(cudaMemcpyAsync(h_term, d_in, sizeof(double) * M * 6, cudaMemcpyDeviceToHost, st),
                       "D2H terminal");
        }
        if (d_phase)
            cuda_check(cudaMemcpyAsync(ctx->phase_host, d_phase, sizeof(unsigned long long) * PHASES,
                                       cudaMemcpyDeviceToHost, st),
                       "D2H phases");
        cuda_check(cudaStreamSynchronize(st), "outputs");
        if (h_term && fail_status == PSWARM_OK)
            for (int64_t i = 0; i < M; ++i) {
                out->terminal_states[7 * i] = boundaries[S];
                for (int c = 0; c < 6; ++c) out->terminal_states[7 * i + 1 + c] = h_term[i * 6 + c];
            }
        float ms = 0.f;
        cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1);
        out->device_ms = ms;
        out->kernel_ms = kernel_ms;
        out->trajectory_iterations = traj_iters;
        out->gpu_launches = ctx->launches;
        out->wall_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - wall0).count();
        trace.mark("outputs");
    }
    if (fail_status != PSWARM_OK) {
        CapiFault f;
        f.e = fail;
        throw f;
    }
}

}  // namespace

// =================================================================== C ABI ==
extern "C" {

int32_t pswarm_abi_version(void) { return PSWARM_ABI_VERSION; }

const char* pswarm_status_name(int32_t s) {
    switch (s) {
    case PSWARM_OK: return "ok";
    case PSWARM_ERR_GENERIC: return "Error";
    case PSWARM_ERR_INVALID_SPAN: return "InvalidSpanError";
    case PSWARM_ERR_INVALID_SIZE: return "InvalidSizeError";
    case PSWARM_ERR_SHAPE: return "ShapeError";
    case PSWARM_ERR_ALIGNMENT: return "AlignmentError";
    case PSWARM_ERR_DIVERGENCE: return "DivergenceError";
    case PSWARM_ERR_SINGULARITY: return "SingularityError";
    case PSWARM_ERR_COVERAGE: return "CoverageError";
    case PSWARM_ERR_NON_ELLIPTIC: return "NonEllipticError";
    case PSWARM_ERR_SOLVER: return "SolverError";
    case PSWARM_ERR_INVALID_PLAN: return "InvalidPlanError";
    case PSWARM_ERR_EMPTY_REDUCTION: return "EmptyReductionError";
    case PSWARM_ERR_TIMEOUT: return "TimeoutError";
    case PSWARM_ERR_INCOMPLETE: return "PropagationIncompleteError";
    case PSWARM_ERR_ORACLE: return "OracleError";
    case PSWARM_ERR_CUDA: return "CudaError";
    case PSWARM_ERR_OOM: return "OutOfMemory";
    case PSWARM_ERR_NO_DEVICE: return "NoDevice";
    default: return "unknown";
    }
}

pswarm_status pswarm_create(int32_t device, pswarm_ctx** out, pswarm_error* err) {
    return guarded(err, [&] {
        if (!out) raise(PSWARM_ERR_GENERIC, "pswarm_create: null output pointer");
        *out = nullptr;
        int count = 0;
        if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0)
            raise(PSWARM_ERR_NO_DEVICE, "pswarm_create: no CUDA device visible (the B200 path has no CPU fallback)");
        int dev = device;
        if (dev < 0) cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
        if (dev >= count) raise(PSWARM_ERR_NO_DEVICE, fmtf("pswarm_create: device %d not present", dev));
        cudaDeviceProp p{};
        cuda_check(cudaGetDeviceProperties(&p, dev), "cudaGetDeviceProperties");
        if (p.major != 10)
            raise(PSWARM_ERR_NO_DEVICE, fmtf("pswarm_create: device %d is sm_%d%d, this build targets sm_100a", dev,
                                             p.major, p.minor));
        auto ctx = std::make_unique<pswarm_ctx>();
        ctx->device = dev;
        ctx->sm_count = p.multiProcessorCount;
        bind(ctx.get());
        cuda_check(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking), "cudaStreamCreate");
        cuda_check(cudaEventCreate(&ctx->ev0), "cudaEventCreate");
        cuda_check(cudaEventCreate(&ctx->ev1), "cudaEventCreate");
        cuda_check(cudaEventCreate(&ctx->evk0), "cudaEventCreate");
        cuda_check(cudaEventCreate(&ctx->evk1), "cudaEventCreate");
        *out = ctx.release();
    });
}

void pswarm_destroy(pswarm_ctx* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    ctx->ops.clear();
    for (auto& b : ctx->buf) {
        if (b.p) cudaFree(b.p);
        b.p = nullptr;
        b.cap = 0;
    }
    if (ctx->copy_stream) {
        cudaStreamSynchronize(ctx->copy_stream);
        cudaStreamDestroy(ctx->copy_stream);
    }
    if (ctx->ev_seg) cudaEventDestroy(ctx->ev_seg);
    if (ctx->ev0) cudaEventDestroy(ctx->ev0);
    if (ctx->ev1) cudaEventDestroy(ctx->ev1);
    if (ctx->evk0) cudaEventDestroy(ctx->evk0);
    if (ctx->evk1) cudaEventDestroy(ctx->evk1);
    if (ctx->stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
}

pswarm_status pswarm_set_option(pswarm_ctx* ctx, const char* key, int64_t value) {
    return guarded(nullptr, [&] {
        const std::string k = key ? key : "";
        if (k == "ctas_per_sm") ctx->ctas_per_sm = static_cast<int>(std::max<int64_t>(1, value));
        else if (k == "max_ctas") ctx->max_ctas = static_cast<int>(std::max<int64_t>(0, value));
        else if (k == "profile_phases") ctx->profile_phases = value != 0;
        else if (k == "slot_kernel") ctx->slot_kernel = static_cast<int>(value);
        else if (k == "poison_outputs") ctx->poison_outputs = value != 0;
        else if (k == "fold") ctx->fold = value != 0;
        else if (k == "b0_mma") ctx->b0_mma = static_cast<int>(std::clamp<int64_t>(value, 0, 2));
        else if (k == "fast_decide") ctx->fast_decide = value != 0;
        else if (k == "force_ns") ctx->force_ns = static_cast<int>(value);
        else if (k == "small_ctas") ctx->small_ctas = value != 0;
        else if (k == "small_max_n") ctx->small_max_n = static_cast<int>(value);
        else if (k == "eph_nc") ctx->eph_nc = value != 0;
        else if (k == "stage") ctx->stage = value != 0;
        else if (k == "unified") ctx->unified = static_cast<int>(std::clamp<int64_t>(value, 0, 2));
        else raise(PSWARM_ERR_GENERIC, "pswarm_set_option: unknown key '" + k + "'");
    });
}

pswarm_status pswarm_get_phase_cycles(pswarm_ctx* ctx, uint64_t* out, int32_t n) {
    return guarded(nullptr, [&] {
        if (!ctx) raise(PSWARM_ERR_NO_DEVICE, "pswarm_get_phase_cycles: null context");
        for (int k = 0; k < n && k < PHASES; ++k) out[k] = ctx->phase_host[k];
    });
}

const char* pswarm_last_kernel(pswarm_ctx* ctx) { return ctx ? ctx->last_kernel : ""; }

pswarm_status pswarm_propagate(pswarm_ctx* ctx, int64_t n_states, const double* states, int64_t n_groups,
                               const int64_t* group_sizes, int64_t n_boundaries, const double* boundaries,
                               int64_t n_nodes, const pswarm_config* config, pswarm_outputs* out,
                               pswarm_error* err) {
    return guarded(err, [&] {
        propagate_impl(ctx, n_states, states, n_groups, group_sizes, n_boundaries, boundaries, n_nodes, config, out,
                       RunSpec{});
    });
}

pswarm_status pswarm_run_batch(pswarm_ctx* ctx, int64_t n_states, const double* states, int64_t n_boundaries,
                               const double* boundaries, int64_t n_nodes, const pswarm_config* config, int32_t mode,
                               int32_t workers, pswarm_outputs* out, pswarm_error* err) {
    return guarded(err, [&] {
        if (workers < 1) throw pswarm::InvalidPlanError("run_batch: need at least one worker");
        if (n_states < 1) throw pswarm::InvalidPlanError("propagate: empty batch");
        int64_t p_groups;  // grouping_for_mode (runner.hpp:47-55)
        if (mode == 0) p_groups = n_states;
        else if (mode == 1 || mode == 2) p_groups = 1;
        else if (mode == 3) p_groups = std::clamp<int64_t>(config->p_groups, 1, n_states);
        else throw pswarm::InvalidPlanError("grouping_for_mode: invalid mode");
        // the sizes of split_groups (block.hpp: larger groups first); the device path needs no
        // per-trajectory assignment tables (24 MB at 1M trajectories)
        const int64_t base = n_states / p_groups, rem = n_states % p_groups;
        std::vector<int64_t> sizes(static_cast<size_t>(p_groups), base);
        for (int64_t g = 0; g < rem; ++g) sizes[g] = base + 1;
        RunSpec spec;
        spec.independent = mode == 0;
        propagate_impl(ctx, n_states, states, p_groups, sizes.data(), n_boundaries, boundaries, n_nodes, config, out,
                       spec);
    });
}

pswarm_status pswarm_picard_update(pswarm_ctx* ctx, int64_t n_nodes, int64_t n_cols, const double* force,
                                   const double* initial_row, double* out, pswarm_error* err) {
    return guarded(err, [&] {
        if (!ctx) raise(PSWARM_ERR_NO_DEVICE, "pswarm_picard_update: null context");
        bind(ctx);
        const OpPack& op = operators(ctx, n_nodes);
        if (n_cols < 1) return;
        const size_t nc = static_cast<size_t>(n_nodes) * n_cols;
        double *dF, *dy0;
        upload(ctx, B_OP_IN, force, nc, &dF);
        upload(ctx, B_OP_IN2, initial_row, static_cast<size_t>(n_cols), &dy0);
        double* dO = ctx->buf[B_OP_OUT].get<double>(nc);
        cuda_check(launch_picard_update(static_cast<int>(n_nodes), op.nkp, static_cast<int>(n_cols), dF, dy0, dO,
                                        reinterpret_cast<const double2*>(op.buf.p), ctx->stream),
                   "k_picard_update");
        ++ctx->launches;
        cuda_check(cudaMemcpyAsync(out, dO, nc * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream), "D2H");
        cuda_check(cudaStreamSynchronize(ctx->stream), "picard_update");
    });
}

pswarm_status pswarm_picard_update_ops(pswarm_ctx* ctx, int64_t n_nodes, int64_t n_cols, const double* update_op,
                                       const double* anchor_op, const double* force, const double* initial_row,
                                       double* out, pswarm_error* err) {
    return guarded(err, [&] {
        if (!ctx) raise(PSWARM_ERR_NO_DEVICE, "pswarm_picard_update_ops: null context");
        if (!update_op || !anchor_op) raise(PSWARM_ERR_SHAPE, "picard_update: operators must be given");
        if (n_nodes < 3 || n_nodes > 264)
            raise(PSWARM_ERR_INVALID_SIZE, fmtf("device operators support 3..264 nodes, got %lld", (long long)n_nodes));
        bind(ctx);
        if (n_cols < 1) return;
        const GemmPlan gp = make_gemm_plan(static_cast<int>(n_nodes));
        const std::vector<double> host = pack_dense_operator(n_nodes, gp, update_op, anchor_op);
        double* dA;
        upload(ctx, B_OP_AUX, host.data(), host.size(), &dA);
        const size_t nc = static_cast<size_t>(n_nodes) * n_cols;
        double *dF, *dy0;
        upload(ctx, B_OP_IN, force, nc, &dF);
        upload(ctx, B_OP_IN2, initial_row, static_cast<size_t>(n_cols), &dy0);
        double* dO = ctx->buf[B_OP_OUT].get<double>(nc);
        cuda_check(launch_picard_update(static_cast<int>(n_nodes), static_cast<int>((n_nodes + 7) / 8),
                                        static_cast<int>(n_cols), dF, dy0, dO, reinterpret_cast<const double2*>(dA),
                                        ctx->stream),
                   "k_picard_update");
        ++ctx->launches;
        cuda_check(cudaMemcpyAsync(out, dO, nc * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream), "D2H");
        cuda_check(cudaStreamSynchronize(ctx->stream), "picard_update");
    });
}

pswarm_status pswarm_eval_force_block(pswarm_ctx* ctx, int64_t n_nodes, int64_t group_size, const double* y,
                                      double omega2, int32_t force_kind, double central_mu, int32_t n_bodies,
                                      const double* body_positions, const double* body_mus,
                                      const char* const* body_names, double proximity_floor_km, double* force,
                                      pswarm_error* err) {
    return guarded(err, [&] {
        if (!ctx) raise(PSWARM_ERR_NO_DEVICE, "pswarm_eval_force_block: null context");
        bind(ctx);
        const int64_t N = n_nodes, m = group_size;
        if (force_kind < 0 || force_kind > 1)
            raise(PSWARM_ERR_INVALID_PLAN, "eval_force_block: the operator entry point takes force kinds 0 (two_body) "
                                           "and 1 (n_body); n_body_1pn needs body velocities (use propagate)");
        const int B = force_kind == 1 ? n_bodies : 0;
        if (B > 63) raise(PSWARM_ERR_INVALID_SIZE, "eval_force_block: at most 63 perturbing bodies are supported");
        const size_t nc = static_cast<size_t>(N) * 6 * m;
        // body table [B][N][3] -> node-major [N][B][3] + indirect term
        std::vector<double> pos(static_cast<size_t>(N) * B * 3), ind(static_cast<size_t>(N) * 3, 0.0);
        for (int64_t j = 0; j < N; ++j)
            for (int b = 0; b < B; ++b) {
                const double* p = body_positions + (static_cast<size_t>(b) * N + j) * 3;
                std::copy(p, p + 3, pos.data() + (j * B + b) * 3);
                const double bn = std::sqrt(p[0] * p[0] + p[1] * p[1] + p[2] * p[2]);
                for (int c = 0; c < 3; ++c) ind[j * 3 + c] += body_mus[b] * (p[c] / (bn * bn * bn));
            }
        double *dy, *dpos, *dmu, *dind;
        upload(ctx, B_OP_IN, y, nc, &dy);
        upload(ctx, B_BODY_POS, pos.data(), pos.size(), &dpos);
        upload(ctx, B_BODY_MU, body_mus, static_cast<size_t>(B), &dmu);
        upload(ctx, B_INDIRECT, ind.data(), ind.size(), &dind);
        double* dF = ctx->buf[B_OP_OUT].get<double>(nc);
        unsigned long long* dkey = reinterpret_cast<unsigned long long*>(ctx->buf[B_OP_KEY].get<double>(1));
        cuda_check(cudaMemsetAsync(dkey, 0xff, sizeof(unsigned long long), ctx->stream), "memset");
        const ForceData fd = make_force_data(dpos, dmu, dind, central_mu, proximity_floor_km, B);
        cuda_check(launch_force_block(static_cast<int>(N), static_cast<int>(m), dy, omega2, fd, force_kind == 1, dF, dkey,
                                      ctx->stream),
                   "k_force_block");
        ++ctx->launches;
        unsigned long long key = 0;
        cuda_check(cudaMemcpyAsync(force, dF, nc * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream), "D2H");
        cuda_check(cudaMemcpyAsync(&key, dkey, sizeof key, cudaMemcpyDeviceToHost, ctx->stream), "D2H");
        cuda_check(cudaStreamSynchronize(ctx->stream), "eval_force_block");
        if (key != ~0ull) {
            // first failing sample in s = j*m + t order (force_model.hpp:130-140); the
            // message quotes the caller's own input, so it is formatted from it here.
            const int64_t s = static_cast<int64_t>(key / 64), chk = static_cast<int64_t>(key % 64);
            const int64_t j = s / m, t = s % m;
            const double* row = y + static_cast<size_t>(j) * 6 * m;
            const double r[3] = {row[t], row[m + t], row[2 * m + t]};
            std::string what, body;
            if (chk == 0) {
                what = "central-body acceleration at zero radius";
            } else {
                const int b = static_cast<int>(chk - 1);
                const double* p = body_positions + (static_cast<size_t>(b) * N + j) * 3;
                const double d[3] = {p[0] - r[0], p[1] - r[1], p[2] - r[2]};
                const double dn = std::sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
                body = body_names && body_names[b] ? body_names[b] : "";
                what = "close approach to body '" + body + "': distance " + std::to_string(dn) + " km below floor " +
                       std::to_string(proximity_floor_km) + " km";
            }
            CapiFault f;
            init_err(&f.e, PSWARM_ERR_SINGULARITY,
                     "node " + std::to_string(j) + ", trajectory " + std::to_string(t) + ": " + what);
            std::snprintf(f.e.body_name, sizeof f.e.body_name, "%s", body.c_str());
            f.e.node = j;
            f.e.trajectory = t;
            f.e.body = static_cast<int32_t>(chk - 1);
            throw f;
        }
    });
}

pswarm_status pswarm_block_iteration_error(pswarm_ctx* ctx, int64_t n_nodes, int64_t group_size, const double* cur,
                                           const double* prev, int32_t error_mode, double* per_state,
                                           double* group_max, pswarm_error* err) {
    return guarded(err, [&] {
        if (!ctx) raise(PSWARM_ERR_NO_DEVICE, "pswarm_block_iteration_error: null context");
        if (group_size < 1) throw pswarm::EmptyReductionError("reduce_max: empty input");
        bind(ctx);
        const size_t nc = static_cast<size_t>(n_nodes) * 6 * group_size;
        double *dc, *dp;
        upload(ctx, B_OP_IN, cur, nc, &dc);
        upload(ctx, B_OP_IN2, prev, nc, &dp);
        unsigned long long* dbits = reinterpret_cast<unsigned long long*>(ctx->buf[B_OP_OUT].get<double>(group_size));
        cuda_check(cudaMemsetAsync(dbits, 0, sizeof(double) * group_size, ctx->stream), "memset");
        cuda_check(launch_block_error(static_cast<int>(n_nodes), static_cast<int>(group_size), dc, dp, error_mode, dbits,
                                      ctx->stream),
                   "k_block_error");
        ++ctx->launches;
        std::vector<double> h(static_cast<size_t>(group_size));
        cuda_check(cudaMemcpyAsync(h.data(), dbits, sizeof(double) * group_size, cudaMemcpyDeviceToHost, ctx->stream),
                   "D2H");
        cuda_check(cudaStreamSynchronize(ctx->stream), "block_error");
        if (per_state) std::memcpy(per_state, h.data(), sizeof(double) * group_size);
        if (group_max) *group_max = *std::max_element(h.begin(), h.end());
    });
}

pswarm_status pswarm_oracle_check(pswarm_ctx* ctx, int64_t n_states, const double* states, int64_t n_times,
                                  const double* times, const pswarm_config* config, double rel_tol, double abs_tol,
                                  int64_t max_steps, const double* candidate, double* samples_out,
                                  double* node_error, double* max_error, pswarm_error* err) {
    return guarded(err, [&] {
        if (!(rel_tol > 0.0) || !(abs_tol > 0.0))
            throw pswarm::OracleError("rk_propagate: tolerances must be positive");  // oracle.hpp:66-68
        const int64_t M = n_states, R = n_times;
        if (M < 1) return;
        for (int64_t i = 0; i < M; ++i)
            if (R < 1 || times[0] != states[7 * i])
                throw pswarm::OracleError("oracle_sample_trajectory: sample times must begin at the state epoch");
        if (!ctx) raise(PSWARM_ERR_NO_DEVICE, "pswarm_oracle_check: null context");
        if (config->force_kind < 0 || config->force_kind > 2)
            raise(PSWARM_ERR_INVALID_PLAN, "oracle_check: unknown force kind " + std::to_string(config->force_kind));
        const int nb = config->force_kind >= 1 ? config->n_bodies : 0;
        if (nb > 16) raise(PSWARM_ERR_INVALID_SIZE, "oracle_check: at most 16 perturbing bodies are supported");
        bind(ctx);
        const BodyUpload bu = flatten_bodies(*config, nb);
        if (bu.first_invalid >= 0) throw pswarm::NonEllipticError(bu.invalid_msg);
        cudaStream_t st = ctx->stream;
        DevBuf tmp[8];  // body table of this call
        auto up = [&](int k, const void* h, size_t bytes) -> void* {
            void* d = tmp[k].get<char>(bytes);
            if (bytes) cuda_check(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, st), "H2D");
            return d;
        };
        RkArgs a{};
        a.M = static_cast<int>(M);
        a.R = static_cast<int>(R);
        a.rel = config->force_kind == 2 ? 1 : 0;
        a.max_steps = max_steps;
        a.rel_tol = rel_tol;
        a.abs_tol = abs_tol;
        a.central_mu = config->central_mu;
        a.floor_km = config->proximity_floor_km;
        a.c_light = config->c_light > 0.0 ? config->c_light : 299792.458;
        a.bt = BodyTable{nb,
                         static_cast<int*>(up(0, bu.kind.data(), sizeof(int) * bu.kind.size())),
                         static_cast<double*>(up(1, bu.elements.data(), sizeof(double) * bu.elements.size())),
                         static_cast<double*>(up(2, bu.mu.data(), sizeof(double) * bu.mu.size())),
                         static_cast<int*>(up(3, bu.seg_off.data(), sizeof(int) * bu.seg_off.size())),
                         static_cast<double*>(up(4, bu.bounds.data(), sizeof(double) * bu.bounds.size())),
                         static_cast<long long*>(up(5, bu.coeff_off.data(), sizeof(long long) * bu.coeff_off.size())),
                         static_cast<int*>(up(6, bu.ncoef.data(), sizeof(int) * bu.ncoef.size())),
                         static_cast<double*>(up(7, bu.coeffs.data(), sizeof(double) * bu.coeffs.size()))};
        double* d_states;
        double* d_times;
        upload(ctx, B_OP_IN, states, static_cast<size_t>(M) * 7, &d_states);
        upload(ctx, B_OP_IN2, times, static_cast<size_t>(R), &d_times);
        a.states = d_states;
        a.times = d_times;
        const size_t ns = static_cast<size_t>(M) * R * 6;
        double* d_cand = nullptr;
        if (candidate) upload(ctx, B_SAMPLES, candidate, ns, &d_cand);
        a.candidate = d_cand;
        a.samples_out = samples_out ? ctx->buf[B_OP_OUT].get<double>(ns) : nullptr;
        a.node_err = node_error && candidate ? ctx->buf[B_OP_AUX].get<double>(static_cast<size_t>(M) * R) : nullptr;
        a.max_err = ctx->buf[B_REP_ERR].get<double>(static_cast<size_t>(M));
        a.fault_t = ctx->buf[B_DEAD].get<double>(static_cast<size_t>(M));
        a.fault_key = reinterpret_cast<unsigned long long*>(ctx->buf[B_OP_KEY].get<double>(1));
        cuda_check(cudaMemsetAsync(a.fault_key, 0xff, sizeof(unsigned long long), st), "memset");
        cuda_check(launch_rk_check(a, st), "k_rk_check");
        ++ctx->launches;
        unsigned long long key = 0;
        cuda_check(cudaMemcpyAsync(&key, a.fault_key, sizeof key, cudaMemcpyDeviceToHost, st), "D2H");
        if (a.samples_out)
            cuda_check(cudaMemcpyAsync(samples_out, a.samples_out, ns * sizeof(double), cudaMemcpyDeviceToHost, st), "D2H");
        if (a.node_err)
            cuda_check(cudaMemcpyAsync(node_error, a.node_err, sizeof(double) * M * R, cudaMemcpyDeviceToHost, st),
                       "D2H");
        if (max_error)
            cuda_check(cudaMemcpyAsync(max_error, a.max_err, sizeof(double) * M, cudaMemcpyDeviceToHost, st), "D2H");
        cuda_check(cudaStreamSynchronize(st), "oracle_check");
        if (key != ~0ull) {  // the lowest failing trajectory, in the reference's wording
            const int64_t tr = static_cast<int64_t>(key >> 24);
            const int code = static_cast<int>((key >> 16) & 0xff);
            double tf = 0.0;
            cuda_check(cudaMemcpy(&tf, a.fault_t + tr, sizeof tf, cudaMemcpyDeviceToHost), "D2H");
            if (code == 200) throw pswarm::OracleError("rk_propagate: step size underflow at t = " + std::to_string(tf));
            if (code == 201)
                throw pswarm::OracleError("rk_propagate: exceeded " + std::to_string(max_steps) + " steps");
            if (code == 1) throw pswarm::SingularityError("central-body acceleration at zero radius");
            if (code >= 100) {
                const int b = code - 100;
                if (bu.kind[b] == 1)
                    throw pswarm::CoverageError("ephemeris for body '" + bu.names[b] + "' does not cover epoch " +
                                                    std::to_string(tf),
                                                tf);
                throw pswarm::SolverError("solve_kepler: Newton iteration did not converge for body '" + bu.names[b] +
                                          "'");
            }
            const int b = code - 2;
            throw pswarm::SingularityError("close approach to body '" + bu.names[b] + "' (trajectory " +
                                               std::to_string(tr) + ")",
                                           bu.names[b]);
        }
    });
}

pswarm_status pswarm_warm_start(pswarm_ctx* ctx, int64_t n_states, const double* states, int64_t n_nodes,
                                const double* times, double central_mu, double* guesses, uint8_t* cold_fallback,
                                pswarm_error* err) {
    return guarded(err, [&] {
        if (!ctx) raise(PSWARM_ERR_NO_DEVICE, "pswarm_warm_start: null context");
        bind(ctx);
        if (n_states < 1) return;
        double *ds, *dt;
        upload(ctx, B_OP_IN, states, static_cast<size_t>(n_states) * 7, &ds);
        upload(ctx, B_OP_IN2, times, static_cast<size_t>(n_nodes), &dt);
        const size_t ng = static_cast<size_t>(n_states) * n_nodes * 6;
        double* dg = ctx->buf[B_OP_OUT].get<double>(ng);
        uint8_t* dfb = ctx->buf[B_FALLBACK].get<uint8_t>(static_cast<size_t>(n_states));
        double* aux = ctx->buf[B_OP_AUX].get<double>(4);
        unsigned long long* dkey = reinterpret_cast<unsigned long long*>(ctx->buf[B_OP_KEY].get<double>(1));
        cuda_check(cudaMemsetAsync(dkey, 0xff, sizeof(unsigned long long), ctx->stream), "memset");
        cuda_check(launch_warm_start(static_cast<int>(n_states), ds, static_cast<int>(n_nodes), dt, central_mu, dg, dfb,
                                     dkey, aux, ctx->stream),
                   "k_warm_start");
        ctx->launches += 2;
        unsigned long long key = 0;
        double vals[2] = {0.0, 0.0};
        cuda_check(cudaMemcpyAsync(guesses, dg, ng * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream), "D2H");
        if (cold_fallback)
            cuda_check(cudaMemcpyAsync(cold_fallback, dfb, static_cast<size_t>(n_states), cudaMemcpyDeviceToHost,
                                       ctx->stream),
                       "D2H");
        cuda_check(cudaMemcpyAsync(&key, dkey, sizeof key, cudaMemcpyDeviceToHost, ctx->stream), "D2H");
        cuda_check(cudaMemcpyAsync(vals, aux, sizeof vals, cudaMemcpyDeviceToHost, ctx->stream), "D2H");
        cuda_check(cudaStreamSynchronize(ctx->stream), "warm_start");
        if (key != ~0ull) {
            const int kind = static_cast<int>(key % 4);
            const int64_t idx = static_cast<int64_t>(key / 4);
            if (kind == CONIC_ZERO_RADIUS) throw pswarm::SingularityError("kepler_propagate: zero-radius state");
            CapiFault f;
            init_err(&f.e, PSWARM_ERR_SOLVER,
                     "solve_kepler: Newton iteration did not converge for M = " + std::to_string(vals[0]) +
                         ", e = " + std::to_string(vals[1]));
            f.e.trajectory = idx / n_nodes;
            f.e.node = idx % n_nodes;
            throw f;
        }
    });
}

pswarm_status pswarm_elements_to_state(const double* el, double mu, double t, double* state_out, pswarm_error* err) {
    return guarded(err, [&] {
        const auto s = pswarm::elements_to_state(pswarm::OrbitalElements{el[0], el[1], el[2], el[3], el[4], el[5], el[6]},
                                                 mu, t);
        state_out[0] = s.epoch;
        for (int c = 0; c < 3; ++c) {
            state_out[1 + c] = s.r[c];
            state_out[4 + c] = s.v[c];
        }
    });
}

static pswarm::StateVector state_from7(const double* s) {
    pswarm::StateVector x;
    x.epoch = s[0];
    x.r = pswarm::Vec3(s[1], s[2], s[3]);
    x.v = pswarm::Vec3(s[4], s[5], s[6]);
    return x;
}

pswarm_status pswarm_osculating_period(const double* state, double mu, double* period, pswarm_error* err) {
    return guarded(err, [&] { *period = pswarm::osculating_period(state_from7(state), mu); });
}

pswarm_status pswarm_plan_segments(const double* rep, double t_start, double t_end, double mu, int32_t policy,
                                   int64_t n_nodes, double max_periods, int64_t capacity, double* boundaries,
                                   int64_t* n_boundaries, pswarm_error* err) {
    return guarded(err, [&] {
        const auto p = pswarm::plan_segments(state_from7(rep), t_start, t_end, mu,
                                             policy == 1 ? pswarm::SegmentPolicy::per_orbit : pswarm::SegmentPolicy::single,
                                             n_nodes, max_periods);
        if (static_cast<int64_t>(p.boundaries.size()) > capacity)
            raise(PSWARM_ERR_GENERIC, "pswarm_plan_segments: boundary buffer too small");
        std::memcpy(boundaries, p.boundaries.data(), sizeof(double) * p.boundaries.size());
        *n_boundaries = static_cast<int64_t>(p.boundaries.size());
    });
}

pswarm_status pswarm_build_grid(int64_t n_nodes, double t_start, double t_end, double* times, double* omega2,
                                pswarm_error* err) {
    return guarded(err, [&] {
        const auto g = pswarm::build_grid(n_nodes, t_start, t_end);
        std::memcpy(times, g.times.data(), sizeof(double) * n_nodes);
        if (omega2) *omega2 = g.omega2;
    });
}

void pswarm_make_clone_batch(const double* base, int64_t count, double spread, uint64_t seed, double* out) {
    const auto b = pswarm::make_clone_batch(state_from7(base), count, spread, seed);
    for (int64_t i = 0; i < count; ++i) {
        out[7 * i] = b[i].epoch;
        for (int c = 0; c < 3; ++c) {
            out[7 * i + 1 + c] = b[i].r[c];
            out[7 * i + 4 + c] = b[i].v[c];
        }
    }
}

void* pswarm_pinned_alloc(size_t bytes) {
    void* p = nullptr;
    if (cudaHostAlloc(&p, std::max<size_t>(bytes, 64), cudaHostAllocDefault) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    return p;
}

void pswarm_pinned_free(void* p) {
    if (p) cudaFreeHost(p);
}

}  // extern "C"

// ============================================================ multi-device ==
// run_batch over several devices of one process (runner.hpp:111-135 + SURVEY §8e):
// contiguous group-aligned shards (block.hpp:83-106), one host thread and one context per
// device (the reference's worker pool, thread_pool.hpp:46-87, over GPUs), no collective in
// the iteration or segment loop, and one gather of the terminal states to devices[0]:
// NCCL send/recv over NVLink (one ncclGroup) when the devices are distinct, a peer /
// device-to-device copy when a device is listed twice (flow testing on one GPU).
namespace {

struct NcclApi {
    void* h = nullptr;
    ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    ncclResult_t (*GetVersion)(int*) = nullptr;
};

const NcclApi* nccl_api() {
    static NcclApi api = [] {
        NcclApi a;
        // an NCCL already in the process (e.g. the one PyTorch links) first: loading a second
        // libnccl.so.2 would shadow it for libraries that resolve it later by soname
        a.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!a.h)
            if (const char* p = std::getenv("PSWARM_NCCL_LIB")) a.h = dlopen(p, RTLD_NOW | RTLD_LOCAL);
        if (!a.h) a.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
        if (!a.h) return a;
        auto sym = [&](auto& fp, const char* n) { fp = reinterpret_cast<std::remove_reference_t<decltype(fp)>>(dlsym(a.h, n)); };
        sym(a.CommInitAll, "ncclCommInitAll");
        sym(a.CommDestroy, "ncclCommDestroy");
        sym(a.GroupStart, "ncclGroupStart");
        sym(a.GroupEnd, "ncclGroupEnd");
        sym(a.Send, "ncclSend");
        sym(a.Recv, "ncclRecv");
        sym(a.GetErrorString, "ncclGetErrorString");
        sym(a.GetVersion, "ncclGetVersion");
        if (!a.CommInitAll || !a.GroupStart || !a.GroupEnd || !a.Send || !a.Recv || !a.CommDestroy) a.h = nullptr;
        return a;
    }();
    return api.h ? &api : nullptr;
}

void nccl_check(const NcclApi* n, ncclResult_t r, const char* what) {
    if (r == ncclSuccess) return;
    raise(PSWARM_ERR_GENERIC, std::string("NCCL failure in ") + what + ": " +
                                  (n && n->GetErrorString ? n->GetErrorString(r) : "?"));
}

}  // namespace

struct pswarm_multi {
    std::vector<pswarm_ctx*> ctx;
    std::vector<int> devices;
    std::vector<ncclComm_t> comms;  // one per device when the devices are distinct
    const char* backend = "peer-copy";
    DevBuf root_term;   // gathered [M][6] on devices[0]
    DevBuf root_term7;  // the same packed to the caller's [M][7] (one D2H)
    PinnedBuf pin_term;
    int nccl_version = 0;
};

extern "C" {

pswarm_status pswarm_create_multi(int32_t n_devices, const int32_t* devices, pswarm_multi** out, pswarm_error* err) {
    return guarded(err, [&] {
        if (!out) raise(PSWARM_ERR_GENERIC, "pswarm_create_multi: null output pointer");
        *out = nullptr;
        if (n_devices < 1 || !devices) raise(PSWARM_ERR_INVALID_PLAN, "pswarm_create_multi: need at least one device");
        auto m = std::make_unique<pswarm_multi>();
        for (int32_t r = 0; r < n_devices; ++r) {
            pswarm_ctx* c = nullptr;
            pswarm_error e{};
            if (pswarm_create(devices[r], &c, &e) != PSWARM_OK) {
                for (pswarm_ctx* x : m->ctx) pswarm_destroy(x);
                CapiFault f;
                f.e = e;
                throw f;
            }
            m->ctx.push_back(c);
            m->devices.push_back(c->device);
        }
        std::vector<int> sorted = m->devices;
        std::sort(sorted.begin(), sorted.end());
        const bool distinct = std::adjacent_find(sorted.begin(), sorted.end()) == sorted.end();
        const NcclApi* n = distinct && n_devices > 1 ? nccl_api() : nullptr;  // loaded only when used
        if (n) {
            m->comms.resize(static_cast<size_t>(n_devices));
            const ncclResult_t r = n->CommInitAll(m->comms.data(), n_devices, m->devices.data());
            if (r != ncclSuccess) {
                m->comms.clear();
                for (pswarm_ctx* x : m->ctx) pswarm_destroy(x);
                nccl_check(n, r, "ncclCommInitAll");
            }
            if (n->GetVersion) n->GetVersion(&m->nccl_version);
            m->backend = "nccl";
        } else if (distinct && n_devices > 1) {
            m->backend = "peer-copy (libnccl not found)";
        }
        *out = m.release();
    });
}

void pswarm_destroy_multi(pswarm_multi* m) {
    if (!m) return;
    const NcclApi* n = m->comms.empty() ? nullptr : nccl_api();
    for (ncclComm_t c : m->comms)
        if (n && c) n->CommDestroy(c);
    if (!m->ctx.empty()) {
        cudaSetDevice(m->ctx[0]->device);
        if (m->root_term.p) cudaFree(m->root_term.p);
        m->root_term.p = nullptr;
        if (m->root_term7.p) cudaFree(m->root_term7.p);
        m->root_term7.p = nullptr;
    }
    for (pswarm_ctx* c : m->ctx) pswarm_destroy(c);
    delete m;
}

const char* pswarm_multi_backend(pswarm_multi* m) { return m ? m->backend : ""; }

int32_t pswarm_multi_devices(pswarm_multi* m) { return m ? static_cast<int32_t>(m->ctx.size()) : 0; }

pswarm_status pswarm_run_batch_multi(pswarm_multi* mc, int64_t n_states, const double* states, int64_t n_boundaries,
                                     const double* boundaries, int64_t n_nodes, const pswarm_config* config,
                                     int32_t mode, int32_t workers, pswarm_outputs* out, pswarm_error* err) {
    return guarded(err, [&] {
        const auto wall0 = std::chrono::steady_clock::now();
        if (!mc || mc->ctx.empty()) raise(PSWARM_ERR_NO_DEVICE, "run_batch_multi: no device contexts");
        if (workers < 1) throw pswarm::InvalidPlanError("run_batch: need at least one worker");
        if (n_states < 1) throw pswarm::InvalidPlanError("propagate: empty batch");
        if (!config) raise(PSWARM_ERR_GENERIC, "propagate: null config");
        int64_t P;  // grouping_for_mode (runner.hpp:47-55) with split_groups sizes (larger first)
        if (mode == 0) P = n_states;
        else if (mode == 1 || mode == 2) P = 1;
        else if (mode == 3) P = std::clamp<int64_t>(config->p_groups, 1, n_states);
        else throw pswarm::InvalidPlanError("grouping_for_mode: invalid mode");
        const int64_t base = n_states / P, rem = n_states % P;
        std::vector<int64_t> sizes(static_cast<size_t>(P), base), off(static_cast<size_t>(P) + 1, 0);
        for (int64_t g = 0; g < rem; ++g) sizes[g] = base + 1;
        for (int64_t g = 0; g < P; ++g) off[g + 1] = off[g] + sizes[g];
        // group-aligned shards balanced by trajectory count (paper_2301_03989_b200/distributed.py)
        const int D = static_cast<int>(mc->ctx.size());
        std::vector<int64_t> g_lo(D), g_hi(D);
        for (int r = 0, g = 0; r < D; ++r) {
            const int64_t hi_traj = (static_cast<int64_t>(r) + 1) * n_states / D;
            g_lo[r] = g;
            while (g < P && off[g] < hi_traj) ++g;
            if (r == D - 1) g = static_cast<int>(P);
            g_hi[r] = g;
        }
        const int64_t S = n_boundaries - 1, N = n_nodes, R = S >= 1 ? 1 + S * (N - 1) : 0;
        const int max_it = std::max(config->max_iterations, 0);
        struct Shard {
            int64_t lo = 0, M = 0, P = 0;
            std::vector<int32_t> iter;
            std::vector<double> ferr, hist;
            std::vector<uint8_t> conv, fb;
            std::vector<double> times;
            pswarm_outputs o{};
            pswarm_error e{};
            pswarm_status st = PSWARM_OK;
            const double* term = nullptr;
            int64_t fail_index = -1;
        };
        std::vector<Shard> sh(static_cast<size_t>(D));
        for (int r = 0; r < D; ++r) {
            Shard& x = sh[r];
            x.lo = off[g_lo[r]];
            x.M = off[g_hi[r]] - x.lo;
            x.P = g_hi[r] - g_lo[r];
            if (x.M == 0 || S < 1) continue;
            x.iter.resize(static_cast<size_t>(S * x.P));
            x.ferr.resize(static_cast<size_t>(S * x.P));
            x.conv.resize(static_cast<size_t>(S * x.P));
            x.o.iterations = x.iter.data();
            x.o.final_error = x.ferr.data();
            x.o.converged = x.conv.data();
            if (out && out->error_history && max_it > 0) {
                x.hist.resize(static_cast<size_t>(S * x.P * max_it));
                x.o.error_history = x.hist.data();
            }
            if (out && out->cold_fallback) {
                x.fb.resize(static_cast<size_t>(S * x.M));
                x.o.cold_fallback = x.fb.data();
            }
            if (out && out->samples) x.o.samples = out->samples + x.lo * R * 6;  // contiguous per trajectory
            if (out && out->times && r == 0) {
                x.times.resize(static_cast<size_t>(R));
                x.o.times = x.times.data();
            }
        }
        auto run_shard = [&](int r) {
            Shard& x = sh[r];
            RunSpec spec;
            spec.independent = mode == 0;
            spec.term_dev = &x.term;
            spec.fail_index = &x.fail_index;
            x.st = guarded(&x.e, [&] {
                propagate_impl(mc->ctx[r], x.M, states + 7 * x.lo, x.P, sizes.data() + g_lo[r], n_boundaries,
                               boundaries, n_nodes, config, &x.o, spec);
            });
        };
        std::vector<std::thread> threads;
        for (int r = 1; r < D; ++r)
            if (sh[r].M > 0) threads.emplace_back(run_shard, r);
        if (sh[0].M > 0) run_shard(0);  // the caller takes shard 0 (thread_pool.hpp:124-142)
        for (auto& t : threads) t.join();

        // ---- the error the serial reference would raise: independent mode = lowest failing
        // trajectory (runner.hpp:63-80); grouped/augmented = first failing segment, exceptions
        // before non-convergence, then the lowest group (propagator.hpp:292-312)
        int pick = -1;
        auto key = [&](int r) {
            const pswarm_error& e = sh[r].e;
            if (mode == 0)  // ephemeris / validation errors (no failing trajectory) come first
                return std::make_tuple(int64_t{0}, int64_t{0}, sh[r].fail_index >= 0 ? sh[r].lo + sh[r].fail_index : -1);
            const int64_t seg = e.segment >= 0 ? e.segment : -1;
            return std::make_tuple(seg, int64_t{e.status == PSWARM_ERR_INCOMPLETE ? 1 : 0},
                                   g_lo[r] + std::max<int64_t>(e.group, 0));
        };
        for (int r = 0; r < D; ++r)
            if (sh[r].M > 0 && sh[r].st != PSWARM_OK && (pick < 0 || key(r) < key(pick))) pick = r;

        if (out) {
            int64_t rep = S, done = S;
            for (int r = 0; r < D; ++r) {
                if (sh[r].M == 0) continue;
                rep = std::min(rep, sh[r].o.segments_reported);
                done = std::min(done, sh[r].o.segments_completed);
            }
            if (pick >= 0 && sh[pick].st == PSWARM_ERR_INCOMPLETE) rep = std::max(rep, sh[pick].o.segments_reported);
            out->segments_reported = rep;
            out->segments_completed = done;
            double dms = 0.0, kms = 0.0;
            int64_t iters = 0, launches = 0;
            for (int r = 0; r < D; ++r) {
                const Shard& x = sh[r];
                launches += mc->ctx[r]->launches;
                if (x.M == 0) continue;
                dms = std::max(dms, x.o.device_ms);
                kms = std::max(kms, x.o.kernel_ms);
                iters += x.o.trajectory_iterations;
                for (int64_t sg = 0; sg < std::min(rep, x.o.segments_reported); ++sg) {
                    const int64_t dst = sg * P + g_lo[r], src = sg * x.P;
                    if (out->iterations) std::memcpy(out->iterations + dst, x.iter.data() + src, sizeof(int32_t) * x.P);
                    if (out->final_error) std::memcpy(out->final_error + dst, x.ferr.data() + src, sizeof(double) * x.P);
                    if (out->converged) std::memcpy(out->converged + dst, x.conv.data() + src, static_cast<size_t>(x.P));
                    if (out->error_history && max_it > 0)
                        std::memcpy(out->error_history + dst * max_it, x.hist.data() + src * max_it,
                                    sizeof(double) * x.P * max_it);
                    if (out->cold_fallback)
                        std::memcpy(out->cold_fallback + sg * n_states + x.lo, x.fb.data() + sg * x.M,
                                    static_cast<size_t>(x.M));
                }
            }
            if (out->times && !sh[0].times.empty()) std::memcpy(out->times, sh[0].times.data(), sizeof(double) * R);
            out->device_ms = dms;
            out->kernel_ms = kms;
            out->trajectory_iterations = iters;
            out->gpu_launches = launches;
        }
        if (pick >= 0) {
            pswarm_error e = sh[pick].e;
            // batch index (a solve singularity names the trajectory within its singleton group)
            if (mode == 0 && e.trajectory >= 0 && !(e.status == PSWARM_ERR_SINGULARITY && e.node >= 0))
                e.trajectory += sh[pick].lo;
            if (mode != 0 && e.group >= 0) e.group += g_lo[pick];
            CapiFault f;
            f.e = e;
            throw f;
        }

        // ---- the single collective: terminal states of every shard -> devices[0]
        if (out && out->terminal_states) {
            pswarm_ctx* root = mc->ctx[0];
            bind(root);
            double* dst = mc->root_term.get<double>(static_cast<size_t>(n_states) * 6);
            if (!mc->comms.empty()) {
                const NcclApi* n = nccl_api();
                nccl_check(n, n->GroupStart(), "ncclGroupStart");
                for (int r = 1; r < D; ++r) {
                    if (sh[r].M == 0) continue;
                    const size_t cnt = static_cast<size_t>(sh[r].M) * 6;
                    nccl_check(n, n->Recv(dst + sh[r].lo * 6, cnt, ncclFloat64, r, mc->comms[0], root->stream), "ncclRecv");
                    nccl_check(n, n->Send(sh[r].term, cnt, ncclFloat64, 0, mc->comms[r], mc->ctx[r]->stream), "ncclSend");
                }
                nccl_check(n, n->GroupEnd(), "ncclGroupEnd");
            } else {
                for (int r = 1; r < D; ++r)
                    if (sh[r].M > 0)
                        cuda_check(cudaMemcpyPeerAsync(dst + sh[r].lo * 6, root->device, sh[r].term, mc->ctx[r]->device,
                                                       sizeof(double) * sh[r].M * 6, root->stream),
                                   "gather peer copy");
            }
            if (sh[0].M > 0)
                cuda_check(cudaMemcpyAsync(dst, sh[0].term, sizeof(double) * sh[0].M * 6, cudaMemcpyDeviceToDevice,
                                           root->stream),
                           "gather root shard");
            // packed to [M][7] on the device: one DMA straight into a page-locked caller buffer
            double* d7 = mc->root_term7.get<double>(static_cast<size_t>(n_states) * 7);
            cuda_check(launch_pack_states7(dst, boundaries[S], d7, n_states, root->stream), "k_pack_states7");
            ++root->launches;
            cudaPointerAttributes pa{};
            const bool direct = cudaPointerGetAttributes(&pa, out->terminal_states) == cudaSuccess &&
                                pa.type == cudaMemoryTypeHost;
            cudaGetLastError();
            double* h = direct ? out->terminal_states : mc->pin_term.get<double>(sizeof(double) * n_states * 7);
            cuda_check(cudaMemcpyAsync(h, d7, sizeof(double) * n_states * 7, cudaMemcpyDeviceToHost, root->stream),
                       "D2H gathered terminal states");
            for (int r = 1; r < D; ++r) {
                bind(mc->ctx[r]);
                cuda_check(cudaStreamSynchronize(mc->ctx[r]->stream), "gather (send side)");
            }
            bind(root);
            cuda_check(cudaStreamSynchronize(root->stream), "gather");
            if (!direct) std::memcpy(out->terminal_states, h, sizeof(double) * n_states * 7);
        }
        if (out) out->wall_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - wall0).count();
    });
}

}  // extern "C"
