/*
 * pswarm_gpu.h — the C-ABI drop-in boundary of the B200-native augmented
 * Picard–Chebyshev (PC) propagator.
 *
 * Plain C types only (no torch, no Eigen, no C++ in the signatures).  Every
 * entry point names the reference interface it replaces; reference paths are
 * relative to /root/reference/proj/include/pswarm/.
 *
 * Conventions:
 *   - the caller owns every host buffer; the context owns device memory;
 *   - one context per host thread, bound to one CUDA device;
 *   - every call blocks until its outputs are in host memory;
 *   - there is NO CPU fallback: without a usable sm_100 device every compute
 *     entry point returns PSWARM_ERR_NO_DEVICE (or PSWARM_ERR_CUDA);
 *   - errors mirror the reference exception hierarchy (errors.hpp:10-113)
 *     through pswarm_status + pswarm_error (coordinates and message).
 *
 * Layouts:
 *   state vector       [epoch, rx, ry, rz, vx, vy, vz]  (state.hpp:11-15)
 *   state block        N x 6m row-major, column = comp*m + t (block.hpp:17-27)
 *   samples            [trajectory][1 + S*(N-1)][6] (propagator.hpp:242-244)
 */
#ifndef PSWARM_GPU_H
#define PSWARM_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PSWARM_ABI_VERSION 2

/* Status codes: one per reference exception type (errors.hpp:10-113,
 * propagator.hpp:173-186) plus device-side failures. */
typedef enum pswarm_status {
    PSWARM_OK = 0,
    PSWARM_ERR_GENERIC = 1,         /* pswarm::Error */
    PSWARM_ERR_INVALID_SPAN = 2,    /* InvalidSpanError */
    PSWARM_ERR_INVALID_SIZE = 3,    /* InvalidSizeError */
    PSWARM_ERR_SHAPE = 4,           /* ShapeError */
    PSWARM_ERR_ALIGNMENT = 5,       /* AlignmentError */
    PSWARM_ERR_DIVERGENCE = 6,      /* DivergenceError (node, column) */
    PSWARM_ERR_SINGULARITY = 7,     /* SingularityError (body) */
    PSWARM_ERR_COVERAGE = 8,        /* CoverageError (epoch) */
    PSWARM_ERR_NON_ELLIPTIC = 9,    /* NonEllipticError */
    PSWARM_ERR_SOLVER = 10,         /* SolverError */
    PSWARM_ERR_INVALID_PLAN = 11,   /* InvalidPlanError */
    PSWARM_ERR_EMPTY_REDUCTION = 12,/* EmptyReductionError */
    PSWARM_ERR_TIMEOUT = 13,        /* TimeoutError */
    PSWARM_ERR_INCOMPLETE = 14,     /* PropagationIncompleteError; partial outputs valid */
    PSWARM_ERR_ORACLE = 15,         /* OracleError (oracle.hpp: RK step underflow / budget) */
    PSWARM_ERR_CUDA = 20,
    PSWARM_ERR_OOM = 21,
    PSWARM_ERR_NO_DEVICE = 23
} pswarm_status;

/* Error record filled on failure.  Fields not meaningful for a status are -1. */
typedef struct pswarm_error {
    int32_t status;          /* pswarm_status */
    int32_t body;            /* body index for singularities, -1 = central body / none */
    int64_t segment;         /* segment index (propagate) */
    int64_t group;           /* group index (divergence / incomplete / timeout) */
    int64_t node;            /* node row (divergence / singularity) */
    int64_t column;          /* block column (divergence) */
    int64_t trajectory;      /* trajectory slot within its group (singularity) or batch index */
    int32_t iterations;      /* iterations performed (incomplete) */
    int32_t reserved;
    double value;            /* distance (singularity), epoch (coverage), final error (incomplete) */
    char body_name[64];
    char message[512];       /* what() of the reference exception, same wording */
} pswarm_error;

/* A perturbing body (ephemeris.hpp:44-50): analytic elements or a tabulated
 * Chebyshev ephemeris.  Lengths km, angles rad, epochs s past J2000. */
typedef struct pswarm_body {
    const char* name;
    double mu;                 /* km^3/s^2 */
    int32_t kind;              /* 0 = analytic OrbitalElements, 1 = tabulated ChebyshevEphemeris */
    int32_t n_segments;        /* tabulated: number of segments */
    double elements[7];        /* analytic: a, e, i, raan, argp, M0, epoch (kepler.hpp:14-22) */
    int32_t n_coeffs;          /* tabulated: coefficients per component */
    int32_t reserved;
    const double* seg_bounds;  /* tabulated: [n_segments][2] = t_start, t_end */
    const double* coeffs;      /* tabulated: [n_segments][3][n_coeffs] (x, y, z series) */
} pswarm_body;

/* PropagationConfig (propagator.hpp:38-49) + ForceModelConfig (force_model.hpp:17-24). */
typedef struct pswarm_config {
    int64_t n_nodes;            /* informational; the segment plan's node count is used (propagator.hpp:218) */
    double tolerance;           /* default 1e-12 */
    int32_t error_mode;         /* 0 relative, 1 absolute (error_metric.hpp:12) */
    int32_t max_iterations;     /* default 100 */
    int32_t start_mode;         /* 0 warm, 1 cold, 2 hot (EXTENSION: warm + the previous segment's
                                   converged-minus-conic correction, Macomber 2015) */
    int32_t segment_policy;     /* 0 single, 1 per_orbit */
    double max_segment_periods; /* default 1.0 */
    int32_t force_kind;         /* 0 two_body, 1 n_body, 2 n_body_1pn (EXTENSION: n_body + the EIH
                                   first post-Newtonian correction) */
    int32_t n_bodies;
    double central_mu;
    const pswarm_body* bodies;
    double proximity_floor_km;  /* default 1.0 */
    int64_t p_groups;           /* grouped mode group count */
    double timeout_s;           /* 0 disables the wall-clock guard; one budget per call, except
                                   run_batch independent mode: one per trajectory, as the
                                   reference's run_independent (runner.hpp:63-80) */
    double c_light;             /* n_body_1pn: speed of light in km/s (0 = 299792.458) */
} pswarm_config;

/* Outputs of pswarm_propagate / pswarm_run_batch (PropagationResult,
 * propagator.hpp:151-169).  Any pointer may be NULL to skip that output;
 * S = segments, P = groups, M = trajectories, R = 1 + S*(N-1). */
typedef struct pswarm_outputs {
    double* terminal_states;   /* [M][7] */
    double* samples;           /* [M][R][6] */
    double* times;             /* [R] */
    int32_t* iterations;       /* [S][P] */
    double* final_error;       /* [S][P] */
    uint8_t* converged;        /* [S][P] */
    double* error_history;     /* [S][P][max_iterations], NaN-padded past the iteration count */
    uint8_t* cold_fallback;    /* [S][M] warm-start fallbacks (warnings) */
    /* filled by the library: */
    int64_t segments_reported; /* segments with valid reports (S, or failing segment + 1) */
    int64_t segments_completed;/* segments whose samples / chained states are valid */
    double device_ms;          /* device time of the solve phase, inputs resident (CUDA events) */
    double kernel_ms;          /* time inside the PC solve kernels only (CUDA events around each launch) */
    int64_t trajectory_iterations; /* sum over trajectories and segments of Picard iterations performed */
    double wall_s;             /* host wall time of the whole call */
    int64_t gpu_launches;      /* CUDA kernels launched by the call */
} pswarm_outputs;

typedef struct pswarm_ctx pswarm_ctx;

int32_t pswarm_abi_version(void);
const char* pswarm_status_name(int32_t status);

/* Device context: one CUDA device, persistent device buffers and operator
 * cache (replaces the process-wide cached_matrices, pc_matrices.hpp:106-116). */
pswarm_status pswarm_create(int32_t device, pswarm_ctx** out, pswarm_error* err);
void pswarm_destroy(pswarm_ctx* ctx);

/* Tuning knobs: "ctas_per_sm" (persistent CTAs per SM, default 1), "max_ctas" (cap
 * on the persistent grid, 0 = SM count * ctas_per_sm), "profile_phases" (1 = record
 * per-phase SM cycles of the generic slot kernel, read with pswarm_get_phase_cycles),
 * "slot_kernel" (0 auto, 1 force the generic slot kernel, 2 prefer the
 * warp-specialised one), "poison_outputs" (1 = NaN-fill the device output buffers
 * before every solve, so an unwritten sample can never read back as a stale value). */
pswarm_status pswarm_set_option(pswarm_ctx* ctx, const char* key, int64_t value);

/* Diagnostics: SM cycles summed over CTAs per kernel phase of the last call (16 slots,
 * the last one = number of CTAs).
 * Generic slot kernel: 0 claim, 1 warm start, 2 force, 3 DMMA, 4 anchor barrier,
 * 5 epilogue, 6 staged epilogue, 7 decisions, 8 retire.  Warp-specialised kernels
 * (MMA group / FP group leaders): 0 wait for F, 1 DMMA, 2 epilogue, 3 wait for b0,
 * 4 wait for Y, 5 staged rows + decisions, 6 retire + claim, 7 warm start, 8 force,
 * 9 b0, 10 force tail (singularity check / fold pass), 11 MMA barrier, 12 MMA staged
 * rows, 13 MMA decisions (folded).  Unified kernel: 0 decisions, 1 retire + claim,
 * 2 warm start, 3 force, 4 b0, 5 DMMA, 6 epilogue. */
pswarm_status pswarm_get_phase_cycles(pswarm_ctx* ctx, uint64_t* out, int32_t n);

/* Diagnostics: name of the solver kernel the last propagate/run_batch call used
 * ("k_pc_ws_fold", "k_pc_uni", "k_pc_ws", "k_pc_segment" or "" before the
 * first call). */
const char* pswarm_last_kernel(pswarm_ctx* ctx);

/* ---- batch API (the drop-in boundary) ---------------------------------- */

/* propagate(states, plan, segment_plan, config, exec) — propagator.hpp:192-347.
 * states [M][7] with a shared epoch == boundaries[0]; group_sizes[P] is the
 * GroupingPlan (block.hpp:83-106); boundaries[S+1] + n_nodes is the SegmentPlan
 * (propagator.hpp:28-34).  Returns PSWARM_ERR_INCOMPLETE with partial outputs
 * when a group does not converge (propagator.hpp:300-312). */
pswarm_status pswarm_propagate(pswarm_ctx* ctx, int64_t n_states, const double* states, int64_t n_groups,
                               const int64_t* group_sizes, int64_t n_boundaries, const double* boundaries,
                               int64_t n_nodes, const pswarm_config* config, pswarm_outputs* out,
                               pswarm_error* err);

/* run_batch(states, config, segments, mode, workers) — runner.hpp:111-135.
 * mode: 0 independent, 1 augmented_sequential, 2 augmented_parallel, 3 grouped
 * (runner.hpp:21).  `workers` has no device meaning and is only validated. */
pswarm_status pswarm_run_batch(pswarm_ctx* ctx, int64_t n_states, const double* states, int64_t n_boundaries,
                               const double* boundaries, int64_t n_nodes, const pswarm_config* config,
                               int32_t mode, int32_t workers, pswarm_outputs* out, pswarm_error* err);

/* ---- multi-device (one process, several GPUs) -------------------------
 * run_batch over the devices of one node (runner.hpp:111-135): contiguous
 * group-aligned trajectory shards (block.hpp:83-106), one host thread + one context per
 * device, no collective inside the iteration or segment loop, and ONE gather of the
 * terminal states to devices[0] — NCCL send/recv over NVLink when the devices are
 * distinct (libnccl opened at run time), a device-to-device / peer copy when a device is
 * listed more than once.  Outputs have the single-device layout and batch order; errors
 * are the one the serial reference would raise (lowest failing trajectory in independent
 * mode; first failing segment, then group, otherwise).  device_ms / kernel_ms are the max
 * over devices, trajectory_iterations and gpu_launches the sums. */
typedef struct pswarm_multi pswarm_multi;
pswarm_status pswarm_create_multi(int32_t n_devices, const int32_t* devices, pswarm_multi** out, pswarm_error* err);
void pswarm_destroy_multi(pswarm_multi* m);
const char* pswarm_multi_backend(pswarm_multi* m);
int32_t pswarm_multi_devices(pswarm_multi* m);
pswarm_status pswarm_run_batch_multi(pswarm_multi* m, int64_t n_states, const double* states, int64_t n_boundaries,
                                     const double* boundaries, int64_t n_nodes, const pswarm_config* config,
                                     int32_t mode, int32_t workers, pswarm_outputs* out, pswarm_error* err);

/* ---- operator-level entry points (host buffers; one device pass each) -- */

/* picard_update_into(mats, F, y0, out) — pc_matrices.hpp:123-151.
 * force [N][C], initial_row [C], out [N][C]; any C >= 1. */
pswarm_status pswarm_picard_update(pswarm_ctx* ctx, int64_t n_nodes, int64_t n_cols, const double* force,
                                   const double* initial_row, double* out, pswarm_error* err);

/* picard_update_into(mats, F, y0, out) with the CALLER's operators (pc_matrices.hpp:123-151
 * applies mats.update_op / mats.anchor_op, whatever they hold — selftest.hpp:24-35
 * perturbs them as a negative control).  update_op [N][N], anchor_op [N]. */
pswarm_status pswarm_picard_update_ops(pswarm_ctx* ctx, int64_t n_nodes, int64_t n_cols, const double* update_op,
                                       const double* anchor_op, const double* force, const double* initial_row,
                                       double* out, pswarm_error* err);

/* eval_force_block_data(y, m, grid, table, config, force) — force_model.hpp:93-142.
 * y [N][6m]; body_positions [B][N][3] frozen per node (ephemeris.hpp:77-86). */
pswarm_status pswarm_eval_force_block(pswarm_ctx* ctx, int64_t n_nodes, int64_t group_size, const double* y,
                                      double omega2, int32_t force_kind, double central_mu, int32_t n_bodies,
                                      const double* body_positions, const double* body_mus,
                                      const char* const* body_names, double proximity_floor_km, double* force,
                                      pswarm_error* err);

/* block_iteration_error(cur, prev, mode) — augment.hpp:32-104.
 * cur/prev [N][6m]; per_state [m] (may be NULL); group_max (may be NULL). */
pswarm_status pswarm_block_iteration_error(pswarm_ctx* ctx, int64_t n_nodes, int64_t group_size, const double* cur,
                                           const double* prev, int32_t error_mode, double* per_state,
                                           double* group_max, pswarm_error* err);

/* warm_start(states, grid, mu) — propagator.hpp:81-103 via kepler_propagate
 * (kepler.hpp:59-98).  states [M][7]; times [N]; guesses [M][N][6]. */
pswarm_status pswarm_warm_start(pswarm_ctx* ctx, int64_t n_states, const double* states, int64_t n_nodes,
                                const double* times, double central_mu, double* guesses, uint8_t* cold_fallback,
                                pswarm_error* err);

/* ---- independent verifier (the CLI's --oracle-check, cli.hpp:238-261) --- */

/* oracle_sample_trajectory + compare_trajectories (oracle.hpp:136-183) for every
 * trajectory at once: adaptive Fehlberg 7(8) (rk_propagate, oracle.hpp:63-132; OracleConfig
 * rel_tol / abs_tol / max_steps) with the continuous-time force (acceleration_at,
 * force_model.hpp:78-87; body positions at every stage epoch), one device thread per
 * trajectory.  states [M][7] with epoch == times[0]; times [R] (propagate's result times);
 * candidate [M][R][6] (e.g. propagate's samples) or NULL.  Outputs, each may be NULL:
 * samples_out [M][R][6] = the RK samples, node_error [M][R] = max(position, velocity)
 * relative discrepancy of candidate vs RK per node, max_error [M] (max_combined). */
pswarm_status pswarm_oracle_check(pswarm_ctx* ctx, int64_t n_states, const double* states, int64_t n_times,
                                  const double* times, const pswarm_config* config, double rel_tol, double abs_tol,
                                  int64_t max_steps, const double* candidate, double* samples_out,
                                  double* node_error, double* max_error, pswarm_error* err);

/* ---- host utilities (no device needed; same code as the C++ headers) ---- */

/* elements_to_state (kepler.hpp:102-131): elements [a e i raan argp M0 epoch] -> state [7]. */
pswarm_status pswarm_elements_to_state(const double* elements, double mu, double t, double* state_out,
                                       pswarm_error* err);
/* osculating_period (kepler.hpp:45-53). */
pswarm_status pswarm_osculating_period(const double* state, double mu, double* period, pswarm_error* err);
/* plan_segments (propagator.hpp:109-148); policy 0 single, 1 per_orbit. */
pswarm_status pswarm_plan_segments(const double* representative, double t_start, double t_end, double mu,
                                   int32_t policy, int64_t n_nodes, double max_periods, int64_t capacity,
                                   double* boundaries, int64_t* n_boundaries, pswarm_error* err);
/* build_grid (chebyshev.hpp:61-84): node times [N] and omega2. */
pswarm_status pswarm_build_grid(int64_t n_nodes, double t_start, double t_end, double* times, double* omega2,
                                pswarm_error* err);
/* make_clone_batch (synthetic.hpp:66-83), bit-exact splitmix64 stream; out [count][7]. */
void pswarm_make_clone_batch(const double* base, int64_t count, double relative_spread, uint64_t seed,
                             double* out);

/* Page-locked host memory for result buffers (no reference analogue): device->host copies
 * into it run at DMA speed and it is never re-faulted between calls.  NULL on failure. */
void* pswarm_pinned_alloc(size_t bytes);
void pswarm_pinned_free(void* p);

#ifdef __cplusplus
}
#endif
#endif /* PSWARM_GPU_H */
