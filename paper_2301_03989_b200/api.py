"""Python mirror of the reference batch-propagation API over the C-ABI.

Names, argument meaning and error behaviour follow /root/reference/proj/include/pswarm
(propagator.hpp, runner.hpp, pc_matrices.hpp, force_model.hpp, augment.hpp,
kepler.hpp, synthetic.hpp).  Every compute call goes through
``libpswarm_b200.so`` (hand-written sm_100a CUDA); there is no CPU fallback —
without a B200 the calls raise ``DeviceError``.  Host utilities (plan_segments,
elements_to_state, make_clone_batch, ...) are the same C++ code the C++ headers
use and run without a device.
"""
from __future__ import annotations

import ctypes as C
import os
import sys
import threading
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _abi

MU_SUN = 1.32712440018e11  # synthetic.hpp:15


# ----------------------------------------------------------------- errors --
class Error(RuntimeError):
    """pswarm::Error (errors.hpp:10-13)."""


class InvalidSpanError(Error): ...
class InvalidSizeError(Error): ...
class ShapeError(Error): ...
class AlignmentError(Error): ...
class NonEllipticError(Error): ...
class SolverError(Error): ...
class InvalidPlanError(Error): ...
class EmptyReductionError(Error): ...
class TimeoutError(Error): ...  # noqa: A001 - reference name
class OracleError(Error): ...
class DeviceError(Error):
    """CUDA / device failure or no B200 visible (no reference analogue)."""


class DivergenceError(Error):
    def __init__(self, msg, node, column):
        super().__init__(msg)
        self.node, self.column = node, column


class SingularityError(Error):
    def __init__(self, msg, body=""):
        super().__init__(msg)
        self.body = body


class CoverageError(Error):
    def __init__(self, msg, epoch):
        super().__init__(msg)
        self.epoch = epoch


class PropagationIncompleteError(Error):
    def __init__(self, msg, segment, group, partial):
        super().__init__(msg)
        self.segment, self.group, self.partial = segment, group, partial


_SIMPLE = {
    _abi.ERR_GENERIC: Error, _abi.ERR_INVALID_SPAN: InvalidSpanError, _abi.ERR_INVALID_SIZE: InvalidSizeError,
    _abi.ERR_SHAPE: ShapeError, _abi.ERR_ALIGNMENT: AlignmentError, _abi.ERR_NON_ELLIPTIC: NonEllipticError,
    _abi.ERR_SOLVER: SolverError, _abi.ERR_INVALID_PLAN: InvalidPlanError,
    _abi.ERR_EMPTY_REDUCTION: EmptyReductionError, _abi.ERR_TIMEOUT: TimeoutError, _abi.ERR_ORACLE: OracleError,
    _abi.ERR_CUDA: DeviceError, _abi.ERR_OOM: DeviceError, _abi.ERR_NO_DEVICE: DeviceError,
}


def raise_for(status: int, err: _abi.PswarmError):
    msg = err.message.decode(errors="replace")
    if status == _abi.ERR_DIVERGENCE:
        raise DivergenceError(msg, err.node, err.column)
    if status == _abi.ERR_SINGULARITY:
        raise SingularityError(msg, err.body_name.decode(errors="replace"))
    if status == _abi.ERR_COVERAGE:
        raise CoverageError(msg, err.value)
    raise _SIMPLE.get(status, Error)(msg)


def _check(status, err):
    if status != _abi.OK:
        raise_for(status, err)


# ------------------------------------------------------------ data types --
@dataclass
class BodySpec:
    """BodySpec (ephemeris.hpp:44-50): analytic elements (a, e, i, raan, argp, M0, epoch)
    or a tabulated Chebyshev ephemeris [(t_start, t_end, cx, cy, cz), ...]."""
    name: str
    mu: float
    elements: Optional[Sequence[float]] = None
    segments: Optional[list] = None


FORCE_KINDS = {"two_body": 0, "n_body": 1, "n_body_1pn": 2}  # n_body_1pn: EXTENSION (EIH 1PN)
START_MODES = {"warm": 0, "cold": 1, "hot": 2}  # hot: EXTENSION (Macomber hot start)


@dataclass
class PropagationConfig:
    """PropagationConfig + ForceModelConfig (propagator.hpp:38-49, force_model.hpp:17-24)."""
    n_nodes: int = 200
    tolerance: float = 1e-12
    error_mode: str = "relative"
    max_iterations: int = 100
    start_mode: str = "warm"
    segment_policy: str = "single"
    max_segment_periods: float = 1.0
    force_kind: str = "two_body"
    central_mu: float = 0.0
    bodies: List[BodySpec] = field(default_factory=list)
    proximity_floor_km: float = 1.0
    p_groups: int = 1
    timeout_s: float = 0.0
    c_light: float = 299792.458  # km/s, force_kind "n_body_1pn" only (EXTENSION)


@dataclass
class SegmentPlan:
    """SegmentPlan (propagator.hpp:28-34)."""
    boundaries: np.ndarray
    n_nodes: int = 200

    @property
    def direction(self) -> str:
        return "forward" if self.boundaries[-1] > self.boundaries[0] else "backward"

    def segments(self) -> int:
        return len(self.boundaries) - 1


@dataclass
class IterationReport:
    iterations: int
    final_error: float
    converged: bool
    per_iteration_errors: np.ndarray


class _Reports(Sequence):
    """reports[segment][group] -> IterationReport, built on access from the flat
    per-(segment, group) arrays the C-ABI fills (a batch of 10^5 groups would
    otherwise pay for 10^5 Python objects per call)."""

    class _Row(Sequence):
        def __init__(self, src, s):
            self.src, self.s = src, s

        def __len__(self):
            return self.src.P

        def __getitem__(self, g):
            if isinstance(g, slice):
                return [self[i] for i in range(*g.indices(len(self)))]
            src, s = self.src, self.s
            if g < 0:
                g += src.P
            if not 0 <= g < src.P:
                raise IndexError(g)
            it = int(src.iters[s, g])
            h = src.hist[s, g, :min(it, src.max_it)].copy() if src.hist is not None else np.zeros(0)
            return IterationReport(it, float(src.ferr[s, g]), bool(src.conv[s, g]), h)

    def __init__(self, iters, ferr, conv, hist, max_it, n_segments):
        self.iters, self.ferr, self.conv, self.hist, self.max_it = iters, ferr, conv, hist, max_it
        self.P = iters.shape[1]
        self.S = n_segments

    def __len__(self):
        return self.S

    def __getitem__(self, s):
        if isinstance(s, slice):
            return [self[i] for i in range(*s.indices(len(self)))]
        if s < 0:
            s += self.S
        if not 0 <= s < self.S:
            raise IndexError(s)
        return _Reports._Row(self, s)


@dataclass
class PropagationResult:
    """PropagationResult (propagator.hpp:151-169) plus device timing."""
    times: np.ndarray
    trajectories: Optional[np.ndarray]  # [M, R, 6]
    terminal_states: Optional[np.ndarray]  # [M, 7]
    reports: Sequence  # reports[segment][group] -> IterationReport
    group_sizes: np.ndarray
    segments: SegmentPlan
    warnings: List[str]
    iterations: np.ndarray  # [S_reported, P]
    converged: np.ndarray
    device_ms: float = 0.0
    kernel_ms: float = 0.0
    trajectory_iterations: int = 0
    gpu_launches: int = 0
    wall_s: float = 0.0

    def max_iterations_used(self) -> int:
        return int(self.iterations.max()) if self.iterations.size else 0


class _ConfigMarshal:
    """Keeps the ctypes view of a PropagationConfig (and its arrays) alive."""

    def __init__(self, cfg: PropagationConfig):
        bodies = list(cfg.bodies)
        self.keep = []
        arr = (_abi.PswarmBody * max(1, len(bodies)))()
        for k, b in enumerate(bodies):
            pb = arr[k]
            name = b.name.encode()
            self.keep.append(name)
            pb.name = name
            pb.mu = b.mu
            if b.segments is None:
                pb.kind = 0
                for i, x in enumerate(b.elements):
                    pb.elements[i] = x
            else:
                nc = max(len(s[2]) for s in b.segments)
                bounds = np.array([[s[0], s[1]] for s in b.segments], dtype=np.float64).ravel()
                coeffs = np.zeros((len(b.segments), 3, nc))
                for si, s in enumerate(b.segments):
                    for c in range(3):
                        coeffs[si, c, :len(s[2 + c])] = s[2 + c]
                coeffs = np.ascontiguousarray(coeffs.ravel())
                self.keep += [bounds, coeffs]
                pb.kind = 1
                pb.n_segments = len(b.segments)
                pb.n_coeffs = nc
                pb.seg_bounds = _abi.dptr(bounds)
                pb.coeffs = _abi.dptr(coeffs)
        self.bodies = arr
        c = _abi.PswarmConfig()
        c.n_nodes = cfg.n_nodes
        c.tolerance = cfg.tolerance
        c.error_mode = 1 if cfg.error_mode == "absolute" else 0
        c.max_iterations = cfg.max_iterations
        c.start_mode = START_MODES[cfg.start_mode]
        c.segment_policy = 1 if cfg.segment_policy == "per_orbit" else 0
        c.max_segment_periods = cfg.max_segment_periods
        c.force_kind = FORCE_KINDS[cfg.force_kind]
        c.n_bodies = len(bodies)
        c.central_mu = cfg.central_mu
        c.bodies = C.cast(arr, C.POINTER(_abi.PswarmBody))
        c.proximity_floor_km = cfg.proximity_floor_km
        c.p_groups = cfg.p_groups
        c.timeout_s = cfg.timeout_s
        c.c_light = cfg.c_light
        self.cfg = c


def pinned_sample_buffer(n_states: int, plan: "SegmentPlan") -> np.ndarray:
    """Page-locked [M, R, 6] buffer for `samples=` of propagate/run_batch: with it the
    library copies each segment's node samples while the next segment computes (the
    overlapped D2H of pswarm_propagate).  Allocate once and reuse across calls."""
    import torch
    R = 1 + (len(plan.boundaries) - 1) * (plan.n_nodes - 1)
    return torch.zeros((n_states, R, 6), dtype=torch.float64, pin_memory=True).numpy()


def pinned_terminal_buffer(n_states: int) -> np.ndarray:
    """Page-locked [M, 7] buffer for `terminal=` of propagate/run_batch: the library then
    writes the terminal states (epoch, r, v) with one device->host DMA straight into it
    (no staging copy, no page faults on a fresh array).  Allocate once and reuse."""
    import torch
    return torch.zeros((n_states, 7), dtype=torch.float64, pin_memory=True).numpy()


_SINGLETONS: dict = {}


def _singletons(m: int) -> np.ndarray:
    """Independent mode's group sizes (all 1) as a cached read-only array: a 1M-trajectory call
    does not allocate and fill 8 MB per call for it."""
    a = _SINGLETONS.get(m)
    if a is None:
        a = np.ones(m, dtype=np.int64)
        a.setflags(write=False)
        _SINGLETONS.clear()
        _SINGLETONS[m] = a
    return a


def _pooled_bytes(pool, n):
    """A zeroed uint8 buffer of n bytes from `pool` (a list kept by the context): a buffer whose
    only reference is the pool's is reused -- memset instead of the first-touch page faults of a
    fresh allocation (14 MB of reports per 1M-trajectory call) -- else a new one joins the pool
    (at most two: a caller that keeps every result keeps getting fresh buffers)."""
    if pool is not None:
        for buf in pool:
            # references: the pool list, the loop variable, getrefcount's argument -- no live
            # result, view or report of an earlier call still points into it
            if buf.nbytes >= n and sys.getrefcount(buf) <= 3:
                view = buf[:n]
                view.fill(0)
                return view
    buf = np.zeros(n, dtype=np.uint8)
    if pool is not None and (1 << 20) <= n <= (256 << 20):  # retained memory stays bounded
        if len(pool) >= 2:
            pool.pop(0)
        pool.append(buf)
    return buf


class _Outputs:
    def __init__(self, M, P, S, N, max_it, samples=True, history=True, terminal=True, pool=None):
        R = 1 + S * (N - 1)
        self.M, self.P, self.S, self.R, self.max_it = M, P, S, R, max(max_it, 0)
        if isinstance(terminal, np.ndarray):  # caller-owned (e.g. pinned_terminal_buffer) output
            if terminal.shape != (M, 7) or terminal.dtype != np.float64 or not terminal.flags.c_contiguous:
                raise ShapeError(f"terminal buffer must be float64 C-contiguous of shape {(M, 7)}")
            self.terminal = terminal
        else:
            # np.empty: the C side writes every element a reported segment / complete call exposes
            self.terminal = np.empty((M, 7)) if terminal else None
        if isinstance(samples, np.ndarray):  # caller-owned (e.g. pinned_sample_buffer) output
            if samples.shape != (M, R, 6) or samples.dtype != np.float64 or not samples.flags.c_contiguous:
                raise ShapeError(f"samples buffer must be float64 C-contiguous of shape {(M, R, 6)}")
            self.samples = samples
        else:
            self.samples = np.zeros((M, R, 6)) if samples else None
        # the small per-call outputs share one buffer: one address lookup instead of five
        # (numpy's data-pointer lookup dominates the wrapper's cost for small batches)
        def al(n):
            return (n + 7) & ~7
        o_t, o_e = 0, al(8 * R)
        o_i = o_e + al(8 * S * P)
        o_c = o_i + al(4 * S * P)
        o_f = o_c + al(S * P)
        small = _pooled_bytes(pool, o_f + al(S * M))  # zeroed: not every writer fills every entry
        base = small.__array_interface__["data"][0]
        self.times = np.ndarray((R,), np.float64, small, o_t)
        self.ferr = np.ndarray((S, P), np.float64, small, o_e)
        self.iters = np.ndarray((S, P), np.int32, small, o_i)
        self.conv = np.ndarray((S, P), np.uint8, small, o_c)
        self.fb = np.ndarray((S, M), np.uint8, small, o_f)
        self.hist = np.zeros((S, P, max(self.max_it, 1))) if history else None
        o = _abi.PswarmOutputs()
        ad = _abi.addr
        o.terminal_states = ad(self.terminal)
        o.samples = ad(self.samples)
        o.times = base + o_t
        o.iterations = base + o_i
        o.final_error = base + o_e
        o.converged = base + o_c
        o.error_history = ad(self.hist)
        o.cold_fallback = base + o_f
        self.out = o

    def result(self, group_sizes, plan: SegmentPlan, complete: bool, independent: bool) -> PropagationResult:
        o = self.out
        S_rep = int(o.segments_reported)
        reports = _Reports(self.iters, self.ferr, self.conv, self.hist, self.max_it, S_rep)
        warnings = []
        for s in range(S_rep):
            for i in np.nonzero(self.fb[s])[0]:
                w = f"segment {s}, trajectory {0 if independent else i}: non-elliptic state, cold start used"
                warnings.append(f"trajectory {i}: {w}" if independent else w)
        return PropagationResult(
            times=self.times, trajectories=self.samples,
            terminal_states=self.terminal if complete else None, reports=reports,
            group_sizes=np.asarray(group_sizes, dtype=np.int64), segments=plan, warnings=warnings,
            iterations=self.iters[:S_rep], converged=self.conv[:S_rep],  # views of this call's buffer
            device_ms=o.device_ms, kernel_ms=o.kernel_ms, trajectory_iterations=int(o.trajectory_iterations),
            gpu_launches=int(o.gpu_launches), wall_s=o.wall_s)


def _states(states) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(states, dtype=np.float64))
    if a.ndim != 2 or a.shape[1] != 7:
        raise ShapeError(f"states must be [M, 7] (epoch, r, v), got {a.shape}")
    return a


RUN_MODES = {"independent": 0, "augmented_sequential": 1, "augmented_parallel": 2, "augmented": 2, "grouped": 3}


def parse_run_mode(name: str) -> str:  # runner.hpp:32-38
    if name not in RUN_MODES:
        raise Error(f"unknown run mode '{name}'")
    return "augmented_parallel" if name == "augmented" else name


class Context:
    """One device context (pswarm_ctx) bound to a CUDA device."""

    def __init__(self, device: int = -1):
        self._report_pool = []  # reusable report buffers of large calls (_pooled_bytes)
        self.lib = _abi.load()
        self.ptr = C.c_void_p()
        err = _abi.PswarmError()
        _check(self.lib.pswarm_create(device, C.byref(self.ptr), C.byref(err)), err)

    def close(self):
        if self.ptr:
            self.lib.pswarm_destroy(self.ptr)
            self.ptr = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_option(self, key: str, value: int):
        if self.lib.pswarm_set_option(self.ptr, key.encode(), int(value)) != _abi.OK:
            raise Error(f"unknown option {key}")

    PHASE_NAMES = ("claim", "warm_start", "force", "dmma", "anchor_barrier", "epilogue", "staged_epilogue",
                   "decisions", "retire")
    WS_PHASE_NAMES = ("mma_wait_f", "mma_dmma", "mma_epilogue", "mma_wait_b0", "fp_wait_y", "fp_staged_decisions",
                      "fp_retire_claim", "fp_warm_start", "fp_force", "fp_b0", "fp_staged",
                      "mma_bar_epi", "mma_staged", "mma_decisions")
    UNI_PHASE_NAMES = ("decisions", "retire_claim", "warm_start", "force", "sing_b0", "dmma", "epilogue", "fold_b0")
    N_PHASES = 16

    def phase_cycles(self) -> dict:
        """Per-phase SM cycles of the last solve (requires set_option('profile_phases', 1)),
        named after the solver kernel that ran."""
        buf = (C.c_uint64 * self.N_PHASES)()
        self.lib.pswarm_get_phase_cycles(self.ptr, buf, self.N_PHASES)
        kn = self.kernel_name()
        names = (self.UNI_PHASE_NAMES if kn == "k_pc_uni" else
                 self.WS_PHASE_NAMES if kn.startswith("k_pc_ws") else self.PHASE_NAMES)
        d = {n: int(buf[k]) for k, n in enumerate(names)}
        d["ctas"] = int(buf[self.N_PHASES - 1])
        return d

    def kernel_name(self) -> str:
        """Solver kernel used by the last propagate/run_batch call."""
        return self.lib.pswarm_last_kernel(self.ptr).decode()

    # ---- batch API ------------------------------------------------------
    def propagate(self, states, group_sizes, plan: SegmentPlan, config: PropagationConfig, *,
                  samples=True, history=True, terminal=True) -> PropagationResult:
        """propagate (propagator.hpp:192-347)."""
        st = _states(states)
        gs = np.ascontiguousarray(np.asarray(group_sizes, dtype=np.int64))
        return self._call(st, gs, plan, config, None, 1, samples, history, terminal)

    def run_batch(self, states, config: PropagationConfig, plan: SegmentPlan, mode: str = "independent",
                  workers: int = 1, *, samples=True, history=True, terminal=True) -> PropagationResult:
        """run_batch (runner.hpp:111-135); independent == per-trajectory convergence masking."""
        st = _states(states)
        mode = parse_run_mode(mode)
        M = st.shape[0]
        if mode == "independent":
            gs = _singletons(M)
        elif mode.startswith("augmented"):
            gs = np.array([M], dtype=np.int64)
        else:
            gs = split_groups(M, min(max(config.p_groups, 1), max(M, 1))) if M > 0 else np.zeros(0, np.int64)
        return self._call(st, gs, plan, config, mode, workers, samples, history, terminal)

    def _marshal(self, config: PropagationConfig) -> "_ConfigMarshal":
        """ctypes view of the config, cached per context on a fingerprint of every value the
        C side reads (a mutated config or body list gets a fresh marshal)."""
        if any(b.segments is not None for b in config.bodies):
            return _ConfigMarshal(config)  # tabulated coefficients may change in place: no cache
        bodies = tuple((b.name, b.mu, tuple(b.elements)) for b in config.bodies)
        key = (config.n_nodes, config.tolerance, config.error_mode, config.max_iterations, config.start_mode,
               config.segment_policy, config.max_segment_periods, config.force_kind, config.central_mu,
               config.proximity_floor_km, config.p_groups, config.timeout_s, config.c_light, bodies)
        cache = self.__dict__.setdefault("_marshal_cache", {})
        cm = cache.get(key)
        if cm is None:
            if len(cache) >= 16:
                cache.clear()
            cm = cache[key] = _ConfigMarshal(config)
        return cm

    def _call(self, st, gs, plan, config, mode, workers, samples, history, terminal):
        cm = self._marshal(config)
        b = np.ascontiguousarray(np.asarray(plan.boundaries, dtype=np.float64))
        S = max(len(b) - 1, 0)
        outs = _Outputs(st.shape[0], len(gs), S, plan.n_nodes, config.max_iterations, samples, history, terminal,
                        pool=self._report_pool)
        err = _abi.PswarmError()
        if mode is None:
            status = self.lib.pswarm_propagate(self.ptr, st.shape[0], _abi.dptr(st), len(gs),
                                               gs.ctypes.data_as(C.POINTER(C.c_int64)), len(b), _abi.dptr(b),
                                               plan.n_nodes, C.byref(cm.cfg), C.byref(outs.out), C.byref(err))
        else:
            status = self.lib.pswarm_run_batch(self.ptr, st.shape[0], _abi.dptr(st), len(b), _abi.dptr(b),
                                               plan.n_nodes, C.byref(cm.cfg), RUN_MODES[mode], workers,
                                               C.byref(outs.out), C.byref(err))
        indep = mode == "independent"
        if status == _abi.ERR_INCOMPLETE:
            partial = outs.result(gs, plan, False, indep)
            raise PropagationIncompleteError(err.message.decode(), err.segment, err.group, partial)
        _check(status, err)
        return outs.result(gs, plan, True, indep)

    # ---- operator-level entry points --------------------------------------
    def picard_update(self, force: np.ndarray, initial_row: np.ndarray, update_op=None,
                      anchor_op=None) -> np.ndarray:
        """picard_update_into (pc_matrices.hpp:123-151) on the device: the context's
        operators for N = rows(force), or the caller's (update_op [N][N], anchor_op [N])."""
        f = np.ascontiguousarray(force, dtype=np.float64)
        y0 = np.ascontiguousarray(initial_row, dtype=np.float64).ravel()
        if f.ndim != 2:
            raise ShapeError("picard_update: force block must be 2-D")
        if y0.size != f.shape[1]:
            raise ShapeError(f"picard_update: initial row has {y0.size} columns, force block has {f.shape[1]}")
        out = np.zeros_like(f)
        err = _abi.PswarmError()
        if update_op is None:
            _check(self.lib.pswarm_picard_update(self.ptr, f.shape[0], f.shape[1], _abi.dptr(f), _abi.dptr(y0),
                                                 _abi.dptr(out), C.byref(err)), err)
            return out
        u = np.ascontiguousarray(update_op, dtype=np.float64)
        a = np.ascontiguousarray(anchor_op, dtype=np.float64).ravel()
        if u.shape != (f.shape[0], f.shape[0]) or a.size != f.shape[0]:
            raise ShapeError(f"picard_update: operators do not match n_nodes = {f.shape[0]}")
        _check(self.lib.pswarm_picard_update_ops(self.ptr, f.shape[0], f.shape[1], _abi.dptr(u), _abi.dptr(a),
                                                 _abi.dptr(f), _abi.dptr(y0), _abi.dptr(out), C.byref(err)), err)
        return out

    def eval_force_block(self, y, group_size, omega2, force_kind, central_mu, body_positions=None, body_mus=None,
                         body_names=None, proximity_floor_km=1.0) -> np.ndarray:
        """eval_force_block_data (force_model.hpp:93-142); body_positions [B, N, 3]."""
        yy = np.ascontiguousarray(y, dtype=np.float64)
        N = yy.shape[0]
        if yy.shape[1] != 6 * group_size:
            raise ShapeError(f"eval_force_block: state block is {yy.shape[0]}x{yy.shape[1]}, expected "
                             f"{N}x{6 * group_size}")
        B = 0 if body_positions is None else len(body_mus)
        pos = np.ascontiguousarray(body_positions if B else np.zeros((1, 1, 3)), dtype=np.float64)
        mus = np.ascontiguousarray(body_mus if B else np.zeros(1), dtype=np.float64)
        names = (C.c_char_p * max(1, B))(*[n.encode() for n in (body_names or [""] * B)])
        out = np.zeros_like(yy)
        err = _abi.PswarmError()
        kind = FORCE_KINDS[force_kind]
        _check(self.lib.pswarm_eval_force_block(self.ptr, N, group_size, _abi.dptr(yy), omega2, kind, central_mu, B,
                                                _abi.dptr(pos), _abi.dptr(mus), names, proximity_floor_km,
                                                _abi.dptr(out), C.byref(err)), err)
        return out

    def block_iteration_error(self, cur, prev, group_size, error_mode="relative"):
        """block_iteration_error (augment.hpp:80-104) -> (per_state, group_max)."""
        c = np.ascontiguousarray(cur, dtype=np.float64)
        p = np.ascontiguousarray(prev, dtype=np.float64)
        if c.shape != p.shape or c.shape[1] != 6 * group_size:
            raise ShapeError("block_iteration_error: block shapes do not match")
        per = np.zeros(group_size)
        gmax = C.c_double(0.0)
        err = _abi.PswarmError()
        _check(self.lib.pswarm_block_iteration_error(self.ptr, c.shape[0], group_size, _abi.dptr(c), _abi.dptr(p),
                                                     1 if error_mode == "absolute" else 0, _abi.dptr(per),
                                                     C.byref(gmax), C.byref(err)), err)
        return per, gmax.value

    def warm_start(self, states, times, central_mu):
        """warm_start (propagator.hpp:81-103) -> (guesses [M, N, 6], cold_fallback [M])."""
        st = _states(states)
        t = np.ascontiguousarray(times, dtype=np.float64)
        g = np.zeros((st.shape[0], t.size, 6))
        fb = np.zeros(st.shape[0], dtype=np.uint8)
        err = _abi.PswarmError()
        _check(self.lib.pswarm_warm_start(self.ptr, st.shape[0], _abi.dptr(st), t.size, _abi.dptr(t), central_mu,
                                          _abi.dptr(g), fb.ctypes.data_as(C.POINTER(C.c_uint8)), C.byref(err)), err)
        return g, fb.astype(bool)

    def oracle_check(self, states, config: "PropagationConfig", times, candidate=None, rel_tol=1e-13,
                     abs_tol=1e-16, max_steps=4000000, samples=True):
        """The CLI's --oracle-check (cli.hpp:238-261) on the device: RKF7(8)
        oracle_sample_trajectory + compare_trajectories (oracle.hpp:63-183) for every
        trajectory.  Returns (rk_samples [M, R, 6] or None, node_error [M, R] or None,
        max_error [M] or None); the errors need `candidate` (e.g. result.trajectories)."""
        st = _states(states)
        t = np.ascontiguousarray(times, dtype=np.float64)
        M, R = st.shape[0], t.size
        m = _ConfigMarshal(config)
        cand = None if candidate is None else np.ascontiguousarray(candidate, dtype=np.float64).reshape(M, R, 6)
        out = np.zeros((M, R, 6)) if samples else None
        node = np.zeros((M, R)) if cand is not None else None
        mx = np.zeros(M) if cand is not None else None
        err = _abi.PswarmError()
        _check(self.lib.pswarm_oracle_check(self.ptr, M, _abi.dptr(st), R, _abi.dptr(t), C.byref(m.cfg), rel_tol,
                                            abs_tol, max_steps, _abi.dptr(cand), _abi.dptr(out), _abi.dptr(node),
                                            _abi.dptr(mx), C.byref(err)), err)
        return out, node, mx


_default = threading.local()


def default_context() -> Context:
    if getattr(_default, "ctx", None) is None:
        _default.ctx = Context(-1)
    return _default.ctx


# ----------------------------------------------------------- host utilities --
def _host(fn, *args):
    err = _abi.PswarmError()
    _check(fn(*args, C.byref(err)), err)


def elements_to_state(elements, mu, t) -> np.ndarray:
    el = np.ascontiguousarray(elements, dtype=np.float64)
    out = np.zeros(7)
    _host(_abi.load().pswarm_elements_to_state, _abi.dptr(el), mu, t, _abi.dptr(out))
    return out


def osculating_period(state, mu) -> float:
    s = np.ascontiguousarray(state, dtype=np.float64)
    p = C.c_double()
    _host(_abi.load().pswarm_osculating_period, _abi.dptr(s), mu, C.byref(p))
    return p.value


def plan_segments(representative, t_start, t_end, mu, policy="single", n_nodes=200, max_periods=1.0) -> SegmentPlan:
    s = np.ascontiguousarray(representative, dtype=np.float64)
    cap = 4096
    b = np.zeros(cap)
    nb = C.c_int64()
    _host(_abi.load().pswarm_plan_segments, _abi.dptr(s), t_start, t_end, mu, 1 if policy == "per_orbit" else 0,
          n_nodes, max_periods, cap, _abi.dptr(b), C.byref(nb))
    return SegmentPlan(b[:nb.value].copy(), n_nodes)


def build_grid(n_nodes, t_start, t_end):
    t = np.zeros(n_nodes)
    w2 = C.c_double()
    _host(_abi.load().pswarm_build_grid, n_nodes, t_start, t_end, _abi.dptr(t), C.byref(w2))
    return t, w2.value


def make_clone_batch(base, count, relative_spread=1e-5, seed=20220411) -> np.ndarray:
    """make_clone_batch (synthetic.hpp:66-83), bit-exact; returns [count, 7]."""
    b = np.ascontiguousarray(base, dtype=np.float64)
    out = np.zeros((count, 7))
    _abi.load().pswarm_make_clone_batch(_abi.dptr(b), count, relative_spread, C.c_uint64(seed), _abi.dptr(out))
    return out


def split_groups(total, p_groups) -> np.ndarray:
    """Balanced contiguous split, larger groups first (block.hpp:110-126)."""
    if total < 1 or p_groups < 1 or p_groups > total:
        raise InvalidPlanError(f"split_groups: cannot split {total} states into {p_groups} groups")
    base, rem = divmod(total, p_groups)
    return np.array([base + 1 if g < rem else base for g in range(p_groups)], dtype=np.int64)


def reference_state() -> np.ndarray:  # synthetic.hpp:31-34
    return elements_to_state([1.25e8, 0.12, 0.030, 0.30, 1.00, 0.0, 0.0], MU_SUN, 0.0)


def reference_bodies() -> List[BodySpec]:  # synthetic.hpp:19-29
    return [BodySpec("venus-like", 3.24858592e5, (1.08208e8, 0.0068, 0.0593, 1.338, 0.958, 2.10, 0.0)),
            BodySpec("earth-like", 3.98600436e5, (1.495979e8, 0.0167, 0.0, 0.0, 1.796, 4.20, 0.0))]


def planets8() -> List[BodySpec]:
    """Mercury..Neptune mean J2000 elements (same table as synthetic.hpp make_planets8)."""
    rows = [
        ("mercury", 2.2031868551e4, 5.7909227e7, 0.20563593, 0.12225995, 0.84353095, 0.50831279, 3.05076572),
        ("venus", 3.24858592e5, 1.08209475e8, 0.00677672, 0.05924827, 1.33831572, 0.95791742, 0.87497675),
        ("earth", 4.03503233e5, 1.49598262e8, 0.01671123, 0.0, 0.0, 1.79676742, 6.25905804),
        ("mars", 4.282837362e4, 2.27943824e8, 0.0933941, 0.03228321, 0.86497712, 5.00040086, 0.33817734),
        ("jupiter", 1.26712764e8, 7.78340821e8, 0.04838624, 0.02276602, 1.75360053, 4.77971377, 0.34894549),
        ("saturn", 3.7940585e7, 1.426666422e9, 0.05386179, 0.04336201, 1.98378354, 5.92354458, 5.53361297),
        ("uranus", 5.794556e6, 2.870658186e9, 0.04725744, 0.01343659, 1.29164837, 1.69118766, 2.48348795),
        ("neptune", 6.836527e6, 4.498396441e9, 0.00859048, 0.03087952, 2.30006864, 4.82257416, 4.47166418),
    ]
    return [BodySpec(n, mu, (a, e, i, raan, argp, m0, 0.0)) for n, mu, a, e, i, raan, argp, m0 in rows]


def reference_force_config(kind="n_body", bodies=None, **kw) -> PropagationConfig:
    """make_reference_force_model (synthetic.hpp:36-44) folded into a PropagationConfig."""
    cfg = PropagationConfig(force_kind=kind, central_mu=MU_SUN, **kw)
    if kind != "two_body":
        cfg.bodies = list(bodies) if bodies is not None else reference_bodies()
    return cfg


def max_state_discrepancy(a: np.ndarray, b: np.ndarray) -> float:
    """runner.hpp:139-159 on sample arrays [M, R, 6] (b normalises)."""
    dr = np.linalg.norm(a[..., :3] - b[..., :3], axis=-1)
    dv = np.linalg.norm(a[..., 3:] - b[..., 3:], axis=-1)
    rn = np.maximum(np.linalg.norm(b[..., :3], axis=-1), 1e-30)
    vn = np.maximum(np.linalg.norm(b[..., 3:], axis=-1), 1e-30)
    return float(max((dr / rn).max(initial=0.0), (dv / vn).max(initial=0.0)))


@dataclass
class BenchmarkRow:  # runner.hpp:160-169
    mode: str = "independent"
    threads: int = 1
    groups: int = 1
    wall_time_s: float = 0.0
    speedup: float = 1.0
    max_iterations: int = 0
    max_discrepancy: float = 0.0
    group_iterations: list = field(default_factory=list)


@dataclass
class BenchmarkReport:
    machine: str = ""
    repeat: int = 1
    rows: list = field(default_factory=list)


def run_benchmark(ctx: "Context", states, config: PropagationConfig, plan: SegmentPlan, thread_counts=(1,),
                  modes=("independent", "augmented_parallel"), repeat: int = 5) -> BenchmarkReport:
    """run_benchmark (runner.hpp:186-253): every (mode, workers) combination `repeat` times,
    median wall time of the C-ABI call, speed-up against the independent single-worker
    baseline and the cross-mode state discrepancy.  `workers` only labels a row on the
    device (one context runs the whole batch); numerical outputs never depend on it."""
    import statistics
    if repeat < 1:
        raise InvalidPlanError("run_benchmark: repeat must be positive")
    rep = BenchmarkReport(machine=f"{os.cpu_count()} hardware threads + B200 (device path)", repeat=repeat)

    def iters_of(r):
        return [int(x) for x in np.asarray(r.iterations).ravel()]

    base_t, base = [], None
    for _ in range(repeat):
        base = ctx.run_batch(states, config, plan, "independent", 1)
        base_t.append(base.wall_s)
    base_med = statistics.median(base_t)
    for mode in modes:
        mode = parse_run_mode(mode)
        for threads in thread_counts:
            row = BenchmarkRow(mode=mode, threads=int(threads))
            if mode == "independent" and threads == 1:
                row.wall_time_s, row.groups = base_med, len(base.group_sizes)
                row.max_iterations = base.max_iterations_used()
                row.group_iterations = iters_of(base)
                rep.rows.append(row)
                continue
            ts, out = [], None
            for _ in range(repeat):
                out = ctx.run_batch(states, config, plan, mode, int(threads))
                ts.append(out.wall_s)
            row.wall_time_s = statistics.median(ts)
            row.groups = len(out.group_sizes)
            row.speedup = base_med / row.wall_time_s
            row.max_iterations = out.max_iterations_used()
            row.max_discrepancy = max_state_discrepancy(out.trajectories, base.trajectories)
            row.group_iterations = iters_of(out)
            rep.rows.append(row)
    return rep


class MultiContext:
    """run_batch over several CUDA devices of this process (pswarm_run_batch_multi): group-aligned
    trajectory shards, one host thread + context per device, one gather of the terminal states
    to devices[0] (NCCL over NVLink for distinct devices; a device copy when a device repeats).
    Results have the single-device layout and batch order."""

    def __init__(self, devices):
        self._report_pool = []  # reusable report buffers of large calls (_pooled_bytes)
        self.lib = _abi.load()
        self.ptr = C.c_void_p()
        devs = (C.c_int32 * len(devices))(*[int(d) for d in devices])
        err = _abi.PswarmError()
        _check(self.lib.pswarm_create_multi(len(devices), devs, C.byref(self.ptr), C.byref(err)), err)
        self.devices = list(devices)

    @property
    def backend(self) -> str:
        return self.lib.pswarm_multi_backend(self.ptr).decode()

    def close(self):
        if self.ptr:
            self.lib.pswarm_destroy_multi(self.ptr)
            self.ptr = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    _marshal = Context._marshal

    def run_batch(self, states, config: PropagationConfig, plan: SegmentPlan, mode: str = "independent",
                  workers: int = 1, *, samples=True, history=True, terminal=True) -> PropagationResult:
        st = _states(states)
        mode = parse_run_mode(mode)
        M = st.shape[0]
        if mode == "independent":
            gs = _singletons(M)
        elif mode.startswith("augmented"):
            gs = np.array([M], dtype=np.int64)
        else:
            gs = split_groups(M, min(max(config.p_groups, 1), max(M, 1))) if M > 0 else np.zeros(0, np.int64)
        cm = self._marshal(config)
        b = np.ascontiguousarray(np.asarray(plan.boundaries, dtype=np.float64))
        outs = _Outputs(M, len(gs), max(len(b) - 1, 0), plan.n_nodes, config.max_iterations, samples, history,
                        terminal, pool=self._report_pool)
        err = _abi.PswarmError()
        status = self.lib.pswarm_run_batch_multi(self.ptr, M, _abi.dptr(st), len(b), _abi.dptr(b), plan.n_nodes,
                                                 C.byref(cm.cfg), RUN_MODES[mode], workers, C.byref(outs.out),
                                                 C.byref(err))
        indep = mode == "independent"
        if status == _abi.ERR_INCOMPLETE:
            raise PropagationIncompleteError(err.message.decode(), err.segment, err.group,
                                             outs.result(gs, plan, False, indep))
        _check(status, err)
        return outs.result(gs, plan, True, indep)

