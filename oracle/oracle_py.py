"""Python handle on the CPU oracle (oracle/liboracle.so).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / ``--impl reference`` leg of bench.py, and only as the checker or
the CPU baseline.  The product never imports this module.  Entry points mirror
the device C-ABI one for one (same descriptors), so every parity test calls the
two sides with identical arguments.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from paper_2301_03989_b200 import _abi
from paper_2301_03989_b200.api import (PropagationIncompleteError, _ConfigMarshal, _Outputs, _states, RUN_MODES,
                                       parse_run_mode, raise_for, split_groups)

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "liboracle.so")
KAT = os.path.join(HERE, "kat_tests")
# the reference's OWN sources compiled here (oracle/Makefile.ref; needs /root/reference
# at build time, the built .so travels to the GPU box)
REF_LIB = os.path.join(HERE, "_ref", "libpswarm_refsrc.so")
REF_SRC = "/root/reference/proj/include/pswarm"

_dp = C.POINTER(C.c_double)
_ep = C.POINTER(_abi.PswarmError)


def build(force: bool = False) -> None:
    """Compile the oracle (g++, -O3 -ffp-contract=off, no -march) with its Makefile."""
    if force or not (os.path.exists(LIB) and os.path.exists(KAT)):
        subprocess.run(["make", "-s", "-C", HERE], check=True)


def build_reference(force: bool = False) -> bool:
    """Compile oracle/_ref from the reference's own sources when they are present
    (this container); returns whether oracle/_ref/libpswarm_refsrc.so exists."""
    if os.path.isdir(REF_SRC) and (force or not os.path.exists(REF_LIB)):
        subprocess.run(["make", "-s", "-C", HERE, "-f", "Makefile.ref"], check=True)
    return os.path.exists(REF_LIB)


def reference_available() -> bool:
    return os.path.exists(REF_LIB)


class Oracle:
    """CPU checker.  Default: the Eigen-free restatement (oracle/pswarm_ref.hpp,
    liboracle.so).  Oracle(reference=True): the reference's own sources
    (oracle/_ref/libpswarm_refsrc.so) behind the same entry points (batch
    propagation, run_batch, operators, Picard update, clone batches)."""

    def __init__(self, reference: bool = False):
        self.is_reference = reference
        if reference:
            if not reference_available():
                raise FileNotFoundError(f"{REF_LIB} not built (oracle/Makefile.ref needs /root/reference)")
            lib = C.CDLL(REF_LIB)
        else:
            build()
            lib = C.CDLL(LIB)
        sig = {
            "ref_propagate": [C.c_int64, _dp, C.c_int64, C.POINTER(C.c_int64), C.c_int64, _dp, C.c_int64,
                              C.POINTER(_abi.PswarmConfig), C.c_int32, C.c_int32, C.POINTER(_abi.PswarmOutputs), _ep],
            "ref_run_batch": [C.c_int64, _dp, C.c_int64, _dp, C.c_int64, C.POINTER(_abi.PswarmConfig), C.c_int32,
                              C.c_int32, C.POINTER(_abi.PswarmOutputs), _ep],
            "ref_picard_update": [C.c_int64, C.c_int64, _dp, _dp, _dp, _ep],
            "ref_build_operators": [C.c_int64, _dp, _dp, _ep],
            "ref_eval_force_block": [C.c_int64, C.c_int64, _dp, C.c_double, C.c_int32, C.c_double, C.c_int32, _dp,
                                     _dp, C.POINTER(C.c_char_p), C.c_double, _dp, _ep],
            "ref_block_iteration_error": [C.c_int64, C.c_int64, _dp, _dp, C.c_int32, _dp, _dp, _ep],
            "ref_warm_start": [C.c_int64, _dp, C.c_int64, _dp, C.c_double, _dp, C.POINTER(C.c_uint8), _ep],
            "ref_kepler_propagate": [_dp, C.c_double, C.c_double, _dp, _ep],
            "ref_elements_to_state": [_dp, C.c_double, C.c_double, _dp, _ep],
            "ref_osculating_period": [_dp, C.c_double, _dp, _ep],
            "ref_plan_segments": [_dp, C.c_double, C.c_double, C.c_double, C.c_int32, C.c_int64, C.c_double,
                                  C.c_int64, _dp, C.POINTER(C.c_int64), _ep],
            "ref_build_grid": [C.c_int64, C.c_double, C.c_double, _dp, _dp, _ep],
            "ref_body_positions": [C.c_int32, C.POINTER(_abi.PswarmBody), C.c_double, C.c_int64, _dp, _dp, _ep],
            "ref_rk_sample": [_dp, C.POINTER(_abi.PswarmConfig), C.c_int64, _dp, _dp, _ep],
        }
        for name, args in sig.items():
            if not hasattr(lib, name):  # the reference-source library exports the batch subset
                continue
            fn = getattr(lib, name)
            fn.restype = C.c_int32
            fn.argtypes = args
        lib.ref_make_clone_batch.restype = None
        lib.ref_make_clone_batch.argtypes = [_dp, C.c_int64, C.c_double, C.c_uint64, _dp]
        lib.ref_reference_state.restype = None
        lib.ref_reference_state.argtypes = [_dp]
        lib.ref_hardware_threads.restype = C.c_uint
        self.lib = lib

    @staticmethod
    def _ok(status, err):
        if status != _abi.OK:
            raise_for(status, err)

    # ---- batch ------------------------------------------------------------
    def propagate(self, states, group_sizes, plan, config, group_workers=1, inner_workers=1, samples=True):
        st = _states(states)
        gs = np.ascontiguousarray(np.asarray(group_sizes, dtype=np.int64))
        cm = _ConfigMarshal(config)
        b = np.ascontiguousarray(plan.boundaries, dtype=np.float64)
        outs = _Outputs(st.shape[0], len(gs), len(b) - 1, plan.n_nodes, config.max_iterations, samples)
        err = _abi.PswarmError()
        s = self.lib.ref_propagate(st.shape[0], _abi.dptr(st), len(gs), gs.ctypes.data_as(C.POINTER(C.c_int64)),
                                   len(b), _abi.dptr(b), plan.n_nodes, C.byref(cm.cfg), group_workers, inner_workers,
                                   C.byref(outs.out), C.byref(err))
        return self._finish(s, err, outs, gs, plan, False)

    def run_batch(self, states, config, plan, mode="independent", workers=1, samples=True):
        st = _states(states)
        mode = parse_run_mode(mode)
        M = st.shape[0]
        gs = (np.ones(M, np.int64) if mode == "independent" else
              np.array([M], np.int64) if mode.startswith("augmented") else
              split_groups(M, min(max(config.p_groups, 1), M)))
        cm = _ConfigMarshal(config)
        b = np.ascontiguousarray(plan.boundaries, dtype=np.float64)
        outs = _Outputs(M, len(gs), len(b) - 1, plan.n_nodes, config.max_iterations, samples)
        err = _abi.PswarmError()
        s = self.lib.ref_run_batch(M, _abi.dptr(st), len(b), _abi.dptr(b), plan.n_nodes, C.byref(cm.cfg),
                                   RUN_MODES[mode], workers, C.byref(outs.out), C.byref(err))
        return self._finish(s, err, outs, gs, plan, mode == "independent")

    def _finish(self, status, err, outs, gs, plan, indep):
        if status == _abi.ERR_INCOMPLETE:
            raise PropagationIncompleteError(err.message.decode(), err.segment, err.group,
                                             outs.result(gs, plan, False, indep))
        self._ok(status, err)
        return outs.result(gs, plan, True, indep)

    # ---- operators --------------------------------------------------------
    def picard_update(self, force, initial_row):
        f = np.ascontiguousarray(force, dtype=np.float64)
        y0 = np.ascontiguousarray(initial_row, dtype=np.float64).ravel()
        out = np.zeros_like(f)
        err = _abi.PswarmError()
        self._ok(self.lib.ref_picard_update(f.shape[0], f.shape[1], _abi.dptr(f), _abi.dptr(y0), _abi.dptr(out),
                                            C.byref(err)), err)
        return out

    def operators(self, n):
        u = np.zeros((n, n))
        a = np.zeros(n)
        err = _abi.PswarmError()
        self._ok(self.lib.ref_build_operators(n, _abi.dptr(u), _abi.dptr(a), C.byref(err)), err)
        return u, a

    def eval_force_block(self, y, group_size, omega2, force_kind, central_mu, body_positions=None, body_mus=None,
                         body_names=None, proximity_floor_km=1.0):
        yy = np.ascontiguousarray(y, dtype=np.float64)
        B = 0 if body_positions is None else len(body_mus)
        pos = np.ascontiguousarray(body_positions if B else np.zeros((1, 1, 3)), dtype=np.float64)
        mus = np.ascontiguousarray(body_mus if B else np.zeros(1), dtype=np.float64)
        names = (C.c_char_p * max(1, B))(*[n.encode() for n in (body_names or [""] * B)])
        out = np.zeros_like(yy)
        err = _abi.PswarmError()
        self._ok(self.lib.ref_eval_force_block(yy.shape[0], group_size, _abi.dptr(yy), omega2,
                                               1 if force_kind == "n_body" else 0, central_mu, B, _abi.dptr(pos),
                                               _abi.dptr(mus), names, proximity_floor_km, _abi.dptr(out),
                                               C.byref(err)), err)
        return out

    def block_iteration_error(self, cur, prev, group_size, error_mode="relative"):
        c = np.ascontiguousarray(cur, dtype=np.float64)
        p = np.ascontiguousarray(prev, dtype=np.float64)
        per = np.zeros(group_size)
        g = C.c_double()
        err = _abi.PswarmError()
        self._ok(self.lib.ref_block_iteration_error(c.shape[0], group_size, _abi.dptr(c), _abi.dptr(p),
                                                    1 if error_mode == "absolute" else 0, _abi.dptr(per), C.byref(g),
                                                    C.byref(err)), err)
        return per, g.value

    def warm_start(self, states, times, mu):
        st = _states(states)
        t = np.ascontiguousarray(times, dtype=np.float64)
        g = np.zeros((st.shape[0], t.size, 6))
        fb = np.zeros(st.shape[0], dtype=np.uint8)
        err = _abi.PswarmError()
        self._ok(self.lib.ref_warm_start(st.shape[0], _abi.dptr(st), t.size, _abi.dptr(t), mu, _abi.dptr(g),
                                         fb.ctypes.data_as(C.POINTER(C.c_uint8)), C.byref(err)), err)
        return g, fb.astype(bool)

    # ---- host helpers -----------------------------------------------------
    def kepler_propagate(self, state, mu, dt):
        s = np.ascontiguousarray(state, dtype=np.float64)
        o = np.zeros(7)
        err = _abi.PswarmError()
        self._ok(self.lib.ref_kepler_propagate(_abi.dptr(s), mu, dt, _abi.dptr(o), C.byref(err)), err)
        return o

    def elements_to_state(self, el, mu, t):
        e = np.ascontiguousarray(el, dtype=np.float64)
        o = np.zeros(7)
        err = _abi.PswarmError()
        self._ok(self.lib.ref_elements_to_state(_abi.dptr(e), mu, t, _abi.dptr(o), C.byref(err)), err)
        return o

    def osculating_period(self, state, mu):
        s = np.ascontiguousarray(state, dtype=np.float64)
        p = C.c_double()
        err = _abi.PswarmError()
        self._ok(self.lib.ref_osculating_period(_abi.dptr(s), mu, C.byref(p), C.byref(err)), err)
        return p.value

    def plan_boundaries(self, rep, t0, t1, mu, policy="single", n_nodes=200, max_periods=1.0):
        s = np.ascontiguousarray(rep, dtype=np.float64)
        b = np.zeros(4096)
        nb = C.c_int64()
        err = _abi.PswarmError()
        self._ok(self.lib.ref_plan_segments(_abi.dptr(s), t0, t1, mu, 1 if policy == "per_orbit" else 0, n_nodes,
                                            max_periods, 4096, _abi.dptr(b), C.byref(nb), C.byref(err)), err)
        return b[:nb.value].copy()

    def build_grid(self, n, t0, t1):
        t = np.zeros(n)
        w = C.c_double()
        err = _abi.PswarmError()
        self._ok(self.lib.ref_build_grid(n, t0, t1, _abi.dptr(t), C.byref(w), C.byref(err)), err)
        return t, w.value

    def body_positions(self, bodies, central_mu, times):
        from paper_2301_03989_b200.api import PropagationConfig
        m = _ConfigMarshal(PropagationConfig(force_kind="n_body", central_mu=central_mu, bodies=list(bodies)))
        t = np.ascontiguousarray(times, dtype=np.float64)
        out = np.zeros((len(bodies), t.size, 3))
        err = _abi.PswarmError()
        self._ok(self.lib.ref_body_positions(len(bodies), m.bodies, central_mu, t.size, _abi.dptr(t), _abi.dptr(out),
                                             C.byref(err)), err)
        return out

    def make_clone_batch(self, base, count, spread=1e-5, seed=20220411):
        b = np.ascontiguousarray(base, dtype=np.float64)
        o = np.zeros((count, 7))
        self.lib.ref_make_clone_batch(_abi.dptr(b), count, spread, C.c_uint64(seed), _abi.dptr(o))
        return o

    def reference_state(self):
        o = np.zeros(7)
        self.lib.ref_reference_state(_abi.dptr(o))
        return o

    def rk_sample(self, state, config, times):
        s = np.ascontiguousarray(state, dtype=np.float64)
        t = np.ascontiguousarray(times, dtype=np.float64)
        cm = _ConfigMarshal(config)
        out = np.zeros((t.size, 6))
        err = _abi.PswarmError()
        self._ok(self.lib.ref_rk_sample(_abi.dptr(s), C.byref(cm.cfg), t.size, _abi.dptr(t), _abi.dptr(out),
                                        C.byref(err)), err)
        return out

    def hardware_threads(self):
        return int(self.lib.ref_hardware_threads())
