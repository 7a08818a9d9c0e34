"""ctypes view of the C-ABI boundary (include/pswarm_gpu.h).

Only plain-C types cross the boundary; this module mirrors the header's structs
field for field and loads the in-tree shared library
``paper_2301_03989_b200/libpswarm_b200.so`` built by ``build.build_library``.
Loading never falls back to anything: a missing library raises ``OSError``.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libpswarm_b200.so")

# pswarm_status (include/pswarm_gpu.h)
OK = 0
ERR_GENERIC = 1
ERR_INVALID_SPAN = 2
ERR_INVALID_SIZE = 3
ERR_SHAPE = 4
ERR_ALIGNMENT = 5
ERR_DIVERGENCE = 6
ERR_SINGULARITY = 7
ERR_COVERAGE = 8
ERR_NON_ELLIPTIC = 9
ERR_SOLVER = 10
ERR_INVALID_PLAN = 11
ERR_EMPTY_REDUCTION = 12
ERR_TIMEOUT = 13
ERR_INCOMPLETE = 14
ERR_ORACLE = 15
ERR_CUDA = 20
ERR_OOM = 21
ERR_NO_DEVICE = 23


class PswarmError(C.Structure):
    _fields_ = [
        ("status", C.c_int32),
        ("body", C.c_int32),
        ("segment", C.c_int64),
        ("group", C.c_int64),
        ("node", C.c_int64),
        ("column", C.c_int64),
        ("trajectory", C.c_int64),
        ("iterations", C.c_int32),
        ("reserved", C.c_int32),
        ("value", C.c_double),
        ("body_name", C.c_char * 64),
        ("message", C.c_char * 512),
    ]


class PswarmBody(C.Structure):
    _fields_ = [
        ("name", C.c_char_p),
        ("mu", C.c_double),
        ("kind", C.c_int32),
        ("n_segments", C.c_int32),
        ("elements", C.c_double * 7),
        ("n_coeffs", C.c_int32),
        ("reserved", C.c_int32),
        ("seg_bounds", C.POINTER(C.c_double)),
        ("coeffs", C.POINTER(C.c_double)),
    ]


class PswarmConfig(C.Structure):
    _fields_ = [
        ("n_nodes", C.c_int64),
        ("tolerance", C.c_double),
        ("error_mode", C.c_int32),
        ("max_iterations", C.c_int32),
        ("start_mode", C.c_int32),
        ("segment_policy", C.c_int32),
        ("max_segment_periods", C.c_double),
        ("force_kind", C.c_int32),
        ("n_bodies", C.c_int32),
        ("central_mu", C.c_double),
        ("bodies", C.POINTER(PswarmBody)),
        ("proximity_floor_km", C.c_double),
        ("p_groups", C.c_int64),
        ("timeout_s", C.c_double),
        ("c_light", C.c_double),
    ]


class PswarmOutputs(C.Structure):
    # caller-owned output arrays as raw addresses (double*, int32_t*, uint8_t* in the
    # header): set from numpy's data pointer without building ctypes pointer objects
    _fields_ = [
        ("terminal_states", C.c_void_p),
        ("samples", C.c_void_p),
        ("times", C.c_void_p),
        ("iterations", C.c_void_p),
        ("final_error", C.c_void_p),
        ("converged", C.c_void_p),
        ("error_history", C.c_void_p),
        ("cold_fallback", C.c_void_p),
        ("segments_reported", C.c_int64),
        ("segments_completed", C.c_int64),
        ("device_ms", C.c_double),
        ("kernel_ms", C.c_double),
        ("trajectory_iterations", C.c_int64),
        ("wall_s", C.c_double),
        ("gpu_launches", C.c_int64),
    ]


_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int64)
_u8 = C.POINTER(C.c_uint8)
_ep = C.POINTER(PswarmError)

# (name, restype, argtypes) for every entry point declared in include/pswarm_gpu.h
SIGNATURES = [
    ("pswarm_abi_version", C.c_int32, []),
    ("pswarm_status_name", C.c_char_p, [C.c_int32]),
    ("pswarm_create", C.c_int32, [C.c_int32, C.POINTER(C.c_void_p), _ep]),
    ("pswarm_destroy", None, [C.c_void_p]),
    ("pswarm_set_option", C.c_int32, [C.c_void_p, C.c_char_p, C.c_int64]),
    ("pswarm_get_phase_cycles", C.c_int32, [C.c_void_p, C.POINTER(C.c_uint64), C.c_int32]),
    ("pswarm_last_kernel", C.c_char_p, [C.c_void_p]),
    ("pswarm_propagate", C.c_int32,
     [C.c_void_p, C.c_int64, _dp, C.c_int64, _ip, C.c_int64, _dp, C.c_int64, C.POINTER(PswarmConfig),
      C.POINTER(PswarmOutputs), _ep]),
    ("pswarm_run_batch", C.c_int32,
     [C.c_void_p, C.c_int64, _dp, C.c_int64, _dp, C.c_int64, C.POINTER(PswarmConfig), C.c_int32, C.c_int32,
      C.POINTER(PswarmOutputs), _ep]),
    ("pswarm_create_multi", C.c_int32, [C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.c_void_p), _ep]),
    ("pswarm_destroy_multi", None, [C.c_void_p]),
    ("pswarm_multi_backend", C.c_char_p, [C.c_void_p]),
    ("pswarm_multi_devices", C.c_int32, [C.c_void_p]),
    ("pswarm_run_batch_multi", C.c_int32,
     [C.c_void_p, C.c_int64, _dp, C.c_int64, _dp, C.c_int64, C.POINTER(PswarmConfig), C.c_int32, C.c_int32,
      C.POINTER(PswarmOutputs), _ep]),
    ("pswarm_picard_update", C.c_int32, [C.c_void_p, C.c_int64, C.c_int64, _dp, _dp, _dp, _ep]),
    ("pswarm_picard_update_ops", C.c_int32, [C.c_void_p, C.c_int64, C.c_int64, _dp, _dp, _dp, _dp, _dp, _ep]),
    ("pswarm_eval_force_block", C.c_int32,
     [C.c_void_p, C.c_int64, C.c_int64, _dp, C.c_double, C.c_int32, C.c_double, C.c_int32, _dp, _dp,
      C.POINTER(C.c_char_p), C.c_double, _dp, _ep]),
    ("pswarm_block_iteration_error", C.c_int32,
     [C.c_void_p, C.c_int64, C.c_int64, _dp, _dp, C.c_int32, _dp, _dp, _ep]),
    ("pswarm_warm_start", C.c_int32, [C.c_void_p, C.c_int64, _dp, C.c_int64, _dp, C.c_double, _dp, _u8, _ep]),
    ("pswarm_oracle_check", C.c_int32, [C.c_void_p, C.c_int64, _dp, C.c_int64, _dp, C.POINTER(PswarmConfig),
                                        C.c_double, C.c_double, C.c_int64, _dp, _dp, _dp, _dp, _ep]),
    ("pswarm_elements_to_state", C.c_int32, [_dp, C.c_double, C.c_double, _dp, _ep]),
    ("pswarm_osculating_period", C.c_int32, [_dp, C.c_double, _dp, _ep]),
    ("pswarm_plan_segments", C.c_int32,
     [_dp, C.c_double, C.c_double, C.c_double, C.c_int32, C.c_int64, C.c_double, C.c_int64, _dp, _ip, _ep]),
    ("pswarm_build_grid", C.c_int32, [C.c_int64, C.c_double, C.c_double, _dp, _dp, _ep]),
    ("pswarm_make_clone_batch", None, [_dp, C.c_int64, C.c_double, C.c_uint64, _dp]),
    ("pswarm_pinned_alloc", C.c_void_p, [C.c_size_t]),
    ("pswarm_pinned_free", None, [C.c_void_p]),
]

_lib = None


def load(path: str = LIB_PATH) -> C.CDLL:
    """Load (once) the in-tree CUDA library; raises OSError when it is missing.
    PSWARM_LIB overrides the path (diagnostic builds of the same library)."""
    global _lib
    if _lib is None:
        path = os.environ.get("PSWARM_LIB", path)
        if not os.path.exists(path):
            raise OSError(f"{path} not built: run __graft_entry__.build() (nvcc, sm_100a); "
                          "the PC path has no CPU fallback")
        lib = C.CDLL(path)
        override = "PSWARM_LIB" in os.environ
        for name, res, args in SIGNATURES:
            if override and not hasattr(lib, name):  # an older diagnostic build (A/B runs)
                continue
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def dptr(a):
    """double* of a C-contiguous float64 numpy array (or None)."""
    return None if a is None else a.ctypes.data_as(_dp)


def addr(a):
    """Raw address of a C-contiguous numpy array (or None) for c_void_p fields."""
    return None if a is None else a.__array_interface__["data"][0]
