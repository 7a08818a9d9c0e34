"""CPU-side checks of the drop-in boundary: the C-ABI library loads and exports
every symbol include/pswarm_gpu.h declares, the host utilities reproduce the
reference (oracle) bit for bit, validation follows the reference's order and
wording, and the compute path refuses to run without a device (no fallback)."""
import os
import re

import numpy as np
import pytest

import paper_2301_03989_b200 as ps
from paper_2301_03989_b200 import _abi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "pswarm_gpu.h")


def declared_symbols():
    text = open(HEADER).read()
    decl = r"^\s*(?:pswarm_status|void\s*\*|void|int32_t|const char\s*\*)\s*(pswarm_[a-z_0-9]+)\s*\("
    return sorted(set(re.findall(decl, text, flags=re.M)))


def test_library_exports_every_declared_symbol():
    lib = _abi.load()
    names = declared_symbols()
    assert len(names) >= 16
    for n in names:
        assert hasattr(lib, n), n
    assert {n for n, _, _ in _abi.SIGNATURES} == set(names)
    abi = int(re.search(r"#define PSWARM_ABI_VERSION (\d+)", open(HEADER).read()).group(1))
    assert lib.pswarm_abi_version() == abi == 2


def test_struct_layouts_match_header():
    # sizes implied by the header (natural alignment on x86-64)
    import ctypes as C
    assert C.sizeof(_abi.PswarmError) == 4 + 4 + 5 * 8 + 4 + 4 + 8 + 64 + 512
    assert C.sizeof(_abi.PswarmBody) == 8 + 8 + 4 + 4 + 7 * 8 + 4 + 4 + 8 + 8
    assert C.sizeof(_abi.PswarmOutputs) == 8 * 8 + 8 * 7
    assert C.sizeof(_abi.PswarmConfig) == 8 + 8 + 4 * 4 + 8 + 4 + 4 + 8 * 6  # ABI 2: + c_light


def test_clone_batch_bit_exact(oracle):
    base = ps.reference_state()
    assert np.array_equal(base, oracle.reference_state())
    for spread, seed in [(1e-5, 20220411), (2e-4, 7), (0.0, 1)]:
        assert np.array_equal(ps.make_clone_batch(base, 513, spread, seed),
                              oracle.make_clone_batch(base, 513, spread, seed))


def test_host_conics_match_oracle(oracle):
    el = [1.3e8, 0.2, 0.1, 0.5, 1.2, 0.3, 0.0]
    for t in [0.0, 1e6, -3e7, 5.5e8]:
        assert np.array_equal(ps.elements_to_state(el, ps.MU_SUN, t), oracle.elements_to_state(el, ps.MU_SUN, t))
    s = ps.reference_state()
    assert ps.osculating_period(s, ps.MU_SUN) == oracle.osculating_period(s, ps.MU_SUN)


@pytest.mark.parametrize("frac,policy,n", [(0.87, "single", 200), (2.5, "per_orbit", 64), (-1.6, "per_orbit", 32),
                                           (3.5, "per_orbit", 200)])
def test_plan_segments_identical_counts(oracle, frac, policy, n):
    s = ps.reference_state()
    p = ps.osculating_period(s, ps.MU_SUN)
    plan = ps.plan_segments(s, 0.0, frac * p, ps.MU_SUN, policy, n)
    assert np.array_equal(plan.boundaries, oracle.plan_boundaries(s, 0.0, frac * p, ps.MU_SUN, policy, n))


def test_grid_matches_oracle(oracle):
    for n, t0, t1 in [(3, 0.0, 10.0), (200, 6.64e8, 6.64e8 + 0.87 * 2.2e7), (17, 10.0, 2.0)]:
        t, w = ps.build_grid(n, t0, t1)
        tr, wr = oracle.build_grid(n, t0, t1)
        assert np.array_equal(t, tr) and w == wr


def test_plan_errors_match_reference():
    s = ps.reference_state()
    p = ps.osculating_period(s, ps.MU_SUN)
    with pytest.raises(ps.InvalidSpanError):
        ps.plan_segments(s, 5.0, 5.0, ps.MU_SUN, "single", 10)
    with pytest.raises(ps.InvalidSpanError, match="per-orbit"):
        ps.plan_segments(s, 0.0, 3.0 * p, ps.MU_SUN, "single", 10)
    hyper = np.array([0.0, 1e8, 0, 0, 0, 60.0, 0])
    with pytest.raises(ps.NonEllipticError):
        ps.plan_segments(hyper, 0.0, 1e6, ps.MU_SUN, "per_orbit", 10)
    with pytest.raises(ps.InvalidSizeError):
        ps.build_grid(2, 0.0, 1.0)


def _null_ctx_call(states, sizes, boundaries, n, cfg=None):
    """pswarm_propagate with a NULL context: validation runs, compute refuses."""
    import ctypes as C
    from paper_2301_03989_b200.api import _ConfigMarshal, _Outputs
    cm = _ConfigMarshal(cfg or ps.reference_force_config("two_body"))
    st = np.ascontiguousarray(states, dtype=np.float64)
    gs = np.ascontiguousarray(sizes, dtype=np.int64)
    b = np.ascontiguousarray(boundaries, dtype=np.float64)
    err = _abi.PswarmError()
    status = _abi.load().pswarm_propagate(None, st.shape[0], _abi.dptr(st), len(gs),
                                          gs.ctypes.data_as(C.POINTER(C.c_int64)), len(b), _abi.dptr(b), n,
                                          C.byref(cm.cfg), None, C.byref(err))
    return status, err.message.decode()


def test_validation_order_and_messages_without_device():
    s = ps.make_clone_batch(ps.reference_state(), 3, 1e-5)
    assert _null_ctx_call(s[:0], [], [0.0, 1.0], 16)[1] == "propagate: empty batch"
    st, msg = _null_ctx_call(s, [2], [0.0, 1.0], 16)
    assert st == _abi.ERR_INVALID_PLAN and msg == "propagate: grouping plan covers 2 states, batch has 3"
    assert _null_ctx_call(s, [3], [0.0], 16)[0] == _abi.ERR_INVALID_SPAN
    bad = s.copy()
    bad[2, 0] = 10.0
    st, msg = _null_ctx_call(bad, [3], [0.0, 1.0], 16)
    assert st == _abi.ERR_ALIGNMENT and "state 2" in msg
    st, msg = _null_ctx_call(s, [3], [1.0, 2.0], 16)
    assert st == _abi.ERR_ALIGNMENT and "first segment boundary" in msg
    assert _null_ctx_call(s, [3], [0.0, 1.0], 2)[0] == _abi.ERR_INVALID_SIZE
    # everything valid -> refuses to run without a device (no CPU fallback)
    st, msg = _null_ctx_call(s, [3], [0.0, 1.0], 16)
    assert st == _abi.ERR_NO_DEVICE


def test_no_device_raises_device_error():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    with pytest.raises(ps.DeviceError):
        ps.Context(0)
    with pytest.raises(ps.DeviceError):
        ps.MultiContext([0, 1])


def test_split_groups_matches_reference_rules():
    g = ps.split_groups(13509, 10)
    assert g.sum() == 13509 and g.max() - g.min() <= 1 and g[0] >= g[-1]
    with pytest.raises(ps.InvalidPlanError):
        ps.split_groups(5, 6)


def test_report_buffer_pool_reuses_only_unreferenced_buffers():
    """Large-call report buffers are recycled only when no result, view or report of an
    earlier call points into them, and come back zeroed."""
    from paper_2301_03989_b200.api import _pooled_bytes
    pool = []
    a = _pooled_bytes(pool, 2 << 20)
    a[:] = 7
    view = a[:16]
    del a
    b = _pooled_bytes(pool, 2 << 20)  # the first buffer is still referenced by `view`
    assert len(pool) == 2 and not np.shares_memory(b, view)
    del view
    b[:] = 5
    del b
    c = _pooled_bytes(pool, 1 << 20)  # both free now: the first one is reused, zeroed
    assert c.nbytes == 1 << 20 and not c.any()
    assert any(np.shares_memory(c, p) for p in pool)
    small = _pooled_bytes(pool, 100)  # small calls never enter the pool
    assert small.nbytes == 100 and len(pool) == 2
