"""B200-native (sm_100a) augmented Picard–Chebyshev batch propagator.

Drop-in for the batch-propagation path of the reference ``pswarm``
(/root/reference/proj/include/pswarm): the C++ API lives in ``include/pswarm/``
and calls the CUDA library ``libpswarm_b200.so`` through the C-ABI declared in
``include/pswarm_gpu.h``; this package is the Python view of the same boundary.
"""
from .api import (  # noqa: F401
    MU_SUN, AlignmentError, BodySpec, Context, MultiContext, CoverageError, DeviceError, DivergenceError, EmptyReductionError,
    Error, InvalidPlanError, InvalidSizeError, InvalidSpanError, IterationReport, NonEllipticError, OracleError,
    PropagationConfig, PropagationIncompleteError, PropagationResult, SegmentPlan, ShapeError, SingularityError,
    SolverError, TimeoutError, build_grid, default_context, elements_to_state, make_clone_batch,
    max_state_discrepancy, osculating_period, parse_run_mode, plan_segments, planets8, reference_bodies,
    reference_force_config, reference_state, split_groups, BenchmarkReport, BenchmarkRow, run_benchmark,
    pinned_sample_buffer, pinned_terminal_buffer,
)
