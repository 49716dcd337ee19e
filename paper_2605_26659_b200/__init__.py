"""B200-native FINOM hot path: O(N) Sinkhorn kernel matvec on sm_100a.

Drop-in for the reference's solver entry points (pkg/src/finom): the
public names mirror ``finom.solver``, ``finom.kernel1d`` and
``finom.errors``; the numerics run only in the CUDA library
``libfinom_b200.so`` (csrc/), loaded through the C ABI in
include/finom_b200.h.
"""

from . import dense, errors, kernel1d, kernel2d, mesh, solver  # noqa: F401
from .errors import *  # noqa: F401,F403
from .mesh import Grid2D, Measure, Measure2D, Mesh1D, Problem  # noqa: F401
from .solver import (  # noqa: F401
    BatchSolver1D,
    GpuAdapter1D,
    Solution,
    SolverConfig,
    SolverState,
    marginal_error,
    plan_dense,
    run_driver,
    sinkhorn_1d,
    sinkhorn_1d_batched,
    transport_cost_fast,
)
from .kernel2d import (  # noqa: F401
    GpuGridAdapter,
    GridSolver2D,
    KernelOperator2D,
    build_operator_2d,
    sinkhorn_2d,
    transport_cost_fast_2d,
)

__version__ = "0.1.0"
