"""B200-native Block-cells solver (arXiv 2405.17363).

The reference's batched per-cell sparse solver path -- ``run_strategy`` /
``solve_block_cells`` / ``bicg_solve`` (/root/reference/proj/core) -- built as
fused sm_100a CUDA kernels behind a C ABI (include/blockcells_b200.h).  This
package is the host-side mirror of that API plus the synthetic workload
generator; see DESIGN.md.
"""
from .solver import (  # noqa: F401
    FLAG_BREAKDOWN,
    FLAG_CONVERGED,
    FLAG_FELL_BACK,
    KERNEL_BLOCK,
    KERNEL_LATENCY,
    KERNEL_LU,
    KERNEL_MULTI,
    KERNEL_THREAD,
    KERNEL_TMEM,
    Algo,
    BatchedSystem,
    CudaError,
    DeviceSet,
    DeviceSpec,
    InvalidGrouping,
    ReductionPlan,
    SingularMatrix,
    SolveOutcome,
    SolveReport,
    Solver,
    Strategy,
    StrategyConfig,
    UnsupportedMechanism,
    bicg_solve,
    default_solver,
    iteration_reduction_ratio,
    run_strategy,
    solve_block_cells,
    solve_multi_cells,
    solve_one_cell,
)
from .workload import REGIME_C, REGIME_P, Mechanism, Regime  # noqa: F401
