"""B200-native restarted PDHG (raPDHG / r2HPDHG) LP engine -- Python binding.

Thin ctypes marshalling over the C ABI in include/lp.h (libmpax_b200.so, built
in-tree for sm_100a).  Every step of the method runs in the library's CUDA
kernels; there is no CPU fallback: importing works without a GPU (so the
symbols can be inspected), but any solve raises if CUDA is unavailable.
"""
from .lp import (  # noqa: F401
    LP_DEVICE, LP_HOST, LP_OPTIMAL, LP_ITERATION_LIMIT, LP_NUMERICAL_ERROR, LP_PRIMAL_INFEASIBLE, LP_DUAL_INFEASIBLE,
    RAPDHG, R2HPDHG,
    PATH_AUTO, PATH_INSTANCE, PATH_GRID, PATH_DMMA, STEP_ADAPTIVE, STEP_CONSTANT, FP64, FP32, LpError, Problem, Options, Result, Solver, BatchSolver,
    create_lp, default_options, lib, library_path, launch_count, selftest_division, EXPORTED_SYMBOLS, RESULT_DTYPE,
    ShardedSolver, row_partition, local_rows, col_partition, local_cols, shard_axis, SHARD_ROWS, SHARD_COLS, SHARD_AUTO, nccl_unique_id, nccl_comm_init, nccl_comm_destroy,
)
