"""B200-native (sm_100a) AA-PDHG / FAA-PDHG LP solver hot path.

Drop-in for the reference C++ solver API (proj/include/aapdhg/solver.hpp);
the compute path is ``lib/libaapdhg_cuda.so`` (hand-written CUDA, C-ABI in
``include/aapdhg_cuda.h``). See DESIGN.md.
"""
from .api import (AAParams, CudaError, DimensionError, DistConfig, Error, FilterParams,
                  InputError, Iterate, KktMetrics, Method, ProblemData, SingularError,
                  SolveOutput, SolveResult, SolveStatus, Solver, SolverConfig, SparseMatrix,
                  StepSizes, UnsupportedError, kkt_metrics, nccl_unique_id, partition,
                  safeguard_pass, select_step_sizes, solve, solve_sweep, sweep_cases,
                  SweepCase, vstack)

__all__ = [
    "AAParams", "CudaError", "DimensionError", "DistConfig", "Error", "FilterParams", "InputError", "Iterate",
    "KktMetrics", "Method", "ProblemData", "SingularError", "SolveOutput", "SolveResult",
    "SolveStatus", "Solver", "SolverConfig", "SparseMatrix", "StepSizes", "UnsupportedError",
    "kkt_metrics", "nccl_unique_id", "partition", "safeguard_pass", "select_step_sizes", "solve", "solve_sweep", "sweep_cases", "SweepCase", "vstack",
]
