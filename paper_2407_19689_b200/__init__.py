"""B200-native PDOT: restarted PDHG for discrete optimal transport on sm_100a.

Drop-in for the reference ``otsolve`` iteration path (pdhg.py:254-399): the
same names, signatures, records and exception types, with every pass over
the m x n plan executed by hand-written CUDA kernels in ``libpdot.so``
(C ABI: include/pdot.h).  There is no CPU fallback.
"""

from .config import (ABSOLUTE, ADAPTIVE, FIXED_BETA, RELATIVE, SolverConfig, SolveTrace, StepState,
                     default_stepsize, primal_weight_update, should_restart)
from .device import DeviceProblem, release_handles
from .engine import solve, solve_device
from .entropic import Potentials, SinkhornConfig, sinkhorn_report_gap, sinkhorn_solve
from .instance_io import load_instance, save_instance
from .instances import CostMatrix, InstanceError, Marginal, OTProblem, grid_cost, grid_problem, make_problem
from .records import Iterate, KKTReport, SolveReport
from .units import (adaptive_stepsize, apply_A, apply_At, duality_gap, kkt_error, pdhg_step,
                    restart_candidate, round_to_feasible, rounded_objective, rounding_bound_check,
                    stepsize_bound)
from .sweep import BenchSummary, geomean_gap, run_bench, sgm10

__all__ = [
    "ABSOLUTE", "ADAPTIVE", "FIXED_BETA", "RELATIVE", "SolverConfig", "SolveTrace", "StepState",
    "default_stepsize", "primal_weight_update", "should_restart", "DeviceProblem", "release_handles",
    "solve", "solve_device", "CostMatrix", "InstanceError", "Marginal", "OTProblem", "make_problem",
    "Iterate", "KKTReport", "SolveReport", "adaptive_stepsize", "apply_A", "apply_At", "duality_gap",
    "kkt_error", "pdhg_step", "restart_candidate", "round_to_feasible", "rounded_objective",
    "stepsize_bound", "Potentials", "SinkhornConfig", "sinkhorn_report_gap", "sinkhorn_solve",
    "rounding_bound_check", "load_instance", "save_instance", "grid_cost", "grid_problem",
    "BenchSummary", "geomean_gap", "run_bench", "sgm10",
]

__version__ = "0.1.0"
