"""Solver status / result types (mirror of fastvol/solver.py:14-32).  The
numeric solvers themselves run on the GPU (csrc/fv_quote.h)."""

import enum
from dataclasses import dataclass


class SolverStatus(enum.Enum):
    CONVERGED = "converged"
    FELL_BACK_TO_BISECTION = "fell_back_to_bisection"
    BELOW_INTRINSIC = "below_intrinsic"
    ABOVE_UPPER_BOUND = "above_upper_bound"
    MAX_ITERATIONS = "max_iterations"

    @property
    def ok(self) -> bool:
        return self in (SolverStatus.CONVERGED, SolverStatus.FELL_BACK_TO_BISECTION)


@dataclass(frozen=True)
class SolverResult:
    sigma: float
    iterations: int
    status: SolverStatus
    residual: float


# C ABI status codes -> reference strings (solver.py:15-19 in order;
# batch.py:270-274 for Greeks)
IV_STATUS_NAMES = tuple(s.value for s in SolverStatus)
GREEK_STATUS_NAMES = ("ok", "step_function_edge")
