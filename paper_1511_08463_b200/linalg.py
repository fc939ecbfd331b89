"""Linear-solver errors and reports, mirroring the reference names (linalg.py:21-50).

The solvers themselves run on the device (libphasefrac_b200.so: PCG with Jacobi
preconditioning, masked inactive-block PCG for the damage VI, field-split MINRES
for the coupled Newton step); their C-ABI status codes map onto these classes.
"""

from __future__ import annotations

from dataclasses import dataclass


class LinearSolverError(Exception):
    """Base class for linear-solver failures (reference linalg.py:21)."""


class BreakdownError(LinearSolverError):
    """Krylov breakdown: indefinite operator or preconditioner (linalg.py:25)."""


class SingularOperatorError(LinearSolverError):
    """Kept for API compatibility; the device path has no LU (linalg.py:29)."""

    def __init__(self, message: str, pivot: int = -1):
        super().__init__(message)
        self.pivot = pivot


class InnerSolverError(LinearSolverError):
    """Failure of an inner field-split solve, tagged with its block (linalg.py:37)."""

    def __init__(self, block: str, cause: Exception):
        super().__init__(f"inner solve on block {block!r} failed: {cause}")
        self.block = block
        self.cause = cause


@dataclass
class LinearSolveReport:
    iterations: int
    final_residual_norm: float
    converged: bool
