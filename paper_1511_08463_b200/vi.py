"""Box-constrained VI vocabulary (reference vi.py:35-115).

The reduced-space active-set solver itself (rsls_solve, vi.py:187-264) runs on the
device inside ``pf_damage_solve`` (damage box QP) and ``pf_newton`` (coupled system);
this module keeps the configuration / report types and the FB function.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _lib


@dataclass
class VIConfig:
    """Reference VIConfig (vi.py:68-75) plus the inner-PCG tolerance of the device solve."""

    zero_tol: Optional[float] = None
    abs_tol: float = 1e-8
    max_iterations: int = 100
    ls_backtrack: float = 0.5
    ls_min_step: float = 1e-10
    armijo: float = 1e-4
    inner_rtol: float = 1e-10
    inner_maxit: int = 0
    fieldsplit_rtol: float = 1e-6
    inner_cycles: int = 0
    inner_mode: int = 0

    def to_c(self) -> _lib.VIOpts:
        return _lib.VIOpts(abs_tol=self.abs_tol, max_iterations=self.max_iterations, precond=0,
                           ls_backtrack=self.ls_backtrack, ls_min_step=self.ls_min_step,
                           armijo=self.armijo, inner_rtol=self.inner_rtol,
                           inner_maxit=self.inner_maxit,
                           zero_tol=-1.0 if self.zero_tol is None else self.zero_tol,
                           fieldsplit_rtol=self.fieldsplit_rtol, inner_cycles=self.inner_cycles,
                           inner_mode=self.inner_mode)


@dataclass
class ActiveSetReport:
    """Reference ActiveSetReport (vi.py:78-86)."""

    iterations: int
    converged: bool
    final_residual_norm: float
    residual_history: list = field(default_factory=list)
    total_krylov_iterations: int = 0
    steepest_descent_steps: int = 0
    linear_failures: int = 0

    @classmethod
    def from_c(cls, r: _lib.VIReport) -> "ActiveSetReport":
        n = min(int(r.n_history), 64)
        return cls(int(r.iterations), bool(r.converged), float(r.final_residual_norm),
                   [float(r.history[k]) for k in range(n)], int(r.total_krylov_iterations),
                   int(r.steepest_descent_steps), int(r.linear_failures))


def new_report() -> _lib.VIReport:
    return _lib.VIReport()


def fb_phi(a, b):
    """Fischer-Burmeister function sqrt(a^2 + b^2) - a - b (vi.py:89-93), host helper."""
    a = np.asarray(a, dtype=float)
    b = np.asarray(b, dtype=float)
    return np.hypot(a, b) - a - b


__all__ = ["VIConfig", "ActiveSetReport", "fb_phi", "C"]
