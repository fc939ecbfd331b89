"""Box-constrained complementarity (reduced-space active set) -- oracle (test infra only).

Restates ``vi.py`` of the reference: the Fischer-Burmeister residual and its
two-sided composition (``vi.py:89-115``), the active-set rule (``:127-141``),
the merit gradient with the (1/sqrt2 - 1) subgradient (``:144-178``) and the
reduced-space semismooth Newton method with projected Armijo backtracking and
steepest-descent fallback, ``rsls_solve`` (``:187-264``).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .krylov import SolverFailure, lu_solver, sub

_S2M1 = 1.0 / np.sqrt(2.0) - 1.0


def fb(a, b):
    return np.hypot(a, b) - a - b


def fb_box(x, F, lo, hi):
    """Phi(x): free rows F; [lo, inf) -> fb(x-lo, F); (-inf, hi] -> -fb(hi-x, -F);
    [lo, hi] -> fb(x - lo, fb(hi - x, -F))."""
    flo = np.isfinite(lo)
    fhi = np.isfinite(hi)
    out = F.astype(float).copy()
    m = flo & ~fhi
    out[m] = fb(x[m] - lo[m], F[m])
    m = ~flo & fhi
    out[m] = -fb(hi[m] - x[m], -F[m])
    m = flo & fhi
    out[m] = fb(x[m] - lo[m], fb(hi[m] - x[m], -F[m]))
    return out


def active_sets(x, F, lo, hi, zeta):
    la = np.isfinite(lo) & (x - lo <= zeta) & (F > 0.0)
    ua = np.isfinite(hi) & (hi - x <= zeta) & (F < 0.0) & ~la
    return la, ua, ~(la | ua)


def _partials(a, b):
    rho = np.hypot(a, b)
    ok = rho > 0.0
    safe = np.where(ok, rho, 1.0)
    return np.where(ok, a / safe - 1.0, _S2M1), np.where(ok, b / safe - 1.0, _S2M1)


def merit_gradient(x, F, phi, Jmv, lo, hi):
    flo = np.isfinite(lo)
    fhi = np.isfinite(hi)
    p = np.zeros_like(x)
    q = np.zeros_like(x)
    q[~flo & ~fhi] = 1.0
    m = flo & ~fhi
    if m.any():
        p[m], q[m] = _partials(x[m] - lo[m], F[m])
    m = ~flo & fhi
    if m.any():
        p[m], q[m] = _partials(hi[m] - x[m], -F[m])
    m = flo & fhi
    if m.any():
        s = hi[m] - x[m]
        inner = fb(s, -F[m])
        pa, pb = _partials(x[m] - lo[m], inner)
        ia, ib = _partials(s, -F[m])
        p[m] = pa - pb * ia
        q[m] = -pb * ib
    return 2.0 * (p * phi + Jmv(q * phi))


@dataclass
class RSLSConfig:
    zero_tol: float | None = None
    abs_tol: float = 1e-8
    max_iterations: int = 100
    ls_backtrack: float = 0.5
    ls_min_step: float = 1e-10
    armijo: float = 1e-4


@dataclass
class RSLSStats:
    iterations: int = 0
    converged: bool = False
    final_residual_norm: float = np.inf
    residual_history: list = field(default_factory=list)
    total_krylov_iterations: int = 0
    steepest_descent_steps: int = 0
    linear_failures: int = 0


def lu_reduced(J, idx, rhs):
    return lu_solver(sub(J, idx, idx))(rhs), None


def rsls(residual, jacobian, lo, hi, x0, cfg: RSLSConfig | None = None, linear=None,
         jac_matvec=None):
    """Reduced-space active-set Newton; returns (x, RSLSStats)."""
    cfg = cfg or RSLSConfig()
    linear = linear or lu_reduced
    x = np.clip(np.asarray(x0, float), lo, hi)
    zeta = cfg.zero_tol
    if zeta is None:
        zeta = 1e-10 * (1.0 + (float(np.max(np.abs(x))) if x.size else 0.0))
    st = RSLSStats()
    F = residual(x)
    phi = fb_box(x, F, lo, hi)
    merit = float(phi @ phi)
    st.residual_history.append(np.sqrt(merit))

    def search(d, bound):
        mu = 1.0
        while mu >= cfg.ls_min_step:
            xt = np.clip(x + mu * d, lo, hi)
            Ft = residual(xt)
            pt = fb_box(xt, Ft, lo, hi)
            mt = float(pt @ pt)
            if mt <= bound(mu):
                return xt, Ft, pt, mt
            mu *= cfg.ls_backtrack
        return None

    for it in range(1, cfg.max_iterations + 1):
        if np.sqrt(merit) <= cfg.abs_tol:
            break
        st.iterations = it
        _, _, free = active_sets(x, F, lo, hi, zeta)
        idx = np.flatnonzero(free)
        J = jacobian(x)
        got = None
        if idx.size:
            d = np.zeros_like(x)
            try:
                dn, rep = linear(J, idx, F[idx])
                d[idx] = -dn
                if rep is not None:
                    st.total_krylov_iterations += rep.iterations
                got = search(d, lambda mu: (1.0 - 2.0 * cfg.armijo * mu) * merit)
            except (SolverFailure, np.linalg.LinAlgError):
                st.linear_failures += 1
        if got is None:
            mv = jac_matvec(J) if jac_matvec is not None else (
                J.matvec if hasattr(J, "matvec") else (lambda v: J.T @ v))
            g = merit_gradient(x, F, phi, mv, lo, hi)
            gn = float(np.linalg.norm(g))
            if gn > 0.0:
                sc = 1.0 / max(1.0, gn)
                got = search(-sc * g, lambda mu: merit - cfg.armijo * mu * sc * gn * gn)
                st.steepest_descent_steps += 1
        if got is None:
            break
        x, F, phi, merit = got
        st.residual_history.append(np.sqrt(merit))
    st.final_residual_norm = float(np.sqrt(merit))
    st.converged = st.final_residual_norm <= cfg.abs_tol
    return x, st
