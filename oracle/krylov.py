"""Sparse linear solvers -- oracle (test infrastructure only).

Restates ``linalg.py`` of the reference: PCG with the true-residual stopping
rule and breakdown checks (``linalg.py:106-152``), preconditioned MINRES in
Paige-Saunders form (``:155-219``), SuperLU factorisation (``:250-262``),
Jacobi / Chebyshev preconditioners (``:294-305, 331-378``) and the symmetric
multiplicative field split (``:398-430``).
"""

from __future__ import annotations

from dataclasses import dataclass

import os

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

# SuperLU column ordering.  The reference calls splu with its default (COLAMD, linalg.py:256);
# the full-size step-local parity runs (tools/steplocal.py) set ORACLE_LU_PERMC=MMD_AT_PLUS_A, a
# symmetric minimum-degree ordering with ~2.3x less fill on these SPD FE blocks -- the solves agree
# to round-off, the factorisation is ~4x faster at 512^2.
LU_PERMC = os.environ.get("ORACLE_LU_PERMC", "COLAMD")


class SolverFailure(Exception):
    """Base class (reference: LinearSolverError, linalg.py:21)."""


class Breakdown(SolverFailure):
    """Krylov breakdown (reference: BreakdownError, linalg.py:25)."""


class SingularMatrix(SolverFailure):
    """Zero pivot in LU (reference: SingularOperatorError, linalg.py:29)."""


class InnerFailure(SolverFailure):
    """Field-split inner failure tagged with its block (linalg.py:37-43)."""

    def __init__(self, block, cause):
        super().__init__(f"inner solve on block {block!r} failed: {cause}")
        self.block = block


@dataclass
class KrylovStats:
    iterations: int
    residual: float
    converged: bool


def _op(A):
    if hasattr(A, "matvec") and not sp.issparse(A):
        return A.matvec
    return lambda x: A @ x


def _prec(M, r):
    if M is None:
        return r
    return M.matvec(r) if hasattr(M, "matvec") else M(r)


def pcg(A, b, M=None, rtol=1e-10, atol=0.0, maxit=None, x0=None):
    """PCG with x0 = 0 by default; stop when ||r|| <= max(rtol ||b||, atol)."""
    mv = _op(A)
    n = b.shape[0]
    maxit = 10 * n if maxit is None else maxit
    bn = float(np.linalg.norm(b))
    tgt = max(rtol * bn, atol)
    if x0 is None:
        x = np.zeros(n)
        if bn == 0.0:
            return x, KrylovStats(0, 0.0, True)
        r = b.copy()
    else:
        x = x0.copy()
        r = b - mv(x)
    rn = float(np.linalg.norm(r))
    if rn <= tgt:
        return x, KrylovStats(0, rn, True)
    z = _prec(M, r)
    rz = float(r @ z)
    if rz <= 0.0:
        raise Breakdown(f"pcg: preconditioner not SPD at iteration 0 (r'z={rz:.3e})")
    p = z.copy()
    k = 0
    while k < maxit and rn > tgt:
        q = mv(p)
        pq = float(p @ q)
        if pq <= 0.0:
            raise Breakdown(f"pcg: p'Ap = {pq:.3e} <= 0 at iteration {k + 1}")
        g = rz / pq
        x += g * p
        r -= g * q
        k += 1
        rn = float(np.linalg.norm(r))
        if rn <= tgt:
            break
        z = _prec(M, r)
        rz2 = float(r @ z)
        if rz2 <= 0.0:
            raise Breakdown(f"pcg: preconditioner not SPD at iteration {k}")
        p = z + (rz2 / rz) * p
        rz = rz2
    return x, KrylovStats(k, rn, rn <= tgt)


def minres(A, b, M=None, rtol=1e-8, atol=0.0, maxit=None):
    """Preconditioned MINRES, x0 = 0; stops on the preconditioned residual phibar."""
    mv = _op(A)
    n = b.shape[0]
    maxit = 10 * n if maxit is None else maxit
    x = np.zeros(n)
    r1 = b.copy()
    y = _prec(M, r1)
    b1 = float(r1 @ y)
    if b1 < 0.0:
        raise Breakdown("minres: preconditioner not SPD")
    b1 = np.sqrt(b1)
    if b1 == 0.0:
        return x, KrylovStats(0, 0.0, True)
    tgt = max(rtol * b1, atol)
    oldb, beta, dbar, eps, phibar = 0.0, b1, 0.0, 0.0, b1
    cs, sn = -1.0, 0.0
    w = np.zeros(n)
    w2 = np.zeros(n)
    r2 = r1
    k = 0
    while k < maxit and phibar > tgt:
        k += 1
        v = (1.0 / beta) * y
        y = mv(v)
        if k >= 2:
            y = y - (beta / oldb) * r1
        alf = float(v @ y)
        y = y - (alf / beta) * r2
        r1, r2 = r2, y
        y = _prec(M, r2)
        oldb = beta
        beta = float(r2 @ y)
        if beta < 0.0:
            raise Breakdown(f"minres: preconditioner not SPD at iteration {k}")
        beta = np.sqrt(beta)
        oldeps = eps
        delta = cs * dbar + sn * alf
        gbar = sn * dbar - cs * alf
        eps = sn * beta
        dbar = -cs * beta
        gam = max(np.hypot(gbar, beta), np.finfo(float).eps)
        cs, sn = gbar / gam, beta / gam
        phi = cs * phibar
        phibar = sn * phibar
        w1, w2 = w2, w
        w = (v - oldeps * w1 - delta * w2) / gam
        x = x + phi * w
    return x, KrylovStats(k, float(phibar), phibar <= tgt)


def lu_solver(A):
    """SuperLU factorisation returning b -> x (linalg.py:250-262)."""
    A = sp.csc_matrix(A)
    if A.shape[0] == 0:
        return lambda b: np.zeros(0)
    try:
        lu = spla.splu(A, permc_spec=LU_PERMC)
    except RuntimeError as exc:
        raise SingularMatrix(str(exc)) from exc
    return lambda b: lu.solve(np.asarray(b, dtype=float))


class Jacobi:
    def __init__(self, A):
        d = np.asarray(A.diagonal(), dtype=float)
        if np.any(d <= 0):
            raise ValueError("jacobi preconditioner needs a positive diagonal")
        self.dinv = 1.0 / d

    def matvec(self, r):
        return self.dinv * r


class Chebyshev:
    """Degree-k Chebyshev in D^-1 A on [lmax/30, 1.1 lmax] (linalg.py:331-378)."""

    def __init__(self, A, degree=3, power_iterations=30):
        self.A = sp.csr_matrix(A)
        d = np.asarray(A.diagonal(), dtype=float)
        if np.any(d <= 0):
            raise ValueError("chebyshev preconditioner needs a positive diagonal")
        self.dinv = 1.0 / d
        n = A.shape[0]
        v = 1.0 + np.arange(n) / max(n - 1, 1)
        v /= np.linalg.norm(v)
        lam = 1.0
        for _ in range(power_iterations):
            w = self.dinv * (self.A @ v)
            lam = np.linalg.norm(w)
            v = w / lam
        hi = 1.1 * lam
        lo = hi / 30.0
        self.theta, self.delta, self.degree = 0.5 * (hi + lo), 0.5 * (hi - lo), degree

    def matvec(self, r):
        th, de = self.theta, self.delta
        s1 = th / de
        rho = 1.0 / s1
        res = self.dinv * r
        d = res / th
        x = d.copy()
        for _ in range(self.degree - 1):
            res = res - self.dinv * (self.A @ d)
            rn = 1.0 / (2.0 * s1 - rho)
            d = rn * rho * d + (2.0 * rn / de) * res
            rho = rn
            x = x + d
        return x


class Block2x2:
    """[[A, B], [B^T, C]] (linalg.py:53-80)."""

    def __init__(self, A, B, C):
        self.A, self.B, self.C = A, B, C
        self.nu = A.shape[0]
        self.shape = (A.shape[0] + C.shape[0],) * 2

    def matvec(self, x):
        xu, xa = x[: self.nu], x[self.nu:]
        return np.concatenate([self.A @ xu + self.B @ xa, self.B.T @ xu + self.C @ xa])

    def csr(self):
        return sp.bmat([[self.A, self.B], [self.B.T, self.C]], format="csr")


class FieldSplit:
    """Symmetric multiplicative split with C as Schur stand-in (linalg.py:398-430)."""

    def __init__(self, blk: Block2x2, inv_a, inv_c):
        self.B = blk.B.tocsr()
        self.Bt = blk.B.T.tocsr()
        self.inv_a, self.inv_c, self.nu = inv_a, inv_c, blk.nu

    def _run(self, f, b, tag):
        try:
            return f(b)
        except Exception as exc:  # noqa: BLE001
            raise InnerFailure(tag, exc) from exc

    def matvec(self, r):
        ru, ra = r[: self.nu], r[self.nu:]
        y1 = self._run(self.inv_a, ru, "A")
        z = self._run(self.inv_c, ra - self.Bt @ y1, "C")
        xu = y1 - self._run(self.inv_a, self.B @ z, "A")
        return np.concatenate([xu, z])


def sub(A, rows, cols):
    return A[rows][:, cols].tocsr()
