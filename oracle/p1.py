"""P1 discretisation of the phase-field energy -- oracle (test infrastructure only).

Restates the reference's centroid-quadrature P1 assembly
(``fem.py:1-15, 101-156`` and ``model.py:23-76``) for simplices in 2D and 3D:

    E(u, a) = sum_e |T_e| [ 1/2 A(ab_e) (B_e u_e - eps0_e)^T D_e (B_e u_e - eps0_e)
                            + (Gc_e / c_w) (w(ab_e)/ell + ell |G_e a_e|^2) ]

ab_e is the element mean of the nodal damage, A(a) = (1-a)^2 + k_ell.
Extensions over the reference (each an exact derivative of the same discrete
functional, checked by finite differences in ``tests/test_oracle_fd.py``):

* damage model AT2: w = a^2, c_w = 2 (reference has AT1 only, ``model.py:20,73-76``);
* plane strain and 3D isotropic D (reference: plane stress, ``model.py:49-55``);
* per-element E and Gc multipliers (reference: scalars);
* 3D Voigt order (e11, e22, e33, g23, g13, g12), engineering shears.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import NamedTuple, Optional

import numpy as np
import scipy.sparse as sp

from .meshgen import SimplexMesh


class EnergyParts(NamedTuple):
    elastic: float
    dissipated: float
    total: float


@dataclass(frozen=True)
class MaterialSpec:
    E: float = 1.0
    nu: float = 0.3
    Gc: float = 1.0
    ell: float = 0.1
    k_ell: float = 1e-6
    beta: float = 1.0
    model: str = "AT1"            # "AT1" | "AT2"
    regime: str = "plane_stress"  # "plane_stress" | "plane_strain" | "3d"

    @property
    def c_w(self) -> float:
        # c_w = 4 int_0^1 sqrt(w): 8/3 for w = a (model.py:20), 2 for w = a^2
        return 8.0 / 3.0 if self.model == "AT1" else 2.0

    def unit_stiffness(self) -> np.ndarray:
        """Voigt stiffness for E = 1 (model.py:49-55 for plane stress)."""
        nu = self.nu
        if self.regime == "plane_stress":
            return (1.0 / (1.0 - nu * nu)) * np.array(
                [[1.0, nu, 0.0], [nu, 1.0, 0.0], [0.0, 0.0, 0.5 * (1.0 - nu)]])
        if self.regime == "plane_strain":
            s = 1.0 / ((1.0 + nu) * (1.0 - 2.0 * nu))
            return s * np.array([[1.0 - nu, nu, 0.0], [nu, 1.0 - nu, 0.0],
                                 [0.0, 0.0, 0.5 * (1.0 - 2.0 * nu)]])
        if self.regime == "3d":
            lam = nu / ((1.0 + nu) * (1.0 - 2.0 * nu))
            mu = 1.0 / (2.0 * (1.0 + nu))
            D = np.zeros((6, 6))
            D[:3, :3] = lam
            D[:3, :3] += 2.0 * mu * np.eye(3)
            D[3:, 3:] = mu * np.eye(3)
            return D
        raise ValueError(f"unknown regime {self.regime!r}")

    def stiffness(self) -> np.ndarray:
        return self.E * self.unit_stiffness()

    # degradation a(.) and dissipation w(.) with derivatives (model.py:64-76)
    def a_triplet(self, ab):
        om = 1.0 - ab
        return om * om + self.k_ell, -2.0 * om, np.full_like(ab, 2.0)

    def w_triplet(self, ab):
        if self.model == "AT1":
            return ab.copy(), np.ones_like(ab), np.zeros_like(ab)
        return ab * ab, 2.0 * ab, np.full_like(ab, 2.0)


def simplex_gradients(mesh: SimplexMesh):
    """(volumes (T,), gradients (T, d, d+1)) of the P1 basis (fem.py:107-123)."""
    P = mesh.vertices[mesh.elements]
    if mesh.dim == 2:
        p1, p2, p3 = P[:, 0], P[:, 1], P[:, 2]
        det = ((p2[:, 0] - p1[:, 0]) * (p3[:, 1] - p1[:, 1])
               - (p2[:, 1] - p1[:, 1]) * (p3[:, 0] - p1[:, 0]))
        if np.any(det <= 0):
            raise ValueError("mesh contains non-CCW or degenerate triangles")
        bx = np.stack([p2[:, 1] - p3[:, 1], p3[:, 1] - p1[:, 1], p1[:, 1] - p2[:, 1]], axis=1)
        cy = np.stack([p3[:, 0] - p2[:, 0], p1[:, 0] - p3[:, 0], p2[:, 0] - p1[:, 0]], axis=1)
        G = np.stack([bx / det[:, None], cy / det[:, None]], axis=1)
        return 0.5 * det, G
    # 3D: rows of inv(J)^T with J = [p1-p0, p2-p0, p3-p0]
    J = np.stack([P[:, 1] - P[:, 0], P[:, 2] - P[:, 0], P[:, 3] - P[:, 0]], axis=2)  # (T,3,3) cols
    det = np.linalg.det(J)
    if np.any(det <= 0):
        raise ValueError("mesh contains inverted or degenerate tetrahedra")
    Jinv = np.linalg.inv(J)              # (T,3,3): row r = grad of lambda_{r+1}
    G = np.empty((P.shape[0], 3, 4))
    G[:, :, 1:] = np.transpose(Jinv, (0, 2, 1))
    G[:, :, 0] = -G[:, :, 1:].sum(axis=2)
    return det / 6.0, G


def voigt_B(G: np.ndarray) -> np.ndarray:
    """Strain-displacement matrices (fem.py:125-131), interleaved nodal dofs."""
    T, d, n = G.shape
    if d == 2:
        B = np.zeros((T, 3, 2 * n))
        B[:, 0, 0::2] = G[:, 0]
        B[:, 1, 1::2] = G[:, 1]
        B[:, 2, 0::2] = G[:, 1]
        B[:, 2, 1::2] = G[:, 0]
        return B
    B = np.zeros((T, 6, 3 * n))
    gx, gy, gz = G[:, 0], G[:, 1], G[:, 2]
    B[:, 0, 0::3] = gx
    B[:, 1, 1::3] = gy
    B[:, 2, 2::3] = gz
    B[:, 3, 1::3] = gz
    B[:, 3, 2::3] = gy
    B[:, 4, 0::3] = gz
    B[:, 4, 2::3] = gx
    B[:, 5, 0::3] = gy
    B[:, 5, 1::3] = gx
    return B


class P1Model:
    """Element geometry + material, with assembled operators in scipy CSR.

    ``E_elem`` / ``Gc_elem`` are optional per-element absolute values that
    replace the scalar E / Gc of ``spec``.  ``eps0`` (T, nvoigt) and
    ``bc = (dofs, values)`` are mutable per-load-step data, as in the
    reference ``Discretization`` (fem.py:93-105).
    """

    def __init__(self, mesh: SimplexMesh, spec: MaterialSpec,
                 E_elem: Optional[np.ndarray] = None, Gc_elem: Optional[np.ndarray] = None):
        self.mesh = mesh
        self.spec = spec
        self.dim = d = mesh.dim
        self.vol, self.G = simplex_gradients(mesh)
        self.B = voigt_B(self.G)
        self.D1 = spec.unit_stiffness()
        T = mesh.n_elements
        self.Ee = np.full(T, spec.E) if E_elem is None else np.asarray(E_elem, float).copy()
        self.Gce = np.full(T, spec.Gc) if Gc_elem is None else np.asarray(Gc_elem, float).copy()
        self.nvoigt = 3 if d == 2 else 6
        self.npe = d + 1
        self.adofs = mesh.elements
        self.udofs = (d * mesh.elements[:, :, None] + np.arange(d)[None, None, :]).reshape(T, -1)
        self.nv = mesh.n_vertices
        self.nu_dofs = d * self.nv
        self.eps0 = np.zeros((T, self.nvoigt))
        self.bc: Optional[tuple] = None
        self.BtDB = np.einsum("tki,kl,tlj->tij", self.B, self.D1, self.B)
        self.GtG = np.einsum("tki,tkj->tij", self.G, self.G)

    # ---- element kinematics ------------------------------------------------
    def abar(self, alpha):
        return alpha[self.adofs].mean(axis=1)

    def strain(self, u):
        return np.einsum("tij,tj->ti", self.B, u[self.udofs]) - self.eps0

    def stress_unit(self, eps):
        return eps @ self.D1.T

    def _sum_to(self, idx, vals, n):
        return np.bincount(idx.ravel(), weights=vals.ravel(), minlength=n)

    # ---- energy and gradients (fem.py:162-218) -----------------------------
    def energy(self, u, alpha) -> EnergyParts:
        s = self.spec
        ab = self.abar(alpha)
        a = s.a_triplet(ab)[0]
        w = s.w_triplet(ab)[0]
        eps = self.strain(u)
        q = self.Ee * np.einsum("ti,ti->t", eps, self.stress_unit(eps))
        el = 0.5 * float(np.dot(self.vol, a * q))
        g = np.einsum("tij,tj->ti", self.G, alpha[self.adofs])
        dens = (self.Gce / s.c_w) * (w / s.ell + s.ell * np.einsum("ti,ti->t", g, g))
        ds = float(np.dot(self.vol, dens))
        return EnergyParts(el, ds, el + ds)

    def residual_u(self, u, alpha, bc_rows: str = "value"):
        """dE/du; bc_rows: 'value' -> u - ubar (fem.py:177-189), 'zero' (solver.py:108-110), 'none'."""
        a = self.spec.a_triplet(self.abar(alpha))[0]
        sig = self.stress_unit(self.strain(u))
        re = ((a * self.vol * self.Ee)[:, None]) * np.einsum("tki,tk->ti", self.B, sig)
        r = self._sum_to(self.udofs, re, self.nu_dofs)
        if self.bc is not None and bc_rows != "none":
            dofs, vals = self.bc
            r[dofs] = (u[dofs] - vals) if bc_rows == "value" else 0.0
        return r

    def load_u(self, alpha):
        """Inelastic-strain load f with residual_u = K u - f (fem.py:192-199)."""
        a = self.spec.a_triplet(self.abar(alpha))[0]
        sig0 = self.stress_unit(self.eps0)
        fe = ((a * self.vol * self.Ee)[:, None]) * np.einsum("tki,tk->ti", self.B, sig0)
        return self._sum_to(self.udofs, fe, self.nu_dofs)

    def residual_alpha(self, u, alpha):
        """dE/dalpha (fem.py:202-218)."""
        s = self.spec
        ab = self.abar(alpha)
        ap = s.a_triplet(ab)[1]
        wp = s.w_triplet(ab)[1]
        eps = self.strain(u)
        q = self.Ee * np.einsum("ti,ti->t", eps, self.stress_unit(eps))
        kc = self.Gce / s.c_w
        nodal = (0.5 * ap * q + kc * wp / s.ell) * self.vol / self.npe
        r = self._sum_to(self.adofs, np.repeat(nodal[:, None], self.npe, axis=1), self.nv)
        g = np.einsum("tij,tj->ti", self.G, alpha[self.adofs])
        ge = (2.0 * kc * s.ell * self.vol)[:, None] * np.einsum("tij,ti->tj", self.G, g)
        return r + self._sum_to(self.adofs, ge, self.nv)

    # ---- Hessian blocks (fem.py:221-276) ------------------------------------
    def _csr(self, rd, cd, data, shape):
        rows = np.repeat(rd, cd.shape[1], axis=1).ravel()
        cols = np.tile(cd, (1, rd.shape[1])).ravel()
        M = sp.coo_matrix((data.ravel(), (rows, cols)), shape=shape).tocsr()
        M.sum_duplicates()
        M.sort_indices()
        return M

    def Kuu(self, alpha, eliminate: bool = True):
        a = self.spec.a_triplet(self.abar(alpha))[0]
        data = (a * self.vol * self.Ee)[:, None, None] * self.BtDB
        K = self._csr(self.udofs, self.udofs, data, (self.nu_dofs, self.nu_dofs))
        if eliminate and self.bc is not None:
            K = eliminate_rows_cols(K, self.bc[0])
        return K

    def Kua(self, u, alpha, mask_bc: bool = True):
        ap = self.spec.a_triplet(self.abar(alpha))[1]
        sig = self.stress_unit(self.strain(u))
        v = ((ap * self.vol * self.Ee) / self.npe)[:, None] * np.einsum("tki,tk->ti", self.B, sig)
        data = np.repeat(v[:, :, None], self.npe, axis=2)
        K = self._csr(self.udofs, self.adofs, data, (self.nu_dofs, self.nv))
        if mask_bc and self.bc is not None:
            m = np.ones(self.nu_dofs)
            m[self.bc[0]] = 0.0
            K = (sp.diags(m) @ K).tocsr()
            K.eliminate_zeros()
        return K

    def Kaa(self, u, alpha):
        s = self.spec
        ab = self.abar(alpha)
        app = s.a_triplet(ab)[2]
        wpp = s.w_triplet(ab)[2]
        eps = self.strain(u)
        q = self.Ee * np.einsum("ti,ti->t", eps, self.stress_unit(eps))
        kc = self.Gce / s.c_w
        react = (0.5 * app * q + kc * wpp / s.ell) * self.vol / (self.npe * self.npe)
        data = react[:, None, None] * np.ones((1, self.npe, self.npe)) \
            + (2.0 * kc * s.ell * self.vol)[:, None, None] * self.GtG
        return self._csr(self.adofs, self.adofs, data, (self.nv, self.nv))

    def element_energy_density(self, u):
        """q_e = eps^T D_e eps per element (the elastic coupling term)."""
        eps = self.strain(u)
        return self.Ee * np.einsum("ti,ti->t", eps, self.stress_unit(eps))

    # ---- Dirichlet (fem.py:282-310) -----------------------------------------
    def lift(self, K_raw, rhs):
        """Symmetric elimination of K_raw x = rhs with the current bc."""
        if self.bc is None:
            return K_raw, rhs
        dofs, vals = self.bc
        g = np.zeros(K_raw.shape[0])
        g[dofs] = vals
        m = np.ones(K_raw.shape[0])
        m[dofs] = 0.0
        r2 = m * (rhs - K_raw @ g)
        r2[dofs] = vals
        return eliminate_rows_cols(K_raw, dofs), r2


def eliminate_rows_cols(K, dofs):
    """Zero rows and columns ``dofs`` of K and put 1 on their diagonal."""
    n = K.shape[0]
    m = np.ones(n)
    m[dofs] = 0.0
    Dm = sp.diags(m)
    K2 = (Dm @ K @ Dm).tocsr()
    e = np.zeros(n)
    e[dofs] = 1.0
    K2 = (K2 + sp.diags(e)).tocsr()
    K2.eliminate_zeros()
    K2.sort_indices()
    return K2


def merge_bcs(*pairs):
    """Combine (dofs, values) pairs; identical duplicates merge, conflicts raise (fem.py:58-90)."""
    dofs = np.concatenate([np.asarray(p[0], dtype=np.intp) for p in pairs])
    vals = np.concatenate([np.asarray(p[1], dtype=float) for p in pairs])
    order = np.argsort(dofs, kind="stable")
    dofs, vals = dofs[order], vals[order]
    same = dofs[1:] == dofs[:-1]
    if np.any(same & (vals[1:] != vals[:-1])):
        raise ValueError("conflicting Dirichlet values")
    keep = np.concatenate([[True], ~same])
    return dofs[keep], vals[keep]
