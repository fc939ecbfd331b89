"""Material data and damage models (reference model.py:20-111).

Extends the reference's plane-stress AT1 material with the regimes and the AT2
model the BASELINE configs need; the constants are consumed by the device kernels
(through pf_desc), never evaluated per element on the host.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

#: normalisation constant of the linear-dissipation (AT1) model, 4 int_0^1 sqrt(w)
C_W = 8.0 / 3.0
_C_W = {"AT1": 8.0 / 3.0, "AT2": 2.0}
_REGIMES = ("plane_stress", "plane_strain", "3d")


@dataclass(frozen=True)
class Material:
    """Isotropic material with fracture properties (reference model.py:23-61).

    ``regime`` selects plane stress (the reference), plane strain, or 3D.
    """

    E: float = 1.0
    nu: float = 0.3
    Gc: float = 1.0
    ell: float = 0.1
    k_ell: float = 1e-6
    beta: float = 1.0
    regime: str = "plane_stress"

    def __post_init__(self):
        if self.E <= 0 or self.Gc <= 0 or self.ell <= 0:
            raise ValueError("E, Gc and ell must be positive")
        if not -1.0 < self.nu < 0.5:
            raise ValueError(f"nu={self.nu} out of the admissible range (-1, 0.5)")
        if self.regime not in _REGIMES:
            raise ValueError(f"unknown regime {self.regime!r}; choose from {_REGIMES}")

    @property
    def mu(self) -> float:
        return self.E / (2.0 * (1.0 + self.nu))

    def stiffness_matrix(self):
        """Voigt stiffness (plane stress: model.py:49-55)."""
        import numpy as np
        E, nu = self.E, self.nu
        if self.regime == "plane_stress":
            c = E / (1.0 - nu * nu)
            return c * np.array([[1.0, nu, 0.0], [nu, 1.0, 0.0], [0.0, 0.0, 0.5 * (1.0 - nu)]])
        if self.regime == "plane_strain":
            c = E / ((1.0 + nu) * (1.0 - 2.0 * nu))
            return c * np.array([[1.0 - nu, nu, 0.0], [nu, 1.0 - nu, 0.0],
                                 [0.0, 0.0, 0.5 * (1.0 - 2.0 * nu)]])
        lam = E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu))
        D = np.zeros((6, 6))
        D[:3, :3] = lam
        D[:3, :3] += 2.0 * self.mu * np.eye(3)
        D[3:, 3:] = self.mu * np.eye(3)
        return D


class DamageModel:
    """The (w, a) pair: AT1 (reference model.py:64-76) or AT2 (w = alpha^2)."""

    def __init__(self, kind: str = "AT1"):
        if kind not in _C_W:
            raise ValueError(f"unknown damage model {kind!r}; choose AT1 or AT2")
        self.kind = kind

    @property
    def c_w(self) -> float:
        return _C_W[self.kind]

    def a_eval(self, alpha, k_ell: float = 1e-6):
        one_m = 1.0 - alpha
        return one_m * one_m + k_ell, -2.0 * one_m, 2.0 + 0.0 * alpha

    def w_eval(self, alpha):
        if self.kind == "AT1":
            return alpha, 1.0 + 0.0 * alpha, 0.0 * alpha
        return alpha * alpha, 2.0 * alpha, 2.0 + 0.0 * alpha


def critical_traction(material: Material, damage: DamageModel | None = None) -> float:
    """AT1 homogeneous damage-onset strain sqrt(3 Gc / (8 E ell)) (model.py:84-91)."""
    m = material
    return math.sqrt(3.0 * m.Gc / (8.0 * m.E * m.ell))


def critical_shock(material: Material) -> float:
    """Shock amplitude below which an isotropic shock stays elastic (AT1).

    Plane stress: the reference's sqrt(3 Gc/(8 E ell))/beta (model.py:94-104).
    Plane strain (laterally constrained, traction-free face): surface stress
    E dT/(1-nu^2), hence dT_c = sqrt(3 Gc (1-nu^2)/(8 E ell))/beta.
    """
    m = material
    if m.beta <= 0:
        raise ValueError("beta must be positive for a thermal shock threshold")
    f = (1.0 - m.nu ** 2) if m.regime == "plane_strain" else 1.0
    return math.sqrt(3.0 * m.Gc * f / (8.0 * m.E * m.ell)) / m.beta


def internal_length(Gc: float, E: float, sigma_c: float) -> float:
    """(3/8) Gc E / sigma_c^2 (model.py:107-111)."""
    if sigma_c <= 0:
        raise ValueError("sigma_c must be positive")
    return 0.375 * Gc * E / (sigma_c * sigma_c)
