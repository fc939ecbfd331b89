"""Pin the oracle's extensions (AT2, plane strain, right/crossed, 3D Kuhn, per-element
E/Gc) by finite-difference consistency and closed forms -- the same oracle
pattern as the reference's tests/conftest.py:20-43 and test_fem.py:33-98,167-218.
CPU only."""

import numpy as np
import pytest

from oracle.meshgen import grid_mesh, kuhn_mesh
from oracle.p1 import MaterialSpec, P1Model


def fd_grad(f, x, h=1e-6):
    g = np.zeros_like(x)
    for i in range(x.size):
        s = h * (1.0 + abs(x[i]))
        xp, xm = x.copy(), x.copy()
        xp[i] += s
        xm[i] -= s
        g[i] = (f(xp) - f(xm)) / (2 * s)
    return g


def fd_jac(F, x, h=1e-6):
    cols = []
    for i in range(x.size):
        s = h * (1.0 + abs(x[i]))
        xp, xm = x.copy(), x.copy()
        xp[i] += s
        xm[i] -= s
        cols.append((F(xp) - F(xm)) / (2 * s))
    return np.column_stack(cols)


CASES = [
    ("union_jack", "AT1", "plane_stress"),
    ("right", "AT2", "plane_strain"),
    ("crossed", "AT1", "plane_strain"),
    ("crossed", "AT2", "plane_stress"),
    ("kuhn6", "AT1", "3d"),
    ("kuhn6", "AT2", "3d"),
]


def build(pattern, model, regime, hetero=True, seed=0):
    rng = np.random.default_rng(seed)
    spec = MaterialSpec(E=1.3, nu=0.27, Gc=0.9, ell=0.2, k_ell=1e-6, model=model, regime=regime)
    mesh = kuhn_mesh(2, 2, 2, 1.0, 0.8, 0.9) if pattern == "kuhn6" else \
        grid_mesh(3, 2, 1.0, 0.7, pattern)
    T = mesh.n_elements
    E = 1.3 * (1 + 0.1 * rng.uniform(-1, 1, T)) if hetero else None
    G = 0.9 * np.exp(0.1 * rng.standard_normal(T)) if hetero else None
    m = P1Model(mesh, spec, E_elem=E, Gc_elem=G)
    m.eps0 = 0.02 * rng.standard_normal(m.eps0.shape)
    u = 0.1 * rng.standard_normal(m.nu_dofs)
    a = rng.uniform(0.05, 0.9, m.nv)
    return m, u, a


@pytest.mark.parametrize("case", CASES)
def test_residuals_are_energy_gradients(case):
    m, u, a = build(*case)
    gu = fd_grad(lambda x: m.energy(x, a).total, u)
    ga = fd_grad(lambda x: m.energy(u, x).total, a)
    assert np.allclose(m.residual_u(u, a, "none"), gu, rtol=1e-5, atol=1e-8)
    assert np.allclose(m.residual_alpha(u, a), ga, rtol=1e-5, atol=1e-8)


@pytest.mark.parametrize("case", CASES)
def test_hessian_blocks_are_jacobians(case):
    m, u, a = build(*case)
    Juu = fd_jac(lambda x: m.residual_u(x, a, "none"), u)
    Jua = fd_jac(lambda x: m.residual_u(u, x, "none"), a)
    Jaa = fd_jac(lambda x: m.residual_alpha(u, x), a)
    assert np.allclose(m.Kuu(a, eliminate=False).toarray(), Juu, rtol=1e-5, atol=1e-7)
    assert np.allclose(m.Kua(u, a, mask_bc=False).toarray(), Jua, rtol=1e-5, atol=1e-7)
    assert np.allclose(m.Kaa(u, a).toarray(), Jaa, rtol=1e-5, atol=1e-7)


@pytest.mark.parametrize("case", CASES)
def test_load_vector_identity(case):
    """residual_u(u) = K u - f (reference test_fem.py:121-129)."""
    m, u, a = build(*case)
    r = m.residual_u(u, a, "none")
    assert np.allclose(r, m.Kuu(a, eliminate=False) @ u - m.load_u(a), rtol=0, atol=1e-12)


@pytest.mark.parametrize("pattern", ["union_jack", "right", "crossed", "kuhn6"])
@pytest.mark.parametrize("model", ["AT1", "AT2"])
def test_fully_damaged_energy_closed_form(pattern, model):
    regime = "3d" if pattern == "kuhn6" else "plane_stress"
    spec = MaterialSpec(Gc=1.7, ell=0.3, model=model, regime=regime)
    mesh = kuhn_mesh(2, 3, 2, 1.0, 1.5, 1.0) if pattern == "kuhn6" else \
        grid_mesh(4, 3, 2.0, 1.5, pattern)
    m = P1Model(mesh, spec)
    vol = 1.5 if pattern == "kuhn6" else 3.0
    e = m.energy(np.zeros(m.nu_dofs), np.ones(m.nv))
    assert e.elastic == 0.0
    assert np.isclose(e.dissipated, spec.Gc / spec.c_w / spec.ell * vol, rtol=1e-13)


@pytest.mark.parametrize("pattern", ["union_jack", "right", "crossed"])
@pytest.mark.parametrize("regime", ["plane_stress", "plane_strain"])
def test_uniform_strain_energy(pattern, regime):
    spec = MaterialSpec(E=2.0, nu=0.25, regime=regime, k_ell=1e-6)
    mesh = grid_mesh(5, 3, 1.0, 0.6, pattern)
    m = P1Model(mesh, spec)
    eps = np.array([0.01, -0.004, 0.006])
    v = mesh.vertices
    u = np.empty(m.nu_dofs)
    u[0::2] = eps[0] * v[:, 0] + 0.5 * eps[2] * v[:, 1]
    u[1::2] = eps[1] * v[:, 1] + 0.5 * eps[2] * v[:, 0]
    D = spec.stiffness()
    expect = 0.5 * (1 + 1e-6) * eps @ D @ eps * 0.6
    assert np.isclose(m.energy(u, np.zeros(m.nv)).elastic, expect, rtol=1e-12)


def test_3d_uniform_strain_energy():
    spec = MaterialSpec(E=1.0, nu=0.3, regime="3d")
    mesh = kuhn_mesh(2, 3, 2, 1.0, 1.5, 1.0)
    m = P1Model(mesh, spec)
    v = mesh.vertices
    g = np.array([[0.01, 0.002, -0.003], [0.0, -0.004, 0.001], [0.005, 0.0, 0.002]])
    u = (v @ g.T).ravel()
    e = 0.5 * (g + g.T)
    voigt = np.array([e[0, 0], e[1, 1], e[2, 2], 2 * e[1, 2], 2 * e[0, 2], 2 * e[0, 1]])
    expect = 0.5 * (1 + 1e-6) * voigt @ spec.stiffness() @ voigt * 1.5
    assert np.isclose(m.energy(u, np.zeros(m.nv)).elastic, expect, rtol=1e-12)


def test_mesh_counts():
    for pat, nvx in (("union_jack", 0), ("right", 0), ("crossed", 1)):
        m = grid_mesh(8, 5, 1.0, 1.0, pat)
        assert m.n_vertices == 9 * 6 + nvx * 40
        assert m.n_elements == (4 if pat == "crossed" else 2) * 40
    k = kuhn_mesh(3, 2, 4)
    assert k.n_vertices == 4 * 3 * 5 and k.n_elements == 6 * 24
