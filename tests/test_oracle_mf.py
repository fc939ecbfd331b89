"""The matrix-free C oracle (oracle/mfapply.c) against the assembled oracle SpMV (oracle/p1.py,
itself pinned to the reference by tests/test_oracle_golden.py): the config-5 checker for the sizes
the assembled matrix cannot reach."""

import numpy as np
import pytest

from oracle import mfapply
from oracle.meshgen import grid_mesh, kuhn_mesh
from oracle.p1 import MaterialSpec, P1Model


def rel(a, b):
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


@pytest.mark.parametrize("pattern", ["union_jack", "right", "crossed"])
@pytest.mark.parametrize("regime,model", [("plane_stress", "AT1"), ("plane_strain", "AT2")])
@pytest.mark.parametrize("shape", [(13, 9), (1, 1), (1, 3), (8, 8)])
def test_mf_2d_matches_assembled(pattern, regime, model, shape):
    nx, ny = shape
    lx, ly = 1.3, 0.7
    spec = MaterialSpec(E=1.7, nu=0.3, Gc=1.3, ell=0.1, k_ell=1e-6, model=model, regime=regime)
    om = P1Model(grid_mesh(nx, ny, lx, ly, pattern), spec)
    rng = np.random.default_rng(nx * 7 + ny)
    a = rng.uniform(0, 1, om.nv)
    u = rng.standard_normal(om.nu_dofs)
    x = rng.standard_normal(om.nu_dofs)
    xa = rng.standard_normal(om.nv)
    for threads in (1, 3):
        y = mfapply.apply("Kuu", (nx, ny), (lx, ly), pattern, spec, alpha=a, x=x, threads=threads)
        assert rel(y, om.Kuu(a, eliminate=False) @ x) < 1e-13
        y = mfapply.apply("Kaa", (nx, ny), (lx, ly), pattern, spec, alpha=a, u=u, x=xa, threads=threads)
        assert rel(y, om.Kaa(u, a) @ xa) < 1e-13


@pytest.mark.parametrize("model", ["AT1", "AT2"])
@pytest.mark.parametrize("shape", [(3, 4, 5), (1, 1, 1), (2, 1, 6)])
def test_mf_3d_matches_assembled(model, shape):
    nx, ny, nz = shape
    spec = MaterialSpec(E=1.0, nu=0.3, Gc=1.0, ell=0.1, k_ell=1e-6, model=model, regime="3d")
    om = P1Model(kuhn_mesh(nx, ny, nz, 1.0, 0.8, 1.2), spec)
    rng = np.random.default_rng(nx + 10 * ny + 100 * nz)
    a = rng.uniform(0, 1, om.nv)
    u = rng.standard_normal(om.nu_dofs)
    x = rng.standard_normal(om.nu_dofs)
    xa = rng.standard_normal(om.nv)
    y = mfapply.apply("Kuu", shape, (1.0, 0.8, 1.2), "kuhn6", spec, alpha=a, x=x, threads=2)
    assert rel(y, om.Kuu(a, eliminate=False) @ x) < 1e-13
    y = mfapply.apply("Kaa", shape, (1.0, 0.8, 1.2), "kuhn6", spec, alpha=a, u=u, x=xa, threads=2)
    assert rel(y, om.Kaa(u, a) @ xa) < 1e-13


def test_mf_matches_assembled_at_config5_size():
    """Overlap with the assembled check at a config-5 size (256^2 union-jack, seeded as bench)."""
    n = 256
    spec = MaterialSpec(E=1.0, nu=0.3, Gc=1.0, ell=0.1, k_ell=1e-6, model="AT2")
    om = P1Model(grid_mesh(n, n, 1.0, 1.0, "union_jack"), spec)
    rng = np.random.default_rng(5)
    a = rng.uniform(0, 1, om.nv)
    x = rng.standard_normal(om.nu_dofs)
    u = rng.standard_normal(om.nu_dofs)
    xa = rng.standard_normal(om.nv)
    assert rel(mfapply.apply("Kuu", (n, n), (1.0, 1.0), "union_jack", spec, alpha=a, x=x),
               om.Kuu(a, eliminate=False) @ x) < 1e-13
    assert rel(mfapply.apply("Kaa", (n, n), (1.0, 1.0), "union_jack", spec, u=u, x=xa),
               om.Kaa(u, a) @ xa) < 1e-13
