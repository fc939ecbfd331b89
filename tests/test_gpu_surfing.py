"""Graded (banded) meshes and the surfing benchmark on the device:
operators vs the oracle's assembled matrices (1e-12), the multigrid elastic solve vs LU, and a
12-step surfing run vs the reference's own goldens (tests/golden/ref_surfing.npz)."""

import os

import numpy as np
import pytest
import torch

from conftest import GOLDEN
from gpu_util import rel
from oracle import am as oam
from oracle.meshgen import banded_rows, grid_mesh
from oracle.p1 import MaterialSpec, P1Model

pytestmark = pytest.mark.gpu


def dev(a):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda")


def host(t):
    return t.cpu().numpy()


def graded_pair(pattern, L=1.0, H=0.8, h=0.05, hc=0.2, bw=0.1):
    import paper_1511_08463_b200 as pf
    nx, ys = banded_rows(L, H, h, hc, bw)
    ny = len(ys) - 1
    mat = pf.Material(E=1.3, nu=0.27, Gc=0.9, ell=0.1, k_ell=1e-6)
    spec = MaterialSpec(E=1.3, nu=0.27, Gc=0.9, ell=0.1, k_ell=1e-6)
    mesh = pf.StructuredMesh(nx, ny, L, H, pattern, 0.0, -H / 2, ys=ys)
    prob = pf.Discretization(mesh, mat)
    om = P1Model(grid_mesh(nx, ny, L, H, pattern, 0.0, -H / 2, ys=ys), spec)
    assert np.array_equal(mesh.vertices, om.mesh.vertices)
    return prob, om


@pytest.mark.parametrize("pattern", ["union_jack", "right", "crossed"])
def test_graded_operators_match_oracle(pattern):
    import paper_1511_08463_b200 as pf
    prob, om = graded_pair(pattern)
    rng = np.random.default_rng(11)
    nv = om.nv
    lb = rng.uniform(0, 0.3, nv)
    a = lb + rng.uniform(0, 1, nv) * (1 - lb)
    u = 0.1 * rng.standard_normal(2 * nv)
    xu, xa = rng.standard_normal(2 * nv), rng.standard_normal(nv)
    left = prob.mesh.boundary_vertices("left")
    b = pf.DirichletBC(np.concatenate([2 * left, 2 * left + 1]), np.full(2 * left.size, 0.01))
    prob.bc = b
    om.bc = (b.dofs.astype(np.intp), b.values)
    st = pf.State(dev(u), dev(a), dev(lb))
    assert rel(np.array(pf.assemble_energy(st, prob)), np.array(om.energy(u, a))) < 1e-12
    assert rel(host(pf.assemble_residual_u(st, prob, apply_bc=False)), om.residual_u(u, a, "none")) < 1e-12
    assert rel(host(pf.assemble_residual_alpha(st, prob)), om.residual_alpha(u, a)) < 1e-12
    assert rel(host(pf.assemble_Kuu(st, prob, apply_bc=True) @ dev(xu)), om.Kuu(a) @ xu) < 1e-12
    assert rel(host(pf.assemble_Kaa(st, prob) @ dev(xa)), om.Kaa(u, a) @ xa) < 1e-12
    K = pf.assemble_Kua(st, prob, apply_bc=True)
    assert rel(host(K @ dev(xa)), om.Kua(u, a) @ xa) < 1e-12
    assert rel(host(K.T @ dev(xu)), om.Kua(u, a).T @ xu) < 1e-12


@pytest.mark.parametrize("pattern", ["union_jack", "crossed"])
def test_graded_multigrid_elastic_step_matches_lu(pattern):
    import paper_1511_08463_b200 as pf
    prob, om = graded_pair(pattern)
    rng = np.random.default_rng(5)
    nv = om.nv
    a = rng.uniform(0, 0.9, nv)
    u = 0.05 * rng.standard_normal(2 * nv)
    left, right = prob.mesh.boundary_vertices("left"), prob.mesh.boundary_vertices("right")
    b = pf.combine_bcs(pf.DirichletBC(np.concatenate([2 * left, 2 * left + 1]), np.zeros(2 * left.size)),
                       pf.DirichletBC(2 * right, np.full(right.size, 0.02)))
    prob.bc = b
    om.bc = (b.dofs.astype(np.intp), b.values)
    st = pf.State(dev(u), dev(a), dev(np.zeros(nv)))
    ou, _ = oam.elastic_half_step(oam.LoadState(u, a, np.zeros(nv)), om, oam.AMConfig())
    ug, its = pf.elastic_step(st, prob, pf.SolverConfig(elastic_solver="cg", elastic_precond="gmg",
                                                        elastic_rtol=1e-12, gmg_reuse=False))
    assert rel(host(ug), ou) < 1e-8 and its < 60


def test_surfing_run_matches_reference_goldens():
    """The reference's surfing benchmark (graded band mesh, translated Mode-I boundary field),
    12 AM steps at omega = 1: energies within 1e-6 relative and alpha within 1e-4 of the
    reference itself."""
    import paper_1511_08463_b200 as pf
    g = np.load(os.path.join(GOLDEN, "ref_surfing.npz"))
    setup = pf.setup_surfing(pf.Material(E=1.0, nu=0.3, Gc=1.0, ell=0.2), h=0.05, n_steps=12, t_end=0.9)
    assert np.array_equal(setup.mesh.vertices, g["surf_vertices"])
    cfg = pf.SolverConfig(method="am", omega=1.0, elastic_solver="cg", elastic_precond="gmg",
                          elastic_rtol=1e-12)
    recs = pf.run_quasistatic(setup, cfg)
    E = np.array([list(r.energy) for r in recs])
    assert np.allclose(E, g["surf_energy"], rtol=1e-6, atol=1e-14)
    assert np.max(np.abs(np.stack([r.alpha for r in recs]) - g["surf_alpha"])) < 1e-4
    diss = E[:, 1]
    assert np.all(np.diff(diss) > 0)  # the crack keeps propagating
