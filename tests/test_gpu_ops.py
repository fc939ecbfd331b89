"""GPU parity of every matrix-free operator against the CPU oracle's assembled CSR
(the reference's own assembled-SpMV check, SURVEY 3.5 / BASELINE config 5): relative
max error <= 1e-12 on identical seeded inputs."""

import numpy as np
import pytest
import torch

from gpu_util import make_pair, random_fields, rel

pytestmark = pytest.mark.gpu

CASES = [
    # pattern, regime, model, nx, ny, hetero, eps0
    ("union_jack", "plane_stress", "AT1", 13, 9, False, False),
    ("union_jack", "plane_strain", "AT2", 40, 71, True, True),
    ("right", "plane_stress", "AT1", 20, 7, False, True),
    ("right", "plane_strain", "AT2", 33, 64, True, False),
    ("crossed", "plane_strain", "AT2", 16, 16, False, False),
    ("crossed", "plane_stress", "AT1", 25, 61, True, True),
    ("union_jack", "plane_stress", "AT1", 1, 1, False, False),
    ("crossed", "plane_strain", "AT1", 1, 3, False, False),
    ("right", "plane_stress", "AT2", 70, 2, False, False),
]
TOL = 1e-12


def dev(a):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda")


def host(t):
    return t.cpu().numpy()


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c[0]}-{c[1]}-{c[2]}-{c[3]}x{c[4]}")
def test_operator_parity(case):
    import paper_1511_08463_b200 as pf
    pattern, regime, model, nx, ny, hetero, eps0 = case
    prob, om, rng = make_pair(pattern, regime, model, nx, ny, hetero=hetero, eps0=eps0)
    u, a, lb = random_fields(om, rng)
    xu = rng.standard_normal(om.nu_dofs)
    xa = rng.standard_normal(om.nv)
    st = pf.State(dev(u), dev(a), dev(lb))
    # energies
    e = pf.assemble_energy(st, prob)
    eo = om.energy(u, a)
    assert rel(np.array(e), np.array(eo)) < TOL
    # residuals
    assert rel(host(pf.assemble_residual_u(st, prob, apply_bc=False)), om.residual_u(u, a, "none")) < TOL
    assert rel(host(pf.assemble_residual_u(st, prob, apply_bc=True)), om.residual_u(u, a, "value")) < TOL
    assert rel(host(pf.assemble_residual_alpha(st, prob)), om.residual_alpha(u, a)) < TOL
    f = host(pf.assemble_load_u(st, prob))
    if eps0:
        assert rel(f, om.load_u(a)) < TOL
    else:
        assert np.max(np.abs(f)) == 0.0
    # optimality residual (solver.py:104-118)
    from oracle.am import LoadState, optimality_residual
    fo = optimality_residual(LoadState(u, a, lb), om)
    got = host(pf.first_order_residual(st, prob))
    assert rel(got, fo) < TOL
    assert abs(pf.residual_norm(st, prob) - np.linalg.norm(fo)) <= TOL * np.linalg.norm(fo)
    # Hessian blocks
    Kraw = om.Kuu(a, eliminate=False)
    assert rel(host(pf.assemble_Kuu(st, prob, apply_bc=False) @ dev(xu)), Kraw @ xu) < TOL
    assert rel(host(pf.assemble_Kuu(st, prob, apply_bc=True) @ dev(xu)), om.Kuu(a) @ xu) < TOL
    Kua = pf.assemble_Kua(st, prob, apply_bc=True)
    assert rel(host(Kua @ dev(xa)), om.Kua(u, a) @ xa) < TOL
    assert rel(host(Kua.T @ dev(xu)), om.Kua(u, a).T @ xu) < TOL
    Kua_raw = pf.assemble_Kua(st, prob, apply_bc=False)
    assert rel(host(Kua_raw @ dev(xa)), om.Kua(u, a, mask_bc=False) @ xa) < TOL
    assert rel(host(pf.assemble_Kaa(st, prob) @ dev(xa)), om.Kaa(u, a) @ xa) < TOL


def test_operators_are_deterministic():
    import paper_1511_08463_b200 as pf
    prob, om, rng = make_pair("crossed", "plane_strain", "AT2", 64, 90, hetero=True, eps0=True)
    u, a, lb = random_fields(om, rng)
    st = pf.State(dev(u), dev(a), dev(lb))
    outs = [pf.assemble_energy(st, prob) for _ in range(3)]
    assert outs[0] == outs[1] == outs[2]
    y = [host(pf.assemble_Kuu(st, prob) @ dev(u)) for _ in range(2)]
    assert np.array_equal(y[0], y[1])


@pytest.mark.parametrize("n", [256, 1024])
def test_sweep_sizes_against_assembled_spmv(n):
    """Config-5 style inputs: alpha~U[0,1], u,x~N(0,1), E=1, nu=0.3, k=1e-6, Gc=1, ell=0.1."""
    import paper_1511_08463_b200 as pf
    for pattern in ("union_jack", "crossed"):
        for model in ("AT1", "AT2"):
            prob, om, rng = make_pair(pattern, "plane_stress", model, n, n, lx=1.0, ly=1.0,
                                      bc=False, E=1.0, nu=0.3, Gc=1.0, ell=0.1, seed=1)
            a = rng.uniform(0, 1, om.nv)
            u = rng.standard_normal(om.nu_dofs)
            x = rng.standard_normal(om.nu_dofs)
            xa = rng.standard_normal(om.nv)
            st = pf.State(dev(u), dev(a), dev(np.zeros(om.nv)))
            if model == "AT1":
                assert rel(host(pf.assemble_Kuu(st, prob, apply_bc=False) @ dev(x)),
                           om.Kuu(a, eliminate=False) @ x) < TOL
            assert rel(host(pf.assemble_Kaa(st, prob) @ dev(xa)), om.Kaa(u, a) @ xa) < TOL


def test_operator_only_context_skips_solver_workspaces():
    """solvers='operators' (pf_desc.skip) plans no GMG / Newton workspace and refuses those solves,
    while the operator applies are unchanged."""
    import paper_1511_08463_b200 as pf
    mesh = pf.StructuredMesh(64, 48, 1.0, 0.75, "crossed")
    mat = pf.Material(E=1.0, nu=0.3, Gc=1.0, ell=0.1, k_ell=1e-6)
    full = pf.Discretization(mesh, mat)
    ops = pf.Discretization(mesh, mat, solvers="operators")
    assert ops._ws.numel() < 0.6 * full._ws.numel()
    g = torch.Generator(device="cuda").manual_seed(3)
    a = torch.rand(mesh.n_vertices, dtype=torch.float64, device="cuda", generator=g)
    x = torch.randn(2 * mesh.n_vertices, dtype=torch.float64, device="cuda", generator=g)
    st = pf.State(torch.zeros_like(x), a, torch.zeros_like(a))
    y1 = pf.assemble_Kuu(st, full, apply_bc=False) @ x
    y2 = pf.assemble_Kuu(st, ops, apply_bc=False) @ x
    assert torch.equal(y1, y2)
    with pytest.raises(Exception, match="PF_SKIP_GMG"):
        pf.elastic_step(st, ops, pf.SolverConfig(elastic_solver="cg", elastic_precond="gmg"))
    with pytest.raises(Exception, match="PF_SKIP_NEWTON"):
        pf.coupled_newton_solve(st, ops, pf.SolverConfig())
    us, its = pf.elastic_step(st, ops, pf.SolverConfig(elastic_solver="cg", elastic_precond="jacobi"))
    assert its >= 0
