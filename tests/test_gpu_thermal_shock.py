"""The reference's own thermal-shock case (cases.py:195-235) on the element-list path, against the
golden trajectory the reference itself produced (tests/golden/make_thermal_shock_golden.py):
the jittered 80 x 40 union-jack rect_mesh (reproduced bit for bit), the erfc inelastic strain at
the element centroids, 12 geometric tau steps at dT = 2 dT_c while the periodic crack pattern
forms, alternate minimisation (method am) at outer_atol 1e-8.  North-star bars at every step:
energies within 1e-6 relative, alpha within 1e-4 (the jitter breaks every symmetry).  Also the
INI front end: ``[case] name = thermal_shock`` now runs (runio.py) and writes its artifacts."""

import os

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu


def test_thermal_shock_matches_reference_trajectory():
    import paper_1511_08463_b200 as pf
    g = np.load(os.path.join(GOLDEN, "ref_thermal_shock.npz"))
    setup = pf.setup_thermal_shock(n_steps=int(g["steps"]), dT_factor=float(g["dT_factor"]))
    assert np.array_equal(setup.mesh.vertices, g["vertices"])  # the reference's jittered mesh
    cfg = pf.SolverConfig(method="am", outer_atol=float(g["atol"]))
    recs = pf.run_quasistatic(setup, cfg)
    E = np.array([tuple(r.energy) for r in recs])
    Eo = g["energy"]
    assert Eo[-1, 1] > 0.5 * Eo[-1, 2]  # the crack pattern formed inside the schedule
    for k in range(E.shape[0]):
        for q in range(3):
            if Eo[k, q] == 0.0:
                assert abs(E[k, q]) <= 1e-12
            else:
                assert abs(E[k, q] - Eo[k, q]) <= 1e-6 * abs(Eo[k, q]), f"step {k} energy {q}"
        assert np.max(np.abs(recs[k].alpha - g["alpha"][k])) <= 1e-4, f"step {k} alpha"


def test_thermal_shock_with_the_structured_twin_multigrid():
    """The elastic half-steps by PCG on the jittered mesh's Kuu with the V-cycle of the un-jittered
    twin as preconditioner (pf_gmg_prepare / pf_gmg_apply): the same trajectory as the reference to
    the north-star bars (first 9 steps, up to the onset of the crack pattern), with a small fraction of
    the Krylov iterations of the Jacobi-PCG run."""
    import paper_1511_08463_b200 as pf
    g = np.load(os.path.join(GOLDEN, "ref_thermal_shock.npz"))
    n = 9
    its = {}
    for mg in (False, True):
        setup = pf.setup_thermal_shock(n_steps=int(g["steps"]), dT_factor=float(g["dT_factor"]), multigrid=mg)
        cfg = pf.SolverConfig(method="am", outer_atol=float(g["atol"]), elastic_precond="gmg" if mg else "jacobi")
        recs = pf.run_quasistatic(setup, cfg, steps=list(range(n)))
        its[mg] = sum(r.report.total_krylov_iterations for r in recs)
        for k, r in enumerate(recs):
            for q in range(3):
                ref = g["energy"][k, q]
                assert abs(tuple(r.energy)[q] - ref) <= 1e-6 * abs(ref) + 1e-12, f"mg={mg} step {k} energy {q}"
            assert np.max(np.abs(r.alpha - g["alpha"][k])) <= 1e-4, f"mg={mg} step {k} alpha"
    assert its[True] < 0.2 * its[False], its


def test_umesh_elastic_solve_gmg_equals_jacobi():
    """One elastic solve on a cracked jittered mesh: both preconditioners reach the same solution."""
    import torch
    import paper_1511_08463_b200 as pf
    setup = pf.setup_thermal_shock(n_steps=4, L=16.0, H=8.0, multigrid=True)
    ops, mesh = setup.ops, setup.mesh
    dofs, vals = setup.apply_load(ops, float(setup.schedule[2]))
    ops.set_dirichlet(np.asarray(dofs, dtype=np.int64))
    rng = np.random.default_rng(0)
    V = mesh.n_vertices
    a = rng.uniform(0.0, 0.3, V)
    a[np.abs(mesh.vertices[:, 0] - 8.0) < 0.4] = 1.0  # a crack band
    alpha = torch.as_tensor(a, device="cuda")
    b = torch.as_tensor(rng.standard_normal(2 * V), device="cuda")
    b[torch.as_tensor(dofs, device="cuda")] = 0.0
    xj, rj = ops.elastic_solve(alpha, b, rtol=1e-11)
    xg, rg = ops.elastic_solve(alpha, b, rtol=1e-11, precond="gmg")
    assert rj.converged and rg.converged
    assert float((xj - xg).abs().max() / xj.abs().max()) < 1e-7
    assert rg.iterations < 0.2 * rj.iterations, (rg.iterations, rj.iterations)


def test_thermal_shock_ini_runs_on_the_device(tmp_path):
    from paper_1511_08463_b200 import runio
    cfg = runio.parse_config("[case]\nname = thermal_shock\nn_steps = 4\nL = 8.0\nH = 4.0\n"
                             "[solver]\nmethod = oram\nomega = 1.4\n")
    rc = runio.run(cfg, output_dir=str(tmp_path))
    assert rc == 0
    assert (tmp_path / "energies.csv").exists() and (tmp_path / "iterations.csv").exists()
    assert sorted(p.name for p in tmp_path.glob("step_*.vtk"))
    text = (tmp_path / "iterations.csv").read_text().splitlines()
    assert len(text) > 4
