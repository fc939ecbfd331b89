"""3D (Kuhn tetrahedra, BASELINE config 4 / config-5 3D sweep) GPU parity against the CPU oracle:
operators vs the assembled CSR at 1e-12; half-steps and coupled Newton vs the oracle solvers."""

import numpy as np
import pytest
import torch

from gpu_util import rel
from oracle import am as oam
from oracle.meshgen import kuhn_mesh
from oracle.p1 import MaterialSpec, P1Model

pytestmark = pytest.mark.gpu
TOL = 1e-12


def dev(a):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda")


def host(t):
    return t.cpu().numpy()


def make3(nx, ny, nz, model="AT1", hetero=True, bc=True, seed=0, E=1.3, nu=0.27, Gc=0.9, ell=0.2):
    import paper_1511_08463_b200 as pf
    rng = np.random.default_rng(seed)
    lx, ly, lz = 1.0, 0.8 * ny / nx, 0.9 * nz / nx
    mat = pf.Material(E=E, nu=nu, Gc=Gc, ell=ell, k_ell=1e-6, regime="3d")
    spec = MaterialSpec(E=E, nu=nu, Gc=Gc, ell=ell, k_ell=1e-6, model=model, regime="3d")
    mesh = pf.StructuredMesh3D(nx, ny, nz, lx, ly, lz)
    ncell = nx * ny * nz
    Ec = E * (1 + 0.2 * rng.uniform(-1, 1, ncell)) if hetero else None
    Gcc = Gc * np.exp(0.2 * rng.standard_normal(ncell)) if hetero else None
    prob = pf.Discretization(mesh, mat, pf.DamageModel(model), E_cell=Ec, Gc_cell=Gcc)
    om_mesh = kuhn_mesh(nx, ny, nz, lx, ly, lz)
    cell = om_mesh.element_cell()
    om = P1Model(om_mesh, spec, E_elem=None if Ec is None else Ec[cell],
                 Gc_elem=None if Gcc is None else Gcc[cell])
    if bc:
        z0 = om_mesh.boundary["z0"]
        z1 = om_mesh.boundary["z1"]
        x1 = om_mesh.boundary["x1"]
        dofs = np.concatenate([3 * z0, 3 * z0 + 1, 3 * z0 + 2, 3 * z1 + 2, 3 * x1])
        vals = np.concatenate([np.zeros(3 * z0.size), np.full(z1.size, 0.05), np.zeros(x1.size)])
        b = pf.DirichletBC(dofs, vals)
        prob.bc = b
        om.bc = (b.dofs.astype(np.intp), b.values)
    return prob, om, rng


SHAPES = [(3, 4, 5), (20, 33, 31), (1, 1, 1), (17, 2, 40)]


@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: "x".join(map(str, s)))
@pytest.mark.parametrize("model", ["AT1", "AT2"])
def test_operator_parity_3d(shape, model):
    import paper_1511_08463_b200 as pf
    prob, om, rng = make3(*shape, model=model)
    nv = om.nv
    lb = rng.uniform(0, 0.3, nv)
    a = lb + rng.uniform(0, 1, nv) * (1 - lb)
    u = 0.1 * rng.standard_normal(3 * nv)
    xu = rng.standard_normal(3 * nv)
    xa = rng.standard_normal(nv)
    st = pf.State(dev(u), dev(a), dev(lb))
    assert rel(np.array(pf.assemble_energy(st, prob)), np.array(om.energy(u, a))) < TOL
    assert rel(host(pf.assemble_residual_u(st, prob, apply_bc=False)), om.residual_u(u, a, "none")) < TOL
    assert rel(host(pf.assemble_residual_u(st, prob, apply_bc=True)), om.residual_u(u, a, "value")) < TOL
    assert rel(host(pf.assemble_residual_alpha(st, prob)), om.residual_alpha(u, a)) < TOL
    fo = oam.optimality_residual(oam.LoadState(u, a, lb), om)
    assert rel(host(pf.first_order_residual(st, prob)), fo) < TOL
    assert rel(host(pf.assemble_Kuu(st, prob, apply_bc=False) @ dev(xu)), om.Kuu(a, eliminate=False) @ xu) < TOL
    assert rel(host(pf.assemble_Kuu(st, prob, apply_bc=True) @ dev(xu)), om.Kuu(a) @ xu) < TOL
    K = pf.assemble_Kua(st, prob, apply_bc=True)
    assert rel(host(K @ dev(xa)), om.Kua(u, a) @ xa) < TOL
    assert rel(host(K.T @ dev(xu)), om.Kua(u, a).T @ xu) < TOL
    assert rel(host(pf.assemble_Kaa(st, prob) @ dev(xa)), om.Kaa(u, a) @ xa) < TOL


def test_elastic_and_damage_steps_3d():
    import paper_1511_08463_b200 as pf
    prob, om, rng = make3(6, 5, 7, model="AT1")
    nv = om.nv
    lb = rng.uniform(0, 0.3, nv)
    a = lb + rng.uniform(0, 1, nv) * (1 - lb)
    u = 0.3 * rng.standard_normal(3 * nv)
    st = pf.State(dev(u), dev(a), dev(lb))
    us, kit = pf.elastic_step(st, prob, pf.SolverConfig(elastic_solver="cg", elastic_rtol=1e-13))
    ou, _ = oam.elastic_half_step(oam.LoadState(u, a, lb), om, oam.AMConfig())
    assert kit > 0 and rel(host(us), ou) < 1e-9
    ad, rep = pf.damage_step(st, prob, pf.SolverConfig(outer_atol=1e-9))
    ao, orep = oam.damage_half_step(oam.LoadState(u, a, lb), om, oam.AMConfig(outer_atol=1e-9))
    assert rep.converged and orep.converged
    assert np.max(np.abs(host(ad) - ao)) < 1e-9


def test_traction3d_config4_shape_run_matches_oracle():
    """Config-4 physics (lognormal Gc, clamped z=0, pulled z=1, ORAM-N) on a coarse cube."""
    import paper_1511_08463_b200 as pf
    from oracle import problems as opb
    n, steps = 6, 6
    setup = pf.setup_traction3d(n=n, n_steps=steps, material=pf.Material(E=1.0, nu=0.3, Gc=1.0, ell=0.3,
                                                                         k_ell=1e-6, regime="3d"))
    spec = MaterialSpec(E=1.0, nu=0.3, Gc=1.0, ell=0.3, k_ell=1e-6, model="AT1", regime="3d")
    osetup = opb.traction3d(n=n, spec=spec, n_steps=steps)
    assert np.allclose(setup.params["Gc_cell"], osetup.params["Gc_cell"], rtol=0, atol=0)
    cfg = pf.SolverConfig(method="oram_newton", omega=1.7, outer_atol=1e-9, elastic_solver="cg",
                          elastic_rtol=1e-12)
    recs = pf.run_quasistatic(setup, cfg)
    orows, _ = opb.run(osetup, oam.AMConfig(method="oram_newton", omega=1.7, outer_atol=1e-9))
    assert max(float(np.max(o.alpha)) for o in orows) > 0.05   # damage does develop
    for r, o in zip(recs, orows):
        for k in range(3):
            assert abs(r.energy[k] - o.energy[k]) <= 1e-6 * abs(o.energy[k]) + 1e-14, (r.step, k)
        assert np.max(np.abs(r.alpha - o.alpha)) < 1e-4


@pytest.mark.parametrize("shape", [(12, 10, 14), (7, 5, 9), (16, 16, 16)], ids=lambda s: "x".join(map(str, s)))
def test_gmg3_elastic_step_matches_oracle(shape):
    """3D multigrid-PCG (pf_gmg3.cu) converges to the oracle's direct elastic solution, in fewer
    iterations than Jacobi-PCG; odd sizes exercise the ceil-rule coarsening."""
    import paper_1511_08463_b200 as pf
    prob, om, rng = make3(*shape, model="AT1")
    nv = om.nv
    lb = rng.uniform(0, 0.3, nv)
    a = lb + rng.uniform(0, 1, nv) * (1 - lb)
    a[rng.uniform(size=nv) < 0.05] = 1.0  # crack-like spots: a = k_ell there
    u = 0.3 * rng.standard_normal(3 * nv)
    st = pf.State(dev(u), dev(a), dev(lb))
    ou, _ = oam.elastic_half_step(oam.LoadState(u, a, lb), om, oam.AMConfig())
    ug, kg = pf.elastic_step(st, prob, pf.SolverConfig(elastic_solver="cg", elastic_rtol=1e-12,
                                                       elastic_precond="gmg", gmg_reuse=False))
    uj, kj = pf.elastic_step(st, prob, pf.SolverConfig(elastic_solver="cg", elastic_rtol=1e-12,
                                                       elastic_precond="jacobi"))
    assert rel(host(ug), ou) < 1e-8 and rel(host(uj), ou) < 1e-8
    assert kg < kj, (kg, kj)


@pytest.mark.parametrize("inner", ["direct", "mg"])
def test_traction3d_config4_shape_gmg_matches_oracle(inner):
    """Config-4 physics through the 3D multigrid path (elastic half-steps and Newton's A block;
    inner="mg": the A block preconditioned by one 3D V-cycle, C by Chebyshev-Jacobi)."""
    import paper_1511_08463_b200 as pf
    from oracle import problems as opb
    n, steps = 8, 6
    mat = pf.Material(E=1.0, nu=0.3, Gc=1.0, ell=0.3, k_ell=1e-6, regime="3d")
    setup = pf.setup_traction3d(n=n, n_steps=steps, material=mat)
    spec = MaterialSpec(E=1.0, nu=0.3, Gc=1.0, ell=0.3, k_ell=1e-6, model="AT1", regime="3d")
    osetup = opb.traction3d(n=n, spec=spec, n_steps=steps)
    cfg = pf.SolverConfig(method="oram_newton", omega=1.7, outer_atol=1e-9, elastic_solver="cg",
                          elastic_rtol=1e-12, elastic_precond="gmg", fieldsplit_inner=inner)
    recs = pf.run_quasistatic(setup, cfg)
    orows, _ = opb.run(osetup, oam.AMConfig(method="oram_newton", omega=1.7, outer_atol=1e-9))
    assert max(float(np.max(o.alpha)) for o in orows) > 0.05
    for r, o in zip(recs, orows):
        for k in range(3):
            assert abs(r.energy[k] - o.energy[k]) <= 1e-6 * abs(o.energy[k]) + 1e-14, (r.step, k)
        assert np.max(np.abs(r.alpha - o.alpha)) < 1e-4


_FUSED_SNIPPET = r"""
import sys, numpy as np
sys.path.insert(0, "tests")
from test_gpu_ops3d import make3, dev, host
import paper_1511_08463_b200 as pf
prob, om, rng = make3(19, 13, 22, model="AT1")
nv = om.nv
lb = rng.uniform(0, 0.3, nv)
a = lb + rng.uniform(0, 1, nv) * (1 - lb)
a[rng.uniform(size=nv) < 0.05] = 1.0
u = 0.3 * rng.standard_normal(3 * nv)
st = pf.State(dev(u), dev(a), dev(lb))
ug, kg = pf.elastic_step(st, prob, pf.SolverConfig(elastic_solver="cg", elastic_rtol=1e-12,
                                                   elastic_precond="gmg", gmg_reuse=False))
np.save(sys.argv[1], host(ug))
print(kg)
"""


@pytest.mark.parametrize("degree", [2, 3])
def test_gmg3_fused_smoother_matches_separate_passes(tmp_path, degree):
    """The 3D V-cycle with the smoother steps fused into the Kuu apply (Op3KuuSm) against the same
    cycle with one vector pass per step (PF_GMG3_UNFUSED=1): same PCG iterations, same solution."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    snippet = _FUSED_SNIPPET.replace('elastic_precond="gmg"', f'elastic_precond="gmg", gmg_degree={degree}')
    out = {}
    for tag, extra in (("fused", {}), ("split", {"PF_GMG3_UNFUSED": "1"})):
        env = dict(os.environ, **extra)
        f = tmp_path / f"{tag}.npy"
        r = subprocess.run([sys.executable, "-c", snippet, str(f)], cwd=root, env=env, capture_output=True,
                           text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        out[tag] = (int(r.stdout.split()[-1]), np.load(f))
    assert abs(out["fused"][0] - out["split"][0]) <= 1, (out["fused"][0], out["split"][0])
    assert rel(out["fused"][1], out["split"][1]) < 1e-10


@pytest.mark.parametrize("model", ["AT1", "AT2"])
def test_persistent_damage_pcg_3d_matches_graph_loop(monkeypatch, model):
    """The 3D damage Jacobi-PCG in one cooperative launch (k_pcg_kaa3, tiles distributed over the
    resident CTAs) against the graph-replayed two-launch loop (PF_PCG_GRAPH=1): same VI iterations,
    Krylov counts within one per VI iteration, same damage field."""
    import paper_1511_08463_b200 as pf
    out = {}
    for graph in (False, True):
        if graph:
            monkeypatch.setenv("PF_PCG_GRAPH", "1")
        else:
            monkeypatch.delenv("PF_PCG_GRAPH", raising=False)
        prob, om, rng = make3(23, 9, 31, model=model)
        nv = om.nv
        lb = rng.uniform(0, 0.3, nv)
        a = lb + rng.uniform(0, 1, nv) * (1 - lb)
        u = 0.5 * rng.standard_normal(3 * nv)
        st = pf.State(dev(u), dev(a), dev(lb))
        out[graph] = pf.damage_step(st, prob, pf.SolverConfig(outer_atol=1e-9))
    (a0, r0), (a1, r1) = out[False], out[True]
    assert r0.converged and r1.converged
    assert r0.iterations == r1.iterations
    assert abs(r0.total_krylov_iterations - r1.total_krylov_iterations) <= r0.iterations
    assert float((a0 - a1).abs().max()) < 1e-9


def test_damage_step_3d_with_a_localised_free_set(monkeypatch, capfd):
    """As the 2D test of the same name (test_gpu_solvers.py): the persistent 3D damage PCG on the
    list of tiles that hold free vertices (k_tile_flags3), against the oracle."""
    import re
    import paper_1511_08463_b200 as pf
    monkeypatch.setenv("PF_TILE_TRACE", "1")
    prob, om, rng = make3(30, 20, 70, model="AT1", ell=0.08)
    x = om.mesh.vertices
    c = np.array([0.55, 0.3, 1.5])
    d2 = ((x - c) ** 2).sum(axis=1)
    u = np.zeros(3 * om.nv)
    for k in range(3):
        u[k::3] = (3.5 - 0.2 * k) * np.exp(-d2 / 0.02) * (x[:, k] - c[k])
    lb = np.where(d2 < 0.005, 0.2, 0.0)
    a = lb.copy()
    st = pf.State(dev(u), dev(a), dev(lb))
    ad, rep = pf.damage_step(st, prob, pf.SolverConfig(outer_atol=1e-9))
    counts = [(int(p), int(q)) for p, q in re.findall(r"damage pcg: (\d+) of (\d+) tiles", capfd.readouterr().err)]
    ao, orep = oam.damage_half_step(oam.LoadState(u, a, lb), om, oam.AMConfig(outer_atol=1e-9))
    assert rep.converged and orep.converged
    # both sides stop at |Phi_FB| <= 1e-9; with or without the tile list the device field differs
    # from the oracle's by the same 3.1e-9 here
    assert np.max(np.abs(host(ad) - ao)) < 1e-8
    assert host(ad).max() > 0.25 and np.count_nonzero(host(ad) > lb + 1e-12) < 0.3 * om.nv
    assert counts and any(2 * free <= total for free, total in counts), counts
