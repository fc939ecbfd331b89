"""Element-list (jittered / unstructured) P1 path -- SURVEY 8(f) row 4, first step.

CPU: the oracle's jitter (oracle/meshgen.jitter_interior) and the package's mesh generator
reproduce the REFERENCE's jittered rect_mesh bit for bit (tests/golden/ref_jitter.npz, made by
running the reference, make_golden.py gen_jitter); the oracle's assembled Kuu / Kaa products on
those meshes match the reference's; the C ABI validates meshes without a device.
GPU: pf_umesh_apply_Kuu / _Kaa against the reference goldens and the oracle's assembled CSR
(relative max error <= 1e-12), 2D and 3D, AT1/AT2, plane stress/strain, per-element fields,
Dirichlet elimination, bitwise reproducibility.
"""

import ctypes as C
import os

import numpy as np
import pytest

from conftest import GOLDEN
from oracle.meshgen import grid_mesh, jitter_interior, kuhn_mesh
from oracle.p1 import MaterialSpec, P1Model, eliminate_rows_cols

TOL = 1e-12


def golden():
    return np.load(os.path.join(GOLDEN, "ref_jitter.npz"))


def rel(a, b):
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


def oracle_model(d, tag):
    L, H, h, jit, seed, E, nu, Gc, ell, k_ell = d[f"{tag}_params"]
    m = jitter_interior(grid_mesh(round(L / h), round(H / h), L, H), jit, int(seed))
    spec = MaterialSpec(E=E, nu=nu, Gc=Gc, ell=ell, k_ell=k_ell, model="AT1", regime="plane_stress")
    return m, P1Model(m, spec)


# ---- CPU -------------------------------------------------------------------------------------
@pytest.mark.parametrize("tag", ["jit", "jit3"])
def test_oracle_jitter_is_the_reference_mesh(tag):
    d = golden()
    m, _ = oracle_model(d, tag)
    assert np.array_equal(m.vertices, d[f"{tag}_vertices"])
    assert np.array_equal(m.elements, d[f"{tag}_triangles"])


@pytest.mark.parametrize("tag", ["jit", "jit3"])
def test_package_jittered_rect_mesh_is_the_reference_mesh(tag):
    import paper_1511_08463_b200 as pf
    d = golden()
    L, H, h, jit, seed = d[f"{tag}_params"][:5]
    m = pf.jittered_rect_mesh(L, H, h, jitter=jit, seed=int(seed))
    assert np.array_equal(m.vertices, d[f"{tag}_vertices"])
    assert np.array_equal(m.elements, d[f"{tag}_triangles"])


@pytest.mark.parametrize("tag", ["jit", "jit3"])
def test_oracle_operators_match_reference_on_jittered_mesh(tag):
    d = golden()
    _, om = oracle_model(d, tag)
    u, a, xu, xa = d[f"{tag}_u"], d[f"{tag}_alpha"], d[f"{tag}_xu"], d[f"{tag}_xa"]
    assert rel(om.Kuu(a, eliminate=False) @ xu, d[f"{tag}_Kuu_raw_x"]) < TOL
    K = eliminate_rows_cols(om.Kuu(a, eliminate=False), d[f"{tag}_bc_dofs"])
    assert rel(K @ xu, d[f"{tag}_Kuu_bc_x"]) < TOL
    assert rel(om.Kaa(u, a) @ xa, d[f"{tag}_Kaa_x"]) < TOL


def test_package_box_mesh_matches_oracle_kuhn():
    import paper_1511_08463_b200 as pf
    m = pf.jittered_box_mesh(3, 4, 5, 1.0, 2.0, 1.5, jitter=0.2, seed=5)
    o = jitter_interior(kuhn_mesh(3, 4, 5, 1.0, 2.0, 1.5), 0.2, 5)
    assert np.array_equal(m.vertices, o.vertices)
    assert np.array_equal(m.elements, o.elements)


def test_jitter_range_rejected():
    import paper_1511_08463_b200 as pf
    with pytest.raises(ValueError, match="jitter"):
        pf.jittered_rect_mesh(1.0, 1.0, 0.25, jitter=0.5)


def _desc(mesh, **kw):
    from paper_1511_08463_b200.umesh import _UDesc
    v, el = mesh.vertices, mesh.elements
    args = dict(dim=mesh.dim, regime=0 if mesh.dim == 2 else 2, model=0, reserved=0,
                n_vertices=v.shape[0], n_elements=el.shape[0], vertices=v.ctypes.data,
                elements=el.ctypes.data, E_elem=None, Gc_elem=None, E=1.0, nu=0.3, Gc=1.0,
                ell=0.1, k_ell=1e-6)
    args.update(kw)
    return _UDesc(**args)


def test_capi_create_validates_without_device():
    import paper_1511_08463_b200 as pf
    from paper_1511_08463_b200 import _lib
    lib = _lib.load()
    mesh = pf.jittered_rect_mesh(1.0, 0.5, 0.125, jitter=0.2, seed=1)
    h = C.c_void_p()
    assert lib.pf_umesh_create(C.byref(_desc(mesh)), C.byref(h)) == _lib.PF_OK
    nv, nt = mesh.n_vertices, mesh.n_elements
    adj = 3 * nt
    n = 2 * nv
    nb = max((n + 255) // 256, (nt + 255) // 256)
    expect = sum((b + 255) // 256 * 256 for b in (nt * 64, nt * 16, (nv + 1) * 4, adj * 4, nv,
                                                  n * 8, n * 8, n * 8, n * 8, n * 8, 2 * nb * 8)) + 256 + 256  # scalars + grid barrier
    assert lib.pf_umesh_workspace_bytes(h) == expect
    lib.pf_umesh_destroy(h)
    # an inverted triangle, an out-of-range index, a regime/dim mismatch
    bad = pf.UnstructuredMesh(mesh.vertices, mesh.elements[:, [0, 2, 1]])
    h = C.c_void_p()
    assert lib.pf_umesh_create(C.byref(_desc(bad)), C.byref(h)) == _lib.PF_EINVAL
    assert b"non-CCW" in lib.pf_umesh_last_error(None)
    oob = pf.UnstructuredMesh(mesh.vertices, np.where(mesh.elements == 3, nv + 7, mesh.elements))
    assert lib.pf_umesh_create(C.byref(_desc(oob)), C.byref(h)) == _lib.PF_EINVAL
    assert b"out of range" in lib.pf_umesh_last_error(None)
    assert lib.pf_umesh_create(C.byref(_desc(mesh, regime=2)), C.byref(h)) == _lib.PF_EINVAL
    box = pf.jittered_box_mesh(2, 2, 2)
    flipped = pf.UnstructuredMesh(box.vertices, box.elements[:, [0, 2, 1, 3]])
    assert lib.pf_umesh_create(C.byref(_desc(flipped)), C.byref(h)) == _lib.PF_EINVAL
    assert b"inverted" in lib.pf_umesh_last_error(None)


# ---- GPU -------------------------------------------------------------------------------------
def _dev(a):
    import torch
    return torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda")


@pytest.mark.gpu
@pytest.mark.parametrize("tag", ["jit", "jit3"])
def test_gpu_umesh_matches_reference_goldens(tag):
    import paper_1511_08463_b200 as pf
    d = golden()
    L, H, h, jit, seed, E, nu, Gc, ell, k_ell = d[f"{tag}_params"]
    mesh = pf.jittered_rect_mesh(L, H, h, jitter=jit, seed=int(seed))
    ops = pf.UnstructuredOperators(mesh, pf.Material(E=E, nu=nu, Gc=Gc, ell=ell, k_ell=k_ell), "AT1")
    u, a, xu, xa = (_dev(d[f"{tag}_{k}"]) for k in ("u", "alpha", "xu", "xa"))
    assert rel(ops.apply_Kuu(a, xu).cpu().numpy(), d[f"{tag}_Kuu_raw_x"]) < TOL
    assert rel(ops.apply_Kaa(u, a, xa).cpu().numpy(), d[f"{tag}_Kaa_x"]) < TOL
    ops.set_dirichlet(d[f"{tag}_bc_dofs"])
    assert rel(ops.apply_Kuu(a, xu, apply_bc=True).cpu().numpy(), d[f"{tag}_Kuu_bc_x"]) < TOL
    assert ops.launches == 3


CASES = [
    # dim, regime, model, shape, jitter, hetero
    (2, "plane_strain", "AT2", (40, 23), 0.2, True),
    (2, "plane_stress", "AT1", (1, 1), 0.0, False),
    (2, "plane_strain", "AT1", (64, 64), 0.25, False),
    (3, "3d", "AT1", (5, 4, 6), 0.1, True),
    (3, "3d", "AT2", (9, 9, 9), 0.1, False),
    (3, "3d", "AT1", (1, 1, 1), 0.0, False),
]


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c[0]}d-{c[1]}-{c[2]}-{'x'.join(map(str, c[3]))}")
def test_gpu_umesh_parity_vs_oracle(case):
    import torch
    import paper_1511_08463_b200 as pf
    dim, regime, model, shape, jit, hetero = case
    om_mesh = (jitter_interior(grid_mesh(*shape, 2.0, 1.0), jit, 11) if dim == 2
               else jitter_interior(kuhn_mesh(*shape), jit, 11))
    rng = np.random.default_rng(sum(shape) + dim)
    T, V = om_mesh.n_elements, om_mesh.n_vertices
    Ee = rng.uniform(0.5, 1.5, T) if hetero else None
    Ge = rng.uniform(0.5, 1.5, T) if hetero else None
    spec = MaterialSpec(E=1.3, nu=0.3, Gc=0.9, ell=0.07, k_ell=1e-6, model=model, regime=regime)
    om = P1Model(om_mesh, spec, Ee, Ge)
    mesh = pf.UnstructuredMesh(om_mesh.vertices, om_mesh.elements)
    ops = pf.UnstructuredOperators(mesh, pf.Material(E=1.3, nu=0.3, Gc=0.9, ell=0.07, k_ell=1e-6,
                                                     regime=regime), model, Ee, Ge)
    a = rng.uniform(0, 1, V)
    u = rng.standard_normal(dim * V)
    xu = rng.standard_normal(dim * V)
    xa = rng.standard_normal(V)
    y = ops.apply_Kuu(_dev(a), _dev(xu))
    assert rel(y.cpu().numpy(), om.Kuu(a, eliminate=False) @ xu) < TOL
    assert rel(ops.apply_Kaa(_dev(u), _dev(a), _dev(xa)).cpu().numpy(), om.Kaa(u, a) @ xa) < TOL
    bc = np.unique(np.concatenate([dim * om_mesh.boundary[next(iter(om_mesh.boundary))] + c
                                   for c in range(dim)]))
    ops.set_dirichlet(bc)
    yb = ops.apply_Kuu(_dev(a), _dev(xu), apply_bc=True).cpu().numpy()
    assert rel(yb, eliminate_rows_cols(om.Kuu(a, eliminate=False), bc) @ xu) < TOL
    # fixed-order gathers: bitwise reproducible
    y2 = ops.apply_Kuu(_dev(a), _dev(xu))
    assert torch.equal(y, y2)


@pytest.mark.gpu
def test_gpu_umesh_rejects_bad_arguments():
    import torch
    import paper_1511_08463_b200 as pf
    ops = pf.UnstructuredOperators(pf.jittered_rect_mesh(1.0, 1.0, 0.25, 0.2), pf.Material())
    with pytest.raises(ValueError, match="float64"):
        ops.apply_Kuu(torch.zeros(ops.n_vertices, device="cuda"), torch.zeros(ops.n_udofs, device="cuda"))
    with pytest.raises(ValueError, match="dof out of range"):
        ops.set_dirichlet([ops.n_udofs])
    with pytest.raises(ValueError, match="does not match"):
        pf.UnstructuredOperators(pf.jittered_box_mesh(2, 2, 2), pf.Material())


@pytest.mark.gpu
@pytest.mark.parametrize("dim", [2, 3])
def test_gpu_umesh_jacobi_pcg_solves_eliminated_system(dim):
    """Device Jacobi PCG (pf_umesh_elastic_solve) against a direct solve of the oracle's
    eliminated Kuu on a jittered mesh; iterates are bitwise reproducible."""
    import scipy.sparse.linalg as spla
    import torch
    import paper_1511_08463_b200 as pf
    from paper_1511_08463_b200.linalg import LinearSolverError
    regime = "plane_strain" if dim == 2 else "3d"
    om_mesh = (jitter_interior(grid_mesh(48, 24, 2.0, 1.0), 0.2, 3) if dim == 2
               else jitter_interior(kuhn_mesh(8, 7, 9), 0.1, 3))
    rng = np.random.default_rng(77 + dim)
    V = om_mesh.n_vertices
    spec = MaterialSpec(E=1.0, nu=0.3, Gc=1.0, ell=0.1, k_ell=1e-6, regime=regime)
    om = P1Model(om_mesh, spec)
    a = rng.uniform(0, 0.9, V)
    left = om_mesh.boundary["left" if dim == 2 else "x0"]
    bc = np.unique(np.concatenate([dim * left + c for c in range(dim)]))
    K = eliminate_rows_cols(om.Kuu(a, eliminate=False), bc).tocsc()
    b = rng.standard_normal(dim * V)
    ref = spla.spsolve(K, b)
    ops = pf.UnstructuredOperators(pf.UnstructuredMesh(om_mesh.vertices, om_mesh.elements),
                                   pf.Material(E=1.0, nu=0.3, Gc=1.0, ell=0.1, k_ell=1e-6, regime=regime))
    ops.set_dirichlet(bc)
    x, rep = ops.elastic_solve(_dev(a), _dev(b), rtol=1e-11, maxit=20000)
    assert rep.converged and rep.iterations > 0
    xh = x.cpu().numpy()
    assert rel(xh, ref) < 1e-8
    assert np.linalg.norm(K @ xh - b) <= 1e-11 * np.linalg.norm(b) * 1.5
    x2, rep2 = ops.elastic_solve(_dev(a), _dev(b), rtol=1e-11, maxit=20000)
    assert rep2.iterations == rep.iterations and torch.equal(x, x2)
    with pytest.raises(LinearSolverError, match="stalled"):
        ops.elastic_solve(_dev(a), _dev(b), rtol=1e-11, maxit=5, check_every=5)


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c[0]}d-{c[1]}-{c[2]}-{'x'.join(map(str, c[3]))}")
def test_gpu_umesh_physics_vs_oracle(case):
    """Energy parts (1e-12 relative) and the raw gradients r_u, r_alpha on element-list meshes."""
    import paper_1511_08463_b200 as pf
    dim, regime, model, shape, jit, hetero = case
    om_mesh = (jitter_interior(grid_mesh(*shape, 2.0, 1.0), jit, 5) if dim == 2
               else jitter_interior(kuhn_mesh(*shape), jit, 5))
    rng = np.random.default_rng(3 * sum(shape) + dim)
    T, V = om_mesh.n_elements, om_mesh.n_vertices
    Ee = rng.uniform(0.5, 1.5, T) if hetero else None
    Ge = rng.uniform(0.5, 1.5, T) if hetero else None
    spec = MaterialSpec(E=1.3, nu=0.3, Gc=0.9, ell=0.07, k_ell=1e-6, model=model, regime=regime)
    om = P1Model(om_mesh, spec, Ee, Ge)
    ops = pf.UnstructuredOperators(pf.UnstructuredMesh(om_mesh.vertices, om_mesh.elements),
                                   pf.Material(E=1.3, nu=0.3, Gc=0.9, ell=0.07, k_ell=1e-6, regime=regime),
                                   model, Ee, Ge)
    a = rng.uniform(0, 1, V)
    u = 0.1 * rng.standard_normal(dim * V)
    (el, ds, tot), ru, ra = ops.physics(_dev(u), _dev(a))
    ref = om.energy(u, a)
    assert abs(el - ref[0]) <= 1e-12 * abs(ref[0])
    assert abs(ds - ref[1]) <= 1e-12 * abs(ref[1])
    assert abs(tot - ref[2]) <= 1e-12 * abs(ref[2])
    assert rel(ru.cpu().numpy(), om.residual_u(u, a, bc_rows="none")) < TOL
    assert rel(ra.cpu().numpy(), om.residual_alpha(u, a)) < TOL


@pytest.mark.gpu
@pytest.mark.parametrize("dim,model", [(2, "AT1"), (2, "AT2"), (3, "AT1"), (3, "AT2")])
def test_gpu_umesh_damage_solve_vs_oracle_rsls(dim, model):
    """Damage box QP at fixed u (damage_half_step: rsls on Kaa(u) a + c over [alpha_lb, 1]) on a
    jittered mesh: the device reduced-space solve and the oracle's rsls reach the same unique
    minimiser; the device result is FB-stationary and bitwise reproducible."""
    import torch
    import paper_1511_08463_b200 as pf
    from oracle.mcp import RSLSConfig, fb_box, rsls
    from paper_1511_08463_b200.vi import VIConfig
    regime = "plane_strain" if dim == 2 else "3d"
    om_mesh = (jitter_interior(grid_mesh(40, 20, 2.0, 1.0), 0.25, 9) if dim == 2
               else jitter_interior(kuhn_mesh(7, 6, 8), 0.1, 9))
    V = om_mesh.n_vertices
    rng = np.random.default_rng(11 * dim + (model == "AT2"))
    spec = MaterialSpec(E=1.0, nu=0.3, Gc=1.0, ell=0.1, k_ell=1e-6, model=model, regime=regime)
    om = P1Model(om_mesh, spec)
    x = om_mesh.vertices
    u = np.zeros(dim * V)
    u[0::dim] = 0.6 * x[:, 0] * (1.0 + 0.5 * np.sin(3.0 * x[:, 1]))
    u += 0.02 * rng.standard_normal(dim * V)
    lb = np.where(rng.uniform(size=V) < 0.3, rng.uniform(0.0, 0.6, V), 0.0)
    a0 = lb.copy()
    K = om.Kaa(u, a0)
    c = om.residual_alpha(u, a0) - K @ a0
    ref, st = rsls(lambda a: K @ a + c, lambda a: K, lb, np.ones(V), a0, RSLSConfig(abs_tol=1e-10),
                   jac_matvec=lambda J: (lambda v: J.T @ v))
    ops = pf.UnstructuredOperators(pf.UnstructuredMesh(om_mesh.vertices, om_mesh.elements),
                                   pf.Material(E=1.0, nu=0.3, Gc=1.0, ell=0.1, k_ell=1e-6, regime=regime),
                                   model)
    cfg = VIConfig(abs_tol=1e-10, inner_rtol=1e-12)
    ad, rep = ops.damage_solve(_dev(u), _dev(lb), _dev(a0), config=cfg)
    assert rep.converged and rep.iterations >= 1 and rep.total_krylov_iterations > 0
    ah = ad.cpu().numpy()
    assert np.all(ah >= lb) and np.all(ah <= 1.0)
    assert np.linalg.norm(fb_box(ah, K @ ah + c, lb, np.ones(V))) <= 1e-9
    assert np.max(np.abs(ah - ref)) < 1e-8
    assert 0 < np.count_nonzero(ah > lb + 1e-12) < V  # the bound is active on part of the mesh
    ad2, rep2 = ops.damage_solve(_dev(u), _dev(lb), _dev(a0), config=cfg)
    assert rep2.iterations == rep.iterations and torch.equal(ad, ad2)


def _am_case(model):
    from oracle.p1 import MaterialSpec, P1Model
    mesh = jitter_interior(grid_mesh(24, 12, 2.0, 1.0), 0.2, 4)
    V = mesh.n_vertices
    Gc, t = (0.05, 0.1) if model == "AT2" else (0.01, 0.45)
    spec = MaterialSpec(E=1.0, nu=0.3, Gc=Gc, ell=0.15, k_ell=1e-6, model=model, regime="plane_strain")
    left, right = mesh.boundary["left"], mesh.boundary["right"]
    dofs = np.concatenate([2 * left, 2 * left + 1, 2 * right])
    vals = np.concatenate([np.zeros(2 * left.size), np.full(right.size, t)])
    order = np.argsort(dofs)
    m = P1Model(mesh, spec)
    m.bc = (dofs[order], vals[order])
    lb = np.zeros(V)
    return mesh, spec, m, dofs[order], vals[order], lb


@pytest.mark.parametrize("model", ["AT1", "AT2"])
def test_oracle_am_case_damages(model):
    """The AM parity case loads past the damage threshold (oracle only, CPU)."""
    from oracle.am import AMConfig, LoadState, am_loop
    mesh, spec, m, dofs, vals, lb = _am_case(model)
    st = LoadState.zeros(m, lb)
    rep = am_loop(st, m, AMConfig(elastic_solver="direct", outer_atol=1e-7, max_am_iterations=400))
    assert rep.converged and st.alpha.max() > 1e-3


@pytest.mark.gpu
@pytest.mark.parametrize("model", ["AT1", "AT2"])
def test_gpu_umesh_am_load_step_vs_oracle(model):
    """One AM load step on a jittered mesh (elastic PCG + damage box QP on the element-list
    path) against the oracle's am_loop with direct elastic solves: same fixed point."""
    import torch
    import paper_1511_08463_b200 as pf
    from oracle.am import AMConfig, LoadState, am_loop
    mesh, spec, m, dofs, vals, lb = _am_case(model)
    st = LoadState.zeros(m, lb)
    rep = am_loop(st, m, AMConfig(elastic_solver="direct", outer_atol=1e-7, max_am_iterations=400))
    assert rep.converged
    ops = pf.UnstructuredOperators(pf.UnstructuredMesh(mesh.vertices, mesh.elements),
                                   pf.Material(E=1.0, nu=0.3, Gc=spec.Gc, ell=0.15, k_ell=1e-6,
                                               regime="plane_strain"), model)
    u = torch.zeros(2 * mesh.n_vertices, dtype=torch.float64, device="cuda")
    a = torch.zeros(mesh.n_vertices, dtype=torch.float64, device="cuda")
    stats = ops.am_load_step(u, a, _dev(lb), dofs, vals, outer_atol=1e-7, max_am_iterations=400)
    assert stats["converged"] and stats["final_residual_norm"] <= 1e-7
    assert abs(stats["am_iterations"] - rep.am_iterations) <= 2
    assert np.max(np.abs(a.cpu().numpy() - st.alpha)) < 1e-5
    assert rel(u.cpu().numpy(), st.u) < 1e-5
    ref_en = m.energy(st.u, st.alpha)
    assert abs(stats["energy_history"][-1][2] - ref_en[2]) <= 1e-6 * abs(ref_en[2])


@pytest.mark.gpu
@pytest.mark.parametrize("seed", [0, 1])
def test_gpu_umesh_damage_steepest_descent_fallback(seed):
    """Element-list damage VI: the merit-gradient fallback and the stagnation break of rsls
    (vi.py:241-256), forced by armijo = 0.6 with ls_min_step = 0.6 (every Newton trial fails):
    same iterations, steepest-descent steps and iterate as the oracle; a trial that fails its
    Armijo test is never accepted (the merit never increases)."""
    import paper_1511_08463_b200 as pf
    from oracle.mcp import RSLSConfig, rsls
    from paper_1511_08463_b200.vi import VIConfig
    om_mesh = jitter_interior(grid_mesh(20, 11, 1.3, 0.9), 0.2, 3)
    V = om_mesh.n_vertices
    spec = MaterialSpec(E=1.7, nu=0.27, Gc=1.3, ell=0.1, k_ell=1e-6, model="AT1", regime="plane_stress")
    om = P1Model(om_mesh, spec)
    rng = np.random.default_rng(seed)
    lb = rng.uniform(0.0, 0.3, V)
    a0 = lb + rng.uniform(0, 1, V) * (1 - lb)
    u = rng.standard_normal(2 * V) * 0.4
    K = om.Kaa(u, a0)
    c = om.residual_alpha(u, a0) - K @ a0
    xo, so = rsls(lambda a: K @ a + c, lambda a: K, lb, np.ones(V), a0,
                  RSLSConfig(abs_tol=1e-10, ls_min_step=0.6, armijo=0.6, max_iterations=8),
                  jac_matvec=lambda J: (lambda v: J.T @ v))
    assert so.steepest_descent_steps >= 1
    ops = pf.UnstructuredOperators(pf.UnstructuredMesh(om_mesh.vertices, om_mesh.elements),
                                   pf.Material(E=1.7, nu=0.27, Gc=1.3, ell=0.1, k_ell=1e-6), "AT1")
    cfg = VIConfig(abs_tol=1e-10, ls_min_step=0.6, armijo=0.6, max_iterations=8, inner_rtol=1e-13)
    ad, rep = ops.damage_solve(_dev(u), _dev(lb), _dev(a0), config=cfg, raise_on_failure=False)
    assert (rep.iterations, rep.steepest_descent_steps, rep.converged) == \
        (so.iterations, so.steepest_descent_steps, so.converged)
    assert np.max(np.abs(ad.cpu().numpy() - xo)) < 1e-10
    h = rep.residual_history
    assert all(h[k + 1] <= h[k] for k in range(len(h) - 1))


@pytest.mark.gpu
@pytest.mark.parametrize("dim,model", [(2, "AT1"), (2, "AT2"), (3, "AT1")])
def test_gpu_umesh_eps0_physics_vs_oracle(dim, model):
    """Inelastic strain on the element-list path (pf_umesh_set_eps0; fem.py eps0, oracle/p1.py
    strain = B u - eps0): energies, raw residuals and the damage Hessian's elastic coupling against
    the oracle at 1e-12; the Kuu apply ignores eps0."""
    import torch
    import paper_1511_08463_b200 as pf
    regime = "plane_stress" if dim == 2 else "3d"
    om_mesh = (jitter_interior(grid_mesh(20, 10, 2.0, 1.0), 0.25, 5) if dim == 2
               else jitter_interior(kuhn_mesh(5, 4, 6), 0.1, 5))
    spec = MaterialSpec(E=1.0, nu=0.3, Gc=1.0, ell=0.2, k_ell=1e-6, model=model, regime=regime)
    om = P1Model(om_mesh, spec)
    rng = np.random.default_rng(17 + dim)
    V, T, nv = om_mesh.n_vertices, om_mesh.n_elements, (3 if dim == 2 else 6)
    om.eps0 = 0.05 * rng.standard_normal((T, nv))
    u = 0.1 * rng.standard_normal(dim * V)
    a = rng.uniform(0, 0.9, V)
    x = rng.standard_normal(V)
    ops = pf.UnstructuredOperators(pf.UnstructuredMesh(om_mesh.vertices, om_mesh.elements),
                                   pf.Material(E=1.0, nu=0.3, Gc=1.0, ell=0.2, k_ell=1e-6, regime=regime), model)
    ops.set_eps0(om.eps0)
    en, ru, ra = ops.physics(_dev(u), _dev(a))
    eo = om.energy(u, a)
    assert abs(en[0] - eo.elastic) <= 1e-12 * abs(eo.elastic)
    assert abs(en[1] - eo.dissipated) <= 1e-12 * abs(eo.dissipated)
    rr = om.residual_u(u, a, bc_rows="none")
    assert np.max(np.abs(ru.cpu().numpy() - rr)) <= 1e-12 * np.max(np.abs(rr))
    rra = om.residual_alpha(u, a)
    assert np.max(np.abs(ra.cpu().numpy() - rra)) <= 1e-12 * np.max(np.abs(rra))
    ya = ops.apply_Kaa(_dev(u), _dev(a), _dev(x)).cpu().numpy()
    yo = om.Kaa(u, a) @ x
    assert np.max(np.abs(ya - yo)) <= 1e-12 * np.max(np.abs(yo))
    xu = rng.standard_normal(dim * V)
    yu = ops.apply_Kuu(_dev(a), _dev(xu)).cpu().numpy()
    yuo = om.Kuu(a, eliminate=False) @ xu
    assert np.max(np.abs(yu - yuo)) <= 1e-12 * np.max(np.abs(yuo))
    ops.set_eps0(None)
    en0, _, _ = ops.physics(_dev(u), _dev(a), want_residuals=False)
    om.eps0 = np.zeros((T, nv))
    assert abs(en0[0] - om.energy(u, a).elastic) <= 1e-12 * abs(en0[0])
    del torch
