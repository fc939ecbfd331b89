"""Generate golden vectors by running the REFERENCE package itself.

Run in the build container only (needs /root/reference):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes ``tests/golden/ref_*.npz``.  The reference cannot travel to the GPU box,
so these committed fixtures are what pins the oracle (``oracle/``) to the
reference; ``tests/test_oracle_golden.py`` checks the oracle against them and
the GPU parity tests check the CUDA path against the oracle.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = os.environ.get("PHASEFRAC_REF", "/root/reference/pkg/src")
sys.path.insert(0, REF)

from phasefrac import cases, fem, linalg, mesh, model, solver, vi  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def random_state(problem, rng, lb_scale=0.3):
    nv = problem.n_vertices
    lb = rng.uniform(0.0, lb_scale, nv)
    alpha = lb + rng.uniform(0.0, 1.0, nv) * (1.0 - lb)
    u = rng.standard_normal(problem.n_udofs) * 0.1
    return fem.State(u=u, alpha=alpha, alpha_lb=lb)


def gen_operators():
    """Energies, residuals and Hessian-block products on small union-jack meshes."""
    out = {}
    rng = np.random.default_rng(1234)
    for tag, (L, H, h, nu) in {"sq4": (1.0, 1.0, 0.25, 0.3), "bar": (1.0, 0.3, 0.05, 0.0),
                               "rect": (2.0, 1.0, 0.125, 0.25)}.items():
        mat = model.Material(E=1.7, nu=nu, Gc=1.3, ell=0.1, k_ell=1e-6)
        m = mesh.rect_mesh(L, H, h)
        prob = fem.Discretization(m, mat)
        st = random_state(prob, rng)
        prob.eps0 = 0.01 * rng.standard_normal(prob.eps0.shape)
        xu = rng.standard_normal(prob.n_udofs)
        xa = rng.standard_normal(prob.n_vertices)
        left = mesh.boundary_dofs(m, "left", "displacement_x1")
        right = mesh.boundary_dofs(m, "right", "displacement_x1")
        prob.bc = fem.combine_bcs(fem.DirichletBC(left, np.zeros(left.size)),
                                  fem.DirichletBC(right, np.full(right.size, 0.07)),
                                  fem.DirichletBC(np.array([1]), np.zeros(1)))
        e = fem.assemble_energy(st, prob)
        Kuu_raw = fem.assemble_Kuu(st, prob, apply_bc=False)
        Kuu_bc = fem.assemble_Kuu(st, prob, apply_bc=True)
        Kua = fem.assemble_Kua(st, prob, apply_bc=True)
        Kua_raw = fem.assemble_Kua(st, prob, apply_bc=False)
        Kaa = fem.assemble_Kaa(st, prob)
        f = fem.assemble_load_u(st, prob)
        Kl, fl = fem.apply_dirichlet(Kuu_raw, f, prob.bc)
        out.update({
            f"{tag}_params": np.array([L, H, h, mat.E, mat.nu, mat.Gc, mat.ell, mat.k_ell]),
            f"{tag}_u": st.u, f"{tag}_alpha": st.alpha, f"{tag}_alpha_lb": st.alpha_lb,
            f"{tag}_eps0": prob.eps0, f"{tag}_xu": xu, f"{tag}_xa": xa,
            f"{tag}_bc_dofs": prob.bc.dofs, f"{tag}_bc_vals": prob.bc.values,
            f"{tag}_energy": np.array(e),
            f"{tag}_ru_bc": fem.assemble_residual_u(st, prob, apply_bc=True),
            f"{tag}_ru_raw": fem.assemble_residual_u(st, prob, apply_bc=False),
            f"{tag}_ra": fem.assemble_residual_alpha(st, prob),
            f"{tag}_f": f,
            f"{tag}_Kuu_raw_x": Kuu_raw @ xu, f"{tag}_Kuu_bc_x": Kuu_bc @ xu,
            f"{tag}_Kua_x": Kua @ xa, f"{tag}_Kua_raw_x": Kua_raw @ xa,
            f"{tag}_KuaT_x": Kua.T @ xu, f"{tag}_Kaa_x": Kaa @ xa,
            f"{tag}_lifted_rhs": fl, f"{tag}_Kuu_diag": Kuu_raw.diagonal(),
            f"{tag}_Kaa_diag": Kaa.diagonal(),
            f"{tag}_first_order": solver.first_order_residual(st, prob),
            f"{tag}_Kuu_nnz": np.array([Kuu_raw.nnz, Kaa.nnz]),
        })
    return out


def gen_vi():
    """rsls_solve on random box QPs, FB values."""
    out = {}
    rng = np.random.default_rng(77)
    xs = []
    for k in range(40):
        n = int(rng.integers(2, 9))
        A = rng.standard_normal((n, n))
        H = A @ A.T + 0.5 * np.eye(n)
        c = rng.standard_normal(n)
        lo = rng.uniform(-1.0, 0.0, n)
        hi = lo + rng.uniform(0.2, 2.0, n)
        x0 = rng.uniform(lo, hi)
        import scipy.sparse as sp
        Hs = sp.csr_matrix(H)
        prob = vi.MCProblem(lambda x, Hs=Hs, c=c: Hs @ x + c, lambda x, Hs=Hs: Hs, lo, hi)
        x, rep = vi.rsls_solve(prob, x0, vi.VIConfig(abs_tol=1e-12, max_iterations=100))
        out[f"qp{k}_H"] = H
        out[f"qp{k}_c"] = c
        out[f"qp{k}_lo"] = lo
        out[f"qp{k}_hi"] = hi
        out[f"qp{k}_x0"] = x0
        out[f"qp{k}_x"] = x
        out[f"qp{k}_hist"] = np.array(rep.residual_history)
        xs.append(x)
    a = rng.standard_normal(50)
    b = rng.standard_normal(50)
    out["fb_a"], out["fb_b"] = a, b
    out["fb_phi"] = vi.fb_phi(a, b)
    lo = np.where(rng.uniform(size=50) < 0.7, rng.uniform(-1, 0, 50), -np.inf)
    hi = np.where(rng.uniform(size=50) < 0.7, rng.uniform(1, 2, 50), np.inf)
    x = np.clip(rng.uniform(-1.5, 2.5, 50), lo, hi)
    F = rng.standard_normal(50)
    out["fbc_x"], out["fbc_F"], out["fbc_lo"], out["fbc_hi"] = x, F, lo, hi
    out["fbc_phi"] = vi.fb_composite(x, F, lo, hi)
    return out


def gen_krylov():
    """cg_solve / minres_solve / field-split / Chebyshev on seeded systems."""
    out = {}
    rng = np.random.default_rng(5)
    n = 60
    A = rng.standard_normal((n, n))
    S = A @ A.T + 0.1 * np.eye(n)
    b = rng.standard_normal(n)
    import scipy.sparse as sp
    Ss = sp.csr_matrix(S)
    x, rep = linalg.cg_solve(Ss, b, precond=linalg.JacobiPreconditioner(Ss), rtol=1e-10)
    out.update(cg_S=S, cg_b=b, cg_x=x, cg_it=np.array([rep.iterations]))
    cheb = linalg.ChebyshevPreconditioner(Ss)
    out["cheb_r"] = b
    out["cheb_z"] = cheb.matvec(b)
    # indefinite block system with field split
    nu_, na = 40, 20
    Au = rng.standard_normal((nu_, nu_))
    Au = Au @ Au.T + np.eye(nu_)
    Cc = rng.standard_normal((na, na))
    Cc = Cc @ Cc.T + np.eye(na)
    Bm = 0.3 * rng.standard_normal((nu_, na))
    blk = linalg.BlockJacobian(sp.csr_matrix(Au), sp.csr_matrix(Bm), sp.csr_matrix(Cc))
    rhs = rng.standard_normal(nu_ + na)
    P = linalg.FieldSplitPreconditioner(blk, linalg.inner_direct(blk.A), linalg.inner_direct(blk.C))
    xm, rm = linalg.minres_solve(blk, rhs, precond=P, rtol=1e-10)
    out.update(mr_A=Au, mr_B=Bm, mr_C=Cc, mr_rhs=rhs, mr_x=xm, mr_it=np.array([rm.iterations]),
               fs_r=rhs, fs_z=P.matvec(rhs))
    xm2, rm2 = linalg.minres_solve(blk, rhs, precond=None, rtol=1e-10)
    out.update(mr_noprec_x=xm2, mr_noprec_it=np.array([rm2.iterations]))
    return out


def gen_steps():
    """Half-steps, AM, Newton and a short quasi-static run on the traction bar."""
    out = {}
    mat = model.Material(ell=0.1)
    setup = cases.setup_traction(mat, h=0.05, n_steps=4)
    prob = setup.problem
    st = fem.State.zeros(setup.mesh)
    t = 1.4 * setup.params["critical_traction"]
    setup.apply_load(prob, st, t)
    st.load = t
    st.u[prob.bc.dofs] = prob.bc.values
    st.alpha = np.maximum(st.alpha, setup.seed_alpha)
    out["half_u0"], out["half_alpha0"] = st.u.copy(), st.alpha.copy()
    cfg = solver.SolverConfig(outer_atol=1e-9)
    u1, _ = solver.elastic_step(st, prob, cfg)
    out["half_u_star"] = u1
    st.u = u1
    a1, rep = solver.damage_step(st, prob, cfg)
    out["half_a_star"] = a1
    out["half_vi_it"] = np.array([rep.iterations])
    st.alpha = a1
    out["half_resnorm"] = np.array([solver.residual_norm(st, prob)])
    # AM to convergence from the same start
    st2 = fem.State.zeros(setup.mesh)
    setup.apply_load(prob, st2, t)
    st2.u[prob.bc.dofs] = prob.bc.values
    st2.alpha = np.maximum(st2.alpha, setup.seed_alpha)
    r = solver.am_solve(st2, prob, solver.SolverConfig(outer_atol=1e-9))
    out["am_u"], out["am_alpha"] = st2.u, st2.alpha
    out["am_its"] = np.array([r.am_iterations])
    out["am_energy_hist"] = np.array([e.total for e in r.energy_history])
    out["am_res_hist"] = np.array(r.residual_history)
    # over-relaxed AM (omega = 1.6)
    st3 = fem.State.zeros(setup.mesh)
    setup.apply_load(prob, st3, t)
    st3.u[prob.bc.dofs] = prob.bc.values
    st3.alpha = np.maximum(st3.alpha, setup.seed_alpha)
    r3 = solver.am_solve(st3, prob, solver.SolverConfig(outer_atol=1e-9, omega=1.6))
    out["oram_alpha"], out["oram_its"] = st3.alpha, np.array([r3.am_iterations])
    out["oram_wbmin"] = np.array([r3.omega_bar_min])
    # ORAM-N
    st4 = fem.State.zeros(setup.mesh)
    setup.apply_load(prob, st4, t)
    st4.u[prob.bc.dofs] = prob.bc.values
    st4.alpha = np.maximum(st4.alpha, setup.seed_alpha)
    r4 = solver.oram_n_solve(st4, prob, solver.SolverConfig(method="oram_newton", omega=1.3,
                                                            outer_atol=1e-9))
    out["oramn_alpha"], out["oramn_u"] = st4.alpha, st4.u
    out["oramn_counts"] = np.array([r4.am_iterations, r4.newton_iterations, r4.newton_attempts])
    out["oramn_energy"] = np.array(fem.assemble_energy(st4, prob))
    # Short quasi-static run (8 steps, AM omega=1, tight tolerance)
    setup8 = cases.setup_traction(mat, h=0.05, n_steps=8)
    recs = cases.run_quasistatic(setup8, solver.SolverConfig(outer_atol=1e-9))
    out["run_loads"] = np.array([r.load for r in recs])
    out["run_energy"] = np.array([list(r.energy) for r in recs])
    out["run_its"] = np.array([r.report.am_iterations for r in recs])
    out["run_alpha_final"] = recs[-1].alpha
    out["run_u_final"] = recs[-1].u
    return out


def gen_surfing():
    """Graded (banded) mesh operators and a short surfing run."""
    out = {}
    rng = np.random.default_rng(4242)
    mat = model.Material(E=1.3, nu=0.27, Gc=0.9, ell=0.1, k_ell=1e-6)
    m = mesh.banded_rect_mesh(1.0, 0.8, 0.05, 0.2, 0.1)
    prob = fem.Discretization(m, mat)
    st = random_state(prob, rng)
    xu = rng.standard_normal(prob.n_udofs)
    xa = rng.standard_normal(prob.n_vertices)
    e = fem.assemble_energy(st, prob)
    out["op_vertices"] = m.vertices
    out["op_u"], out["op_alpha"], out["op_lb"] = st.u, st.alpha, st.alpha_lb
    out["op_xu"], out["op_xa"] = xu, xa
    out["op_energy"] = np.array([e.elastic, e.dissipated, e.total])
    out["op_ru"] = fem.assemble_residual_u(st, prob)
    out["op_ra"] = fem.assemble_residual_alpha(st, prob)
    out["op_Kuu_x"] = fem.assemble_Kuu(st, prob, apply_bc=False) @ xu
    out["op_Kaa_x"] = fem.assemble_Kaa(st, prob) @ xa
    out["op_Kua_x"] = fem.assemble_Kua(st, prob, apply_bc=False) @ xa
    smat = model.Material(E=1.0, nu=0.3, Gc=1.0, ell=0.2)
    setup = cases.setup_surfing(smat, h=0.05, n_steps=12, t_end=0.9)
    recs = cases.run_quasistatic(setup, solver.SolverConfig(method="am", omega=1.0), snapshot_stride=1)
    out["surf_vertices"] = setup.mesh.vertices
    out["surf_energy"] = np.array([[r.energy.elastic, r.energy.dissipated, r.energy.total] for r in recs])
    out["surf_am"] = np.array([r.report.am_iterations for r in recs])
    out["surf_alpha"] = np.stack([r.alpha for r in recs])
    out["surf_loads"] = np.array([r.load for r in recs])
    return out


def gen_jitter():
    """Hessian-block products on the reference's JITTERED rect meshes (mesh.py:134-141), the
    mesh family of its thermal-shock case (cases.py:195-234): pins the element-list path."""
    out = {}
    rng = np.random.default_rng(4321)
    for tag, (L, H, h, jit, seed) in {"jit": (2.0, 1.0, 0.125, 0.25, 0),
                                      "jit3": (1.0, 0.5, 0.0625, 0.3, 7)}.items():
        mat = model.Material(E=1.7, nu=0.3, Gc=1.3, ell=0.1, k_ell=1e-6)
        m = mesh.rect_mesh(L, H, h, jitter=jit, seed=seed)
        prob = fem.Discretization(m, mat)
        st = random_state(prob, rng)
        xu = rng.standard_normal(prob.n_udofs)
        xa = rng.standard_normal(prob.n_vertices)
        left = mesh.boundary_dofs(m, "left", "displacement_x1")
        bottom = mesh.boundary_dofs(m, "bottom", "displacement_x2")
        prob.bc = fem.combine_bcs(fem.DirichletBC(left, np.zeros(left.size)),
                                  fem.DirichletBC(bottom, np.zeros(bottom.size)))
        out.update({
            f"{tag}_params": np.array([L, H, h, jit, seed, mat.E, mat.nu, mat.Gc, mat.ell, mat.k_ell]),
            f"{tag}_vertices": m.vertices, f"{tag}_triangles": m.triangles,
            f"{tag}_u": st.u, f"{tag}_alpha": st.alpha, f"{tag}_xu": xu, f"{tag}_xa": xa,
            f"{tag}_bc_dofs": prob.bc.dofs,
            f"{tag}_Kuu_raw_x": fem.assemble_Kuu(st, prob, apply_bc=False) @ xu,
            f"{tag}_Kuu_bc_x": fem.assemble_Kuu(st, prob, apply_bc=True) @ xu,
            f"{tag}_Kaa_x": fem.assemble_Kaa(st, prob) @ xa,
        })
    return out


def main():
    if len(sys.argv) > 1 and sys.argv[1] == "surfing":  # regenerate only the surfing fixture
        np.savez_compressed(os.path.join(OUT, "ref_surfing.npz"), **gen_surfing())
        return
    if len(sys.argv) > 1 and sys.argv[1] == "jitter":  # regenerate only the jittered-mesh fixture
        np.savez_compressed(os.path.join(OUT, "ref_jitter.npz"), **gen_jitter())
        return
    np.savez_compressed(os.path.join(OUT, "ref_jitter.npz"), **gen_jitter())
    np.savez_compressed(os.path.join(OUT, "ref_surfing.npz"), **gen_surfing())
    np.savez_compressed(os.path.join(OUT, "ref_operators.npz"), **gen_operators())
    np.savez_compressed(os.path.join(OUT, "ref_vi.npz"), **gen_vi())
    np.savez_compressed(os.path.join(OUT, "ref_krylov.npz"), **gen_krylov())
    np.savez_compressed(os.path.join(OUT, "ref_steps.npz"), **gen_steps())
    print("golden fixtures written to", OUT)


if __name__ == "__main__":
    main()
