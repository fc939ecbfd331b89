"""SENT (config 2): the Newton phase of one load step with the field-split inner solves to a
tolerance (default) vs fixed multigrid/Chebyshev block preconditioners (fieldsplit_inner="mg")."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1511_08463_b200 as pf
from paper_1511_08463_b200 import solver as S

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
k = int(sys.argv[2]) if len(sys.argv) > 2 else 8
setup = pf.setup_sent(n=n)
prob = setup.problem
base = dict(method="oram_newton", omega=1.8, outer_atol=1e-6, am_switch_atol=1e-3, elastic_solver="cg",
            elastic_rtol=1e-8, elastic_precond="gmg", max_am_iterations=2000)
cfg = pf.SolverConfig(**base)
st = pf.State.zeros(setup.mesh, setup.initial_alpha_lb)
pf.run_quasistatic(setup, cfg, snapshot_stride=0, state=st, steps=list(range(k)))
t = float(setup.schedule[k])
st.load = t
st.alpha_lb = st.alpha.clone()
setup.apply_load(prob, st, t)
st.u[prob._bc_dofs_dev] = prob._bc_vals_dev
S._snap_bc(st, prob)
S.am_solve(st, prob, cfg, rtol=cfg.am_rtol, cycle=0)
ref = None
for tag, extra in [("tol", {}), ("mg6", dict(fieldsplit_inner="mg", fieldsplit_cheb_degree=6)),
                   ("mg12", dict(fieldsplit_inner="mg", fieldsplit_cheb_degree=12)),
                   ("mg20", dict(fieldsplit_inner="mg", fieldsplit_cheb_degree=20)),
                   ("mg30", dict(fieldsplit_inner="mg", fieldsplit_cheb_degree=30))]:
    c2 = pf.SolverConfig(**{**base, **extra})
    for rep in range(2):
        s = st.copy()
        torch.cuda.synchronize(); t0 = time.perf_counter()
        ns, nr = S.coupled_newton_solve(s, prob, c2)
        torch.cuda.synchronize(); dt = time.perf_counter() - t0
    e = pf.assemble_energy(ns, prob)
    if ref is None:
        ref = (ns, e)
    da = float((ns.alpha - ref[0].alpha).abs().max())
    print(f"{tag:5s} its={nr.iterations} kry={nr.total_krylov_iterations} conv={nr.converged} "
          f"res={nr.final_residual_norm:.3e} E={e.total:.12e} dE={abs(e.total-ref[1].total)/abs(ref[1].total):.1e} "
          f"dalpha={da:.1e} wall={1e3*dt:.1f} ms")
