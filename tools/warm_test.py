"""SENT (config 2): Krylov iterations and wall time of one load step's AM phase with the elastic
initial iterate = the relaxed u (reference order) or the previous elastic solution u*."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1511_08463_b200 as pf
from paper_1511_08463_b200 import solver as S

k = int(sys.argv[1]) if len(sys.argv) > 1 else 8
setup = pf.setup_sent(n=512)
prob = setup.problem
base = dict(method="oram_newton", omega=1.8, outer_atol=1e-6, am_switch_atol=1e-3, elastic_solver="cg",
            elastic_rtol=1e-8, elastic_precond="gmg", max_am_iterations=2000, fieldsplit_inner="mg")
st = pf.State.zeros(setup.mesh, setup.initial_alpha_lb)
pf.run_quasistatic(setup, pf.SolverConfig(**base), snapshot_stride=0, state=st, steps=list(range(k)))
for guess in sys.argv[2:] or ("relaxed", "previous"):
    cfg = pf.SolverConfig(**base, elastic_guess=guess)
    s = st.copy()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    recs = pf.run_quasistatic(setup, cfg, snapshot_stride=0, state=s, steps=[k, k + 1])
    torch.cuda.synchronize(); dt = time.perf_counter() - t0
    print(f"{guess:9s} 2 steps {1e3*dt:.1f} ms  AM its {[r.report.am_iterations for r in recs]} "
          f"kry {[r.report.total_krylov_iterations for r in recs]} E {recs[-1].energy.total:.12e}")
