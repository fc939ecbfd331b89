"""Device vs host MINRES in the Newton phase (debugging aid): PF_NEWTON_TRACE per mode."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1511_08463_b200 as pf
from paper_1511_08463_b200 import solver as S
setup = pf.setup_traction(pf.Material(ell=0.1), nx=40, ny=12, n_steps=12, pattern="right")
base = pf.SolverConfig(method="am", elastic_solver="cg", elastic_precond="gmg", outer_atol=1e-3)
st = pf.State.zeros(setup.mesh)
pf.run_quasistatic(setup, base, snapshot_stride=0, state=st, steps=list(range(9)))
cfg = pf.SolverConfig(outer_atol=1e-9, elastic_solver="cg", elastic_precond="gmg", fieldsplit_inner="mg")
os.environ["PF_NEWTON_TRACE"] = "1"
for mode in ("host", "eager", "graph"):
    os.environ.pop("PF_NEWTON_HOST_MINRES", None); os.environ.pop("PF_MR_EAGER", None)
    if mode == "host": os.environ["PF_NEWTON_HOST_MINRES"] = "1"
    if mode == "eager": os.environ["PF_MR_EAGER"] = "1"
    print("=== mode", mode, file=sys.stderr, flush=True)
    s1, r1 = S.coupled_newton_solve(st, setup.problem, cfg)
    print(mode, r1.iterations, r1.converged, r1.total_krylov_iterations, r1.linear_failures, r1.residual_history, file=sys.stderr, flush=True)
