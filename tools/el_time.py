"""Elastic GMG-PCG solve timing on a loaded SENT state: repeated cold-start solves (unprofiled)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1511_08463_b200 as pf
from paper_1511_08463_b200 import solver as S
n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
setup = pf.setup_sent(n=n)
prob = setup.problem
cfg = pf.SolverConfig(elastic_solver="cg", elastic_rtol=1e-8, elastic_precond="gmg", warm_start=False)
st = pf.State.zeros(setup.mesh, setup.initial_alpha_lb)
setup.apply_load(prob, st, 3e-3)
st.u[prob._bc_dofs_dev] = prob._bc_vals_dev
S.elastic_step(st, prob, cfg)
torch.cuda.synchronize(); t0 = time.perf_counter()
REPS = int(os.environ.get("REPS", "10"))
for _ in range(REPS):
    _, kit = S.elastic_step(st, prob, cfg)
torch.cuda.synchronize()
print(f"{os.environ.get('TAG','')}: elastic cold-start solve {1e3*(time.perf_counter()-t0)/REPS:.3f} ms its={kit}")
