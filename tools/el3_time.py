"""Config 4 (128^3 Kuhn): elastic 3D multigrid-PCG solves on a loaded state (graph mode, warm
start from zero), REPS timed solves after one warm-up."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1511_08463_b200 as pf
from paper_1511_08463_b200 import solver as S

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
reps = int(os.environ.get("REPS", "5"))
setup = pf.setup_traction3d(n=n)
prob = setup.problem
st = pf.State.zeros(setup.mesh)
t = float(setup.schedule[4])
setup.apply_load(prob, st, t)
st.u[prob._bc_dofs_dev] = prob._bc_vals_dev
cfg = pf.SolverConfig(elastic_solver="cg", elastic_rtol=1e-8, elastic_precond="gmg", warm_start=False,
                      gmg_degree=int(os.environ.get("DEG", "2")))
S.elastic_step(st, prob, cfg)
torch.cuda.synchronize(); t0 = time.perf_counter()
for _ in range(reps):
    _, kit = S.elastic_step(st, prob, cfg)
torch.cuda.synchronize()
print(f"3D elastic cold-start solve {1e3*(time.perf_counter()-t0)/reps:.3f} ms its={kit}")
