"""3D damage half-step (masked VI, persistent Jacobi-PCG k_pcg_kaa3) on a loaded 128^3 config-4
state: one warm-up solve, then REPS timed solves (for ncu captures of the persistent kernel)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1511_08463_b200 as pf
from paper_1511_08463_b200 import solver as S

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
reps = int(os.environ.get("REPS", "3"))
setup = pf.setup_traction3d(n=n)
prob = setup.problem
st = pf.State.zeros(setup.mesh)
t = float(setup.schedule[12])
setup.apply_load(prob, st, t)
st.u[prob._bc_dofs_dev] = prob._bc_vals_dev
cfg = pf.SolverConfig(elastic_solver="cg", elastic_rtol=1e-8, elastic_precond="gmg")
u, _ = S.elastic_step(st, prob, cfg)
st.u = u
S.damage_step(st, prob, cfg)
torch.cuda.synchronize(); t0 = time.perf_counter()
for _ in range(reps):
    a, rep = S.damage_step(st, prob, cfg)
torch.cuda.synchronize()
print(f"3D damage step {1e3*(time.perf_counter()-t0)/reps:.3f} ms vi_its={rep.iterations} krylov={rep.total_krylov_iterations} max_alpha={float(a.max()):.3e}")
