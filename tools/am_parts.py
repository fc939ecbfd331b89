"""SENT (config 2): unprofiled wall time of each component of one AM iteration on a loaded state
(elastic GMG-PCG solve, damage rsls solve, relaxations, residual+energy), averaged over repeats."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1511_08463_b200 as pf
from paper_1511_08463_b200 import solver as S

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
k = int(sys.argv[2]) if len(sys.argv) > 2 else 8
setup = pf.setup_sent(n=n)
prob = setup.problem
cfg = pf.SolverConfig(method="oram_newton", omega=1.8, outer_atol=1e-6, am_switch_atol=1e-3,
                      elastic_solver="cg", elastic_rtol=1e-8, elastic_precond="gmg",
                      max_am_iterations=2000)
st = pf.State.zeros(setup.mesh, setup.initial_alpha_lb)
pf.run_quasistatic(setup, cfg, snapshot_stride=0, state=st, steps=list(range(k)))
t = float(setup.schedule[k])
st.alpha_lb = st.alpha.clone()
setup.apply_load(prob, st, t)
st.u[prob._bc_dofs_dev] = prob._bc_vals_dev


def timeit(name, fn, reps=10):
    fn()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(reps):
        r = fn()
    torch.cuda.synchronize()
    print(f"{name:28s} {1e3*(time.perf_counter()-t0)/reps:8.3f} ms  {r if isinstance(r,(int,float,str)) else ''}")


def el():
    _, kit = S.elastic_step(st, prob, cfg)
    return kit
def el_cold():
    c2 = pf.SolverConfig(**{**cfg.__dict__, "warm_start": False})
    _, kit = S.elastic_step(st, prob, c2)
    return kit
def dmg():
    _, rep = S.damage_step(st, prob, cfg)
    return f"its={rep.iterations} kry={rep.total_krylov_iterations}"
us, _ = S.elastic_step(st, prob, cfg)
ast, _ = S.damage_step(st, prob, cfg)
timeit("elastic (warm)", el)
timeit("elastic (cold)", el_cold)
timeit("damage", dmg)
timeit("relax_u", lambda: S.relax_u(st.u, us, 1.8, prob) is None)
timeit("relax_alpha", lambda: S.relax_alpha(st.alpha, ast, st.alpha_lb, 1.8, prob)[1])
timeit("residual_and_energy", lambda: S.residual_and_energy(st, prob)[0])
timeit("Kuu apply x100", lambda: [prob.call("pf_apply_Kuu", pf.fem._lib.ptr(st.alpha), pf.fem._lib.ptr(st.u), pf.fem._lib.ptr(us), 1, pf.fem._stream()) for _ in range(100)] and 0)
