"""SENT (config 2): march to a loaded step, then time the AM phase and the Newton phase of one
load step separately (wall, eager) and with per-class kernel profiling."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1511_08463_b200 as pf
from paper_1511_08463_b200 import solver as S
from bench import read_profile

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
k = int(sys.argv[2]) if len(sys.argv) > 2 else 8
setup = pf.setup_sent(n=n)
prob = setup.problem
cfg = pf.SolverConfig(method="oram_newton", omega=1.8, outer_atol=1e-6, am_switch_atol=1e-3,
                      elastic_solver="cg", elastic_rtol=1e-8, elastic_precond="gmg",
                      max_am_iterations=2000, fieldsplit_inner="mg")
st = pf.State.zeros(setup.mesh, setup.initial_alpha_lb)
pf.run_quasistatic(setup, cfg, snapshot_stride=0, state=st, steps=list(range(k)))


def prep():
    s = st.copy()
    t = float(setup.schedule[k])
    s.load = t
    s.alpha_lb = s.alpha.clone()
    setup.apply_load(prob, s, t)
    s.u[prob._bc_dofs_dev] = prob._bc_vals_dev
    S._snap_bc(s, prob)
    return s


def show(tag):
    p = read_profile(prob)
    tot = sum(v["ms"] for v in p.values())
    print(f"[{tag}] kernel ms={tot:.2f}")
    for name, v in sorted(p.items(), key=lambda kv: -kv[1]["ms"]):
        print(f"   {name:10s} n={int(v['count']):6d} ms={v['ms']:8.3f} avg_us={1e3*v['ms']/v['count']:7.2f}"
              f" GB/s={v['bytes']/(v['ms']*1e-3)/1e9 if v['ms'] else 0:7.1f}")


for prof in (0, 1):
    prob.call("pf_profile", prof)
    s = prep()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    am = S.am_solve(s, prob, cfg, rtol=cfg.am_rtol, cycle=0)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    print(f"profile={prof} AM its={am.am_iterations} kry={am.total_krylov_iterations} wall={1e3*(t1-t0):.1f} ms")
    if prof:
        show("AM")
    ns, nr = S.coupled_newton_solve(s, prob, cfg)
    torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"profile={prof} Newton its={nr.iterations} kry={nr.total_krylov_iterations} conv={nr.converged} "
          f"wall={1e3*(t2-t1):.1f} ms")
    if prof:
        show("Newton")
prob.call("pf_profile", 0)
