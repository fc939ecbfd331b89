"""Config 4 (3D AT1 traction, lognormal Gc, Kuhn tets): per-load-step time and iteration counts."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1511_08463_b200 as pf
from bench import read_profile

n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
steps = [int(s) for s in sys.argv[2].split(",")] if len(sys.argv) > 2 else [0, 10, 12]
prof = len(sys.argv) > 3 and sys.argv[3] == "prof"
prec = sys.argv[4] if len(sys.argv) > 4 else "gmg"
setup = pf.setup_traction3d(n=n)
prob = setup.problem
cfg = pf.SolverConfig(method="oram_newton", omega=1.7, outer_atol=1e-6, elastic_solver="cg",
                      elastic_rtol=1e-8, elastic_precond=prec, max_am_iterations=3000)
st = pf.State.zeros(setup.mesh, setup.initial_alpha_lb)
done = -1
for k in steps:
    if k > done + 1:
        pf.run_quasistatic(setup, cfg, snapshot_stride=0, state=st, steps=list(range(done + 1, k)))
    if prof:
        prob.call("pf_profile", 1)
        read_profile(prob)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    r = pf.run_quasistatic(setup, cfg, snapshot_stride=0, state=st, steps=[k])[0]
    torch.cuda.synchronize(); t1 = time.perf_counter()
    done = k
    print(f"n={n} step {k:2d} t={r.load:.4f} {t1-t0:8.3f} s AM={r.report.am_iterations} "
          f"N={r.report.newton_iterations}/{r.report.newton_attempts} kry={r.report.total_krylov_iterations} "
          f"E=({r.energy.elastic:.6e},{r.energy.dissipated:.6e}) amax={float(st.alpha.max()):.3f}", flush=True)
    if prof:
        p = read_profile(prob)
        prob.call("pf_profile", 0)
        tot = sum(v["ms"] for v in p.values())
        for name, v in sorted(p.items(), key=lambda kv: -kv[1]["ms"])[:8]:
            print(f"    {name:10s} n={int(v['count']):7d} ms={v['ms']:9.1f} ({v['ms']/tot:.2f}) "
                  f"GB/s={v['bytes']/(v['ms']*1e-3)/1e9:7.1f}")
