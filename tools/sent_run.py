"""Run the SENT (config 2) schedule on the device; per-step timing and iteration counts."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1511_08463_b200 as pf

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
nsteps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
atol = float(sys.argv[3]) if len(sys.argv) > 3 else 1e-6
stride = int(sys.argv[4]) if len(sys.argv) > 4 else 1
setup = pf.setup_sent(n=n)
cfg = pf.SolverConfig(method="oram_newton", omega=1.8, outer_atol=atol, am_switch_atol=1e-3,
                      elastic_solver="cg", elastic_rtol=1e-8, elastic_precond="gmg",
                      max_am_iterations=2000)
st = pf.State.zeros(setup.mesh, setup.initial_alpha_lb)
t_all = time.perf_counter()
steps = list(range(0, len(setup.schedule), stride))[:nsteps]
for k in steps:
    torch.cuda.synchronize(); t0 = time.perf_counter()
    recs = pf.run_quasistatic(setup, cfg, snapshot_stride=0, state=st, steps=[k])
    torch.cuda.synchronize(); t1 = time.perf_counter()
    r = recs[0]
    print(f"step {k:3d} t={r.load:.2e} {1e3*(t1-t0):8.1f} ms AM={r.report.am_iterations:4d} "
          f"N={r.report.newton_iterations:3d}/{r.report.newton_attempts} kry={r.report.total_krylov_iterations:6d} "
          f"res={r.report.final_residual_norm:.2e} E=({r.energy.elastic:.6e},{r.energy.dissipated:.6e}) "
          f"amax={float(st.alpha.max()):.3f}", flush=True)
print(f"total {time.perf_counter()-t_all:.1f} s launches={setup.problem.launches()}")
