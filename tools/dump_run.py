"""Debug: run the 8-step golden traction case on the device, save per-step alpha."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1511_08463_b200 as pf

mat = pf.Material(E=1.0, nu=0.3, Gc=1.0, ell=0.1, k_ell=1e-6)
setup = pf.setup_traction(mat, L=1.0, H=0.3, nx=20, ny=6, n_steps=8)
hist = []
cfg = pf.SolverConfig(outer_atol=1e-9, log_callback=lambda d: hist.append(d))
recs = pf.run_quasistatic(setup, cfg)
np.savez("gpurun_out/dump_run.npz", alpha=np.array([r.alpha for r in recs]),
         E=np.array([list(r.energy) for r in recs]), its=np.array([r.report.am_iterations for r in recs]),
         res=np.array([h["residual"] for h in hist]), tot=np.array([h["total"] for h in hist]))
print("its", [r.report.am_iterations for r in recs])
