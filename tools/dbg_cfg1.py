import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1511_08463_b200 as pf
os.environ["PF_STRIP2"] = sys.argv[1]
mat = pf.Material(E=1.0, nu=0.0, Gc=1.0, ell=0.05, k_ell=1e-6)
setup = pf.setup_traction(mat, L=1.0, H=0.1, nx=100, ny=10, n_steps=8, pattern="right")
recs = pf.run_quasistatic(setup, pf.SolverConfig(outer_atol=1e-8))
print(sys.argv[1], os.environ.get("PF_STRIP2_KINDS"), [tuple(round(x, 9) for x in r.energy) for r in recs[5:6]], recs[5].report.am_iterations if hasattr(recs[5].report,'am_iterations') else recs[5].report)
