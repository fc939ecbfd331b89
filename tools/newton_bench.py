"""Time the Newton phase of SENT 512^2 step 18 (the nucleation step of the driver's window) under
environment toggles, to attribute the MINRES cost.  Input: the device state after step 17
(steplocal_in/sent512_state17.npz).  The AM phase of step 18 runs once up to the hand-off; then
the coupled Newton solve is timed from that state with each variant (PF_NEWTON_NO_KEEP=1 so every
call builds its own hierarchy and all variants see the same start).

    python tools/newton_bench.py [--reps 2]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
import paper_1511_08463_b200 as pf
from paper_1511_08463_b200 import solver as S

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--state", default="steplocal_in/sent512_state17.npz")
ap.add_argument("--step", type=int, default=18)
ap.add_argument("--only", default="")
ap.add_argument("--workload", default="sent", choices=["sent", "traction3d"])
ap.add_argument("--n", type=int, default=512)
args = ap.parse_args()
os.environ["PF_NEWTON_NO_KEEP"] = "1"
s0 = np.load(args.state)
if args.workload == "sent":
    setup, mkcfg = pf.setup_sent(n=args.n), bench.sent_config
else:
    setup, mkcfg = pf.setup_traction3d(n=args.n), bench.traction3d_config
cfg = mkcfg(pf)
st = pf.State.from_numpy(s0["u"], s0["alpha"], s0["alpha_lb"])
t = float(setup.schedule[args.step])
st.load = t
st.alpha_lb = st.alpha.clone()
setup.apply_load(setup.problem, st, t)
st.u[setup.problem._bc_dofs_dev] = setup.problem._bc_vals_dev
rep = S.am_solve(st, setup.problem, cfg, rtol=cfg.am_rtol, cycle=0)
if os.environ.get("PF_NEWTON_TRACE"):
    pass
print(f"AM to hand-off: {rep.am_iterations} its, residual {rep.final_residual_norm:.3e}", flush=True)
VARIANTS = {
    "default": {},
    "no_stall_keep": {"PF_NEWTON_NO_STALL_KEEP": "1"},
    "cold_minres": {"PF_MINRES_COLD": "1"},
    "host_minres": {"PF_NEWTON_HOST_MINRES": "1"},
    "cheb_deg12": {"__deg": 12},
    "cheb_deg3": {"__deg": 3},
    "cheb_deg4": {"__deg": 4},
    "cheb_deg8": {"__deg": 8},
    "multiplicative": {"__mult": 1},
    "inner_direct": {"__inner": "direct"},          # A, C blocks solved to fieldsplit_rtol
    "coupled_direct": {"__coupled": "direct"},      # MINRES at direct_rtol (the LU stand-in)
    "mg_rtol1e-8": {"__fsrtol": 1e-8},              # the mg split, MINRES to 1e-8
    "no_forcing": {"__noforce": 1},                 # MINRES at fieldsplit_rtol every iteration
}
for name, env in VARIANTS.items():
    if args.only and name not in args.only.split(","):
        continue
    c = mkcfg(pf)
    for k, v in env.items():
        if k == "__deg":
            c.fieldsplit_cheb_degree = v
        elif k == "__mult":
            c.fieldsplit_additive = False
        elif k == "__inner":
            c.fieldsplit_inner = v
        elif k == "__coupled":
            c.coupled_solver = v
        elif k == "__fsrtol":
            c.fieldsplit_rtol = v
        elif k == "__noforce":
            c.newton_forcing = False
        else:
            os.environ[k] = v
    ts = []
    for _ in range(args.reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ns, nr = S.coupled_newton_solve(st, setup.problem, c)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    for k in env:
        if not k.startswith("__"):
            os.environ.pop(k, None)
    print(f"{name:12s} {min(ts) * 1e3:9.1f} ms  newton its {nr.iterations:3d} krylov {nr.total_krylov_iterations:6d} "
          f"-> {1e6 * min(ts) / max(1, nr.total_krylov_iterations):.2f} us/krylov  res {nr.final_residual_norm:.3e}",
          flush=True)
