"""Trace one SENT load step (bench sent_config): AM residuals, Newton residual histories, MINRES
counts (PF_NEWTON_TRACE=1 prints the inner detail to stderr).

    python tools/sent_step_trace.py [--n 512] [--step 18] [--save-before]
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

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=512)
ap.add_argument("--step", type=int, default=18)
ap.add_argument("--save-before", action="store_true")
ap.add_argument("--atol", type=float, default=None)
args = ap.parse_args()

setup = pf.setup_sent(n=args.n)
cfg = bench.sent_config(pf)
st = pf.State.zeros(setup.mesh, setup.initial_alpha_lb)
pf.run_quasistatic(setup, cfg, snapshot_stride=0, state=st, steps=list(range(args.step)))
torch.cuda.synchronize()
if args.save_before:
    os.makedirs("gpurun_out", exist_ok=True)
    np.savez(f"gpurun_out/sent{args.n}_state{args.step - 1}.npz", u=st.u.cpu().numpy(),
             alpha=st.alpha.cpu().numpy(), alpha_lb=st.alpha_lb.cpu().numpy(),
             load=float(setup.schedule[args.step - 1]))
log = []


def cb(d):
    log.append(d)
    if d["phase"] == "am":
        print(f"  am c{d['cycle']} it{d['iteration']:4d} res={d['residual']:.3e} wbar={d['omega_bar']:.3f} "
              f"E=({d['elastic']:.9e},{d['dissipated']:.9e})", flush=True)
    else:
        print(f"  newton c{d['cycle']} it{d['iteration']:3d} res={d['residual']:.3e}", flush=True)


if args.atol is not None:
    cfg.outer_atol = args.atol
cfg.log_callback = cb
t0 = time.perf_counter()
r = pf.run_quasistatic(setup, cfg, snapshot_stride=0, state=st, steps=[args.step])[0]
torch.cuda.synchronize()
print(f"step {args.step}: {time.perf_counter() - t0:.3f} s AM={r.report.am_iterations} "
      f"N={r.report.newton_iterations}/{r.report.newton_attempts} kry={r.report.total_krylov_iterations} "
      f"E={tuple(r.energy)}")
