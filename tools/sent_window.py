"""SENT 512^2 (config 2, bench.py's sent_config): every schedule step with its time, AM / Newton /
Krylov counts and the split into elastic, damage and Newton phases.

    python tools/sent_window.py [--n 512] [--steps 60] [--save 9,10] [--out gpurun_out/sent_window.json]

Pass 1 times every step with CUDA events (no extra syncs, the bench's own measurement).  Pass 2
replays from the same start with synchronised wrappers around the half-steps to attribute time.
``--save k,...`` writes the device state after step k (u, alpha, alpha_lb, load) to
gpurun_out/sent{n}_state{k}.npz -- the input of the full-size step-local parity check.
"""
import argparse
import json
import os
import sys
import time
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
import paper_1511_08463_b200 as pf
from paper_1511_08463_b200 import solver as S

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=512)
ap.add_argument("--steps", type=int, default=60)
ap.add_argument("--save", default="")
ap.add_argument("--out", default="gpurun_out/sent_window.json")
ap.add_argument("--no-split", action="store_true")
ap.add_argument("--cheb-deg", type=int, default=0, help="override fieldsplit_cheb_degree")
ap.add_argument("--workload", default="sent", choices=["sent", "traction3d", "thermal"])
ap.add_argument("--save-dir", default="gpurun_out")
args = ap.parse_args()
save = {int(s) for s in args.save.split(",") if s}
os.makedirs("gpurun_out", exist_ok=True)

if args.workload == "sent":
    setup = pf.setup_sent(n=args.n)
    cfg = bench.sent_config(pf)
elif args.workload == "thermal":   # config 3: --n is ny, the slab is 4 n x n cells
    setup = pf.setup_thermal_slab(nx=4 * args.n, ny=args.n)
    cfg = bench.thermal_config(pf)
else:
    setup = pf.setup_traction3d(n=args.n)
    cfg = bench.traction3d_config(pf)
args.steps = min(args.steps, len(setup.schedule))
if args.cheb_deg:
    cfg.fieldsplit_cheb_degree = args.cheb_deg
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float64, device="cuda")


def plain_pass():
    st = pf.State.zeros(setup.mesh, setup.initial_alpha_lb)
    rows = []
    for k in range(args.steps):
        flush.add_(1.0)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        r = pf.run_quasistatic(setup, cfg, snapshot_stride=0, state=st, steps=[k])[0]
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        rep = r.report
        rows.append({"step": k, "load": r.load, "ms": round(ms, 3), "am": rep.am_iterations,
                     "newton": rep.newton_iterations, "newton_attempts": rep.newton_attempts,
                     "krylov": rep.total_krylov_iterations,
                     "E": [r.energy.elastic, r.energy.dissipated, r.energy.total],
                     "amax": float(st.alpha.max())})
        print(f"step {k:3d} t={r.load:.2e} {ms:8.1f} ms AM={rep.am_iterations:4d} "
              f"N={rep.newton_iterations:3d}/{rep.newton_attempts} kry={rep.total_krylov_iterations:6d} "
              f"E=({r.energy.elastic:.6e},{r.energy.dissipated:.6e}) amax={rows[-1]['amax']:.3f}",
              flush=True)
        if k in save:
            np.savez_compressed(f"{args.save_dir}/{args.workload}{args.n}_state{k}.npz", u=st.u.cpu().numpy(),
                     alpha=st.alpha.cpu().numpy(), alpha_lb=st.alpha_lb.cpu().numpy(), load=r.load,
                     E=np.array(rows[-1]["E"]), am=rep.am_iterations)
    return rows


def split_pass(rows):
    acc = defaultdict(lambda: [0, 0.0, 0])
    orig = {}
    for name in ("elastic_step", "damage_step", "coupled_newton_solve"):
        f = getattr(S, name)
        orig[name] = f

        def wrap(*a, _f=f, _n=name, **kw):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            r = _f(*a, **kw)
            torch.cuda.synchronize()
            acc[_n][0] += 1
            acc[_n][1] += time.perf_counter() - t0
            if _n == "elastic_step":
                acc[_n][2] += r[1]
            else:
                acc[_n][2] += r[1].total_krylov_iterations
            return r
        setattr(S, name, wrap)
    st = pf.State.zeros(setup.mesh, setup.initial_alpha_lb)
    for k in range(args.steps):
        acc.clear()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        pf.run_quasistatic(setup, cfg, snapshot_stride=0, state=st, steps=[k])
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        sp = {n: {"calls": c, "ms": round(1e3 * t, 2), "krylov": it} for n, (c, t, it) in acc.items()}
        rows[k]["split"] = sp
        rows[k]["split_wall_ms"] = round(1e3 * wall, 2)
        print(f"step {k:3d} wall {1e3 * wall:7.1f} ms  " + "  ".join(
            f"{n[:8]}: {v['calls']}x {v['ms']:.1f} ms ({v['krylov']} its)" for n, v in sp.items()),
            flush=True)
    for n, f in orig.items():
        setattr(S, n, f)


rows = plain_pass()
if not args.no_split:
    split_pass(rows)
win = [r["ms"] for r in rows[5:25]] if args.workload == "sent" else [r["ms"] for r in rows[5:]]
summary = {"n": args.n, "steps": args.steps, "rows": rows,
           "driver_window_5_24_s_per_step": (sum(win) / len(win) / 1e3) if win else None,
           "all_steps_s_per_step": sum(r["ms"] for r in rows) / len(rows) / 1e3}
with open(args.out, "w") as f:
    json.dump(summary, f)
print(json.dumps({k: v for k, v in summary.items() if k != "rows"}))
