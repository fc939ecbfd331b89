"""Full-size step-local parity: the device state after step k-1 is the input
of ONE load step k, run on the device (GPU box) and on the CPU oracle (here, any length of time),
then compared (north-star bars: energies 1e-6 relative, max|d alpha| 1e-4).

    # GPU box: state k-1 -> device step k at parity tolerances; writes <dir>/<tag>_dev{k}.npz
    python tools/steplocal.py device --state gpurun_out/sent512_state9.npz --step 10
    # build container: the oracle from the same input; writes <dir>/<tag>_ora{k}.npz
    ORACLE_LU_PERMC=MMD_AT_PLUS_A python tools/steplocal.py oracle --state ... --step 10
    python tools/steplocal.py compare --state ... --step 10     # prints / writes the JSON summary

Parity settings (SURVEY 8(c) rule): outer_atol 1e-9 on both sides, device elastic PCG rtol 1e-12,
damage VI abs_tol 0.1 outer_atol; everything else is config 2 (bench.sent_config: ORAM omega 1.8,
Newton hand-off at |Phi| < 1e-3, multigrid field split).  The oracle solves directly (SuperLU).
``--workload traction3d`` runs config 4 (the 3D problem at --n cells per side), ``--workload
thermal`` config 3 (the quenched slab, 4 n x n cells).
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np

ap = argparse.ArgumentParser()
ap.add_argument("mode", choices=["device", "oracle", "compare"])
ap.add_argument("--state", required=True)
ap.add_argument("--step", type=int, required=True)
ap.add_argument("--workload", default="sent", choices=["sent", "traction3d", "thermal"])
ap.add_argument("--n", type=int, default=512)
ap.add_argument("--atol", type=float, default=1e-9)
ap.add_argument("--literal", action="store_true", help="config-literal tolerances instead")
ap.add_argument("--outdir", default="gpurun_out/steplocal")
ap.add_argument("--oracle-cg", action="store_true",
                help="oracle elastic half-steps by Jacobi-PCG at rtol 1e-13 instead of SuperLU (3D sizes)")
args = ap.parse_args()
d = args.outdir
os.makedirs(d, exist_ok=True)
tag = f"{args.workload}{args.n}_{'lit' if args.literal else 'par'}"
dev_path = os.path.join(d, f"{tag}_dev{args.step}.npz")
ora_path = os.path.join(d, f"{tag}_ora{args.step}.npz")
s0 = np.load(args.state)


def run_device():
    import torch
    import bench
    import paper_1511_08463_b200 as pf
    if args.workload == "sent":
        setup, cfg = pf.setup_sent(n=args.n), bench.sent_config(pf)
    elif args.workload == "thermal":
        setup, cfg = pf.setup_thermal_slab(nx=4 * args.n, ny=args.n), bench.thermal_config(pf)
    else:
        setup, cfg = pf.setup_traction3d(n=args.n), bench.traction3d_config(pf)
    if not args.literal:
        cfg.outer_atol = args.atol
        cfg.elastic_rtol = 1e-12
    st = pf.State.from_numpy(s0["u"], s0["alpha"], s0["alpha_lb"])
    hist = []
    cfg.log_callback = lambda e: hist.append((e["phase"], e["cycle"], e["iteration"], e["residual"]))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = pf.run_quasistatic(setup, cfg, snapshot_stride=1, state=st, steps=[args.step])[0]
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    np.savez_compressed(dev_path, u=r.u, alpha=r.alpha, energy=np.array(tuple(r.energy)), load=r.load,
             am=r.report.am_iterations, newton=r.report.newton_iterations,
             attempts=r.report.newton_attempts, wall=wall,
             residual=r.report.final_residual_norm,
             hist=np.array([(0 if p == "am" else 1, c, i, x) for p, c, i, x in hist]))
    print(f"device step {args.step}: {wall:.3f} s AM={r.report.am_iterations} "
          f"N={r.report.newton_iterations}/{r.report.newton_attempts} E={tuple(r.energy)}")


def run_oracle():
    from oracle import am as oam
    from oracle import problems as opb
    if args.workload == "sent":
        s = opb.sent(n=args.n)
        cfg = oam.AMConfig(method="oram_newton", omega=1.8, outer_atol=1e-6 if args.literal else args.atol,
                           am_switch_atol=1e-3, max_am_iterations=3000)
    elif args.workload == "thermal":
        s = opb.thermal_slab(nx=4 * args.n, ny=args.n)
        cfg = oam.AMConfig(method="oram_newton", omega=1.5, outer_atol=1e-7 if args.literal else args.atol,
                           max_am_iterations=2000)
    else:
        s = opb.traction3d(n=args.n)
        cfg = oam.AMConfig(method="oram_newton", omega=1.7, outer_atol=1e-6 if args.literal else args.atol,
                           max_am_iterations=3000)
    if args.oracle_cg:
        cfg.elastic_solver, cfg.elastic_precond, cfg.elastic_rtol = "cg", "jacobi", 1e-13
        cfg.fieldsplit_inner = "cg"   # the Newton field split's elastic block by PCG too (no 3D LU of Kuu)
    hist = []

    def log(e):
        hist.append((0 if e["phase"] == "am" else 1, e["cycle"], e["iteration"], e["residual"]))
        print(f"  {e['phase']} c{e['cycle']} it{e['iteration']} res={e['residual']:.3e} "
              f"t={time.perf_counter() - t0:.0f}s", flush=True)
    cfg.log = log
    st = oam.LoadState(s0["u"].copy(), s0["alpha"].copy(), s0["alpha_lb"].copy(), float(s0["load"]))
    t0 = time.perf_counter()
    rows, _ = opb.run(s, cfg, snapshot_stride=1, steps=[args.step], state=st)
    r = rows[0]
    wall = time.perf_counter() - t0
    np.savez(ora_path, u=r.u, alpha=r.alpha,
             energy=np.array([r.energy.elastic, r.energy.dissipated, r.energy.total]), load=r.load,
             am=r.stats.am_iterations, newton=r.stats.newton_iterations,
             attempts=r.stats.newton_attempts, wall=wall, residual=r.stats.final_residual_norm,
             hist=np.array(hist), lu=os.environ.get("ORACLE_LU_PERMC", "COLAMD"))
    print(f"oracle step {args.step}: {wall:.1f} s AM={r.stats.am_iterations} "
          f"N={r.stats.newton_iterations}/{r.stats.newton_attempts} E={tuple(r.energy)}")


def compare():
    a, b = np.load(dev_path), np.load(ora_path)
    ea, eb = a["energy"], b["energy"]
    rel = np.abs(ea - eb) / np.abs(eb)
    out = {"workload": args.workload, "n": args.n, "step": args.step, "load": float(b["load"]),
           "input": os.path.basename(args.state),
           "settings": "config-literal (outer_atol 1e-6)" if args.literal else
           f"parity (outer_atol {args.atol:g}, device elastic rtol 1e-12, oracle SuperLU)",
           "energy_device": ea.tolist(), "energy_oracle": eb.tolist(),
           "energy_rel_diff": {"elastic": rel[0], "dissipated": rel[1], "total": rel[2]},
           "alpha_max_abs_diff": float(np.max(np.abs(a["alpha"] - b["alpha"]))),
           "u_max_abs_diff_rel": float(np.max(np.abs(a["u"] - b["u"])) / np.max(np.abs(b["u"]))),
           "device": {"am": int(a["am"]), "newton": int(a["newton"]), "attempts": int(a["attempts"]),
                      "wall_s": float(a["wall"]), "residual": float(a["residual"])},
           "oracle": {"am": int(b["am"]), "newton": int(b["newton"]), "attempts": int(b["attempts"]),
                      "wall_s": float(b["wall"]), "residual": float(b["residual"]),
                      "lu_ordering": str(b["lu"]) if "lu" in b.files else "MMD_AT_PLUS_A"}}
    out["pass"] = bool(rel.max() <= 1e-6 and out["alpha_max_abs_diff"] <= 1e-4)
    print(json.dumps(out, indent=1))
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", f"r02_steplocal_{tag}_step{args.step}.json"), "w") as f:
        json.dump(out, f, indent=1)


{"device": run_device, "oracle": run_oracle, "compare": compare}[args.mode]()
