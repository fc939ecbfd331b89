"""Benchmark: quasi-static phase-field load steps on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload traction1|sent512] [--sweep/--no-sweep]

A bench "step" is one pass of the hot path over one batch of synthetic input: for
``traction1`` (BASELINE config 1) one full 20-load-step quasi-static run; for ``sent512``
(BASELINE config 2) one load step of the SENT schedule.  ``value`` is seconds per load step
of the whole job (lower is better), timed with CUDA events on the solver stream (max over
ranks), inputs resident in HBM; ``e2e`` is the same metric through the public API with the
state coming from / going to pinned host memory every load step.  The dominant kernel's
roofline is measured live (library CUDA-event brackets, pf_profile) over the timed region.
Multi-GPU: replicas only (each rank runs an independent replica).
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fp64 operator-apply GDOF/s & HBM GB/s vs peak; sec per load step (AM+Newton)"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:  # noqa: BLE001
        return 6650.0, "fallback"


# ---- clocks sampler ----------------------------------------------------------------------------
class ClockSampler:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, dev_index=0):
        self.dev = dev_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:  # noqa: BLE001
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:  # noqa: BLE001
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for k, n in enumerate(names):
                if f[5 + k] == "Active":
                    reasons.add(n)
        sm.sort()
        med = sm[len(sm) // 2] if sm else None
        return {"sm_mhz": med, "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def flush_l2(buf):
    buf.add_(1.0)  # 512 MB write > 126 MB L2


# ---- workloads -----------------------------------------------------------------------------------
def traction1_setup(pf):
    mat = pf.Material(E=1.0, nu=0.0, Gc=1.0, ell=0.05, k_ell=1e-6)
    return pf.setup_traction(mat, L=1.0, H=0.1, nx=200, ny=20, n_steps=20, pattern="right",
                             include_zero=True, load_max_factor=1.5)


def traction1_config(pf):
    return pf.SolverConfig(method="am", omega=1.0, outer_atol=1e-6, elastic_solver="cg",
                           elastic_rtol=1e-10)


def oracle_traction1():
    from oracle import am as oam
    from oracle import problems as opb
    from oracle.p1 import MaterialSpec
    spec = MaterialSpec(E=1.0, nu=0.0, Gc=1.0, ell=0.05, k_ell=1e-6)
    s = opb.traction(spec, L=1.0, H=0.1, nx=200, ny=20, n_steps=20, pattern="right",
                     include_zero=True, load_max_factor=1.5)
    return s, oam.AMConfig(method="am", omega=1.0, outer_atol=1e-6, elastic_solver="direct")


def run_oracle_traction1(reps=1):
    from oracle import problems as opb
    t0 = time.perf_counter()
    n = 0
    for _ in range(reps):
        s, cfg = oracle_traction1()
        rows, _ = opb.run(s, cfg, snapshot_stride=0)
        n += len(rows)
    return time.perf_counter() - t0, n


def dominant_roofline(prof, peak, peak_kind):
    """Pick the kernel class with the largest total time; achieved = alg bytes / time."""
    best = max(prof.items(), key=lambda kv: kv[1]["ms"]) if prof else None
    if not best or best[1]["ms"] <= 0:
        return None
    name, p = best
    gbs = p["bytes"] / (p["ms"] * 1e-3) / 1e9
    total = sum(v["ms"] for v in prof.values())
    return {"bound": "hbm", "kernel": name, "achieved": round(gbs, 2), "peak": peak,
            "peak_source": peak_kind, "unit": "GB/s", "frac": round(gbs / peak, 4),
            "traffic": None, "launches": int(p["count"]),
            "avg_launch_us": round(1e3 * p["ms"] / max(p["count"], 1), 3),
            "bytes_per_launch": p["bytes"] / max(p["count"], 1),
            "share_of_kernel_time": round(p["ms"] / total, 4) if total > 0 else None}


def read_profile(problem, lib):
    import ctypes as C
    from paper_1511_08463_b200 import _lib
    n = len(_lib.KERNEL_KINDS)
    buf = (C.c_double * (3 * n))()
    problem.call("pf_profile_read", buf, n)
    out = {}
    for k, name in enumerate(_lib.KERNEL_KINDS):
        if buf[3 * k] > 0:
            out[name] = {"count": buf[3 * k], "ms": buf[3 * k + 1], "bytes": buf[3 * k + 2]}
    return out


def operator_sweep(pf, torch, peak, sizes=(1024, 4096, 8192), reps=10):
    """Config 5: matrix-free Kuu / Kaa applies, cold L2 (flush between reps)."""
    import numpy as np
    res = []
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float64, device="cuda")
    for n in sizes:
        mat = pf.Material(E=1.0, nu=0.3, Gc=1.0, ell=0.1, k_ell=1e-6)
        mesh = pf.StructuredMesh(n, n, 1.0, 1.0, "union_jack")
        prob = pf.Discretization(mesh, mat, pf.DamageModel("AT1"))
        V = mesh.n_vertices
        g = torch.Generator(device="cuda").manual_seed(n)
        alpha = torch.rand(V, dtype=torch.float64, device="cuda", generator=g)
        x = torch.randn(2 * V, dtype=torch.float64, device="cuda", generator=g)
        u = torch.randn(2 * V, dtype=torch.float64, device="cuda", generator=g)
        xa = torch.randn(V, dtype=torch.float64, device="cuda", generator=g)
        st = pf.State(u, alpha, torch.zeros_like(alpha))
        K = pf.assemble_Kuu(st, prob, apply_bc=False)
        A = pf.assemble_Kaa(st, prob)
        for name, op, xin, bpv in (("Kuu", K, x, 40.0), ("Kaa", A, xa, None)):
            y = op @ xin
            times = []
            for _ in range(reps):
                flush_l2(flush)
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record()
                op.matvec(xin)
                e1.record()
                torch.cuda.synchronize()
                times.append(e0.elapsed_time(e1) * 1e-3)
            t = sorted(times)[len(times) // 2]
            if name == "Kuu":
                nbytes = V * 40.0
                dofs = 2 * V
            else:
                # pf_apply_Kaa = kappa pass (u -> kappa, c) + apply; report the apply share only
                nbytes = V * 16.0 + prob.n_elements * 8.0
                dofs = V
            res.append({"op": name, "n": n, "dofs": dofs, "median_s": t,
                        "GDOF_s": round(dofs / t / 1e9, 3), "GB_s": round(nbytes / t / 1e9, 1),
                        "frac": round(nbytes / t / 1e9 / peak, 3),
                        "bytes_per_dof": round(nbytes / dofs, 2)})
            del y
        del prob
        torch.cuda.empty_cache()
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="traction1", choices=["traction1"])
    ap.add_argument("--no-sweep", action="store_true")
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        if rank != 0:
            return 0
        os.environ.setdefault("OPENBLAS_NUM_THREADS", str(os.cpu_count()))
        for _ in range(args.warmup):
            run_oracle_traction1(1)
        t, n = run_oracle_traction1(args.steps)
        v = t / n
        line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "s/load-step",
                "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": 1e3 * t / args.steps, "higher_is_better": False,
                "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": "traction1: BASELINE config 1, 200x20 right-diagonal AT1 "
                           "bar, 20 load steps, AM omega=1, atol 1e-6",
                           "parallelism": "cpu"},
                "cpu_baseline": {"value": v, "unit": "s/load-step", "cores": 1, "kind": "port",
                                 "sample": f"{args.steps} full config-1 runs ({n} load steps) of "
                                           "the oracle restatement (SuperLU direct, as the "
                                           "reference's default path)"},
                "e2e": {"value": v, "unit": "s/load-step", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        return 0

    import numpy as np
    import torch
    import paper_1511_08463_b200 as pf
    from paper_1511_08463_b200 import _lib

    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    peak, peak_kind = peaks()

    setup = traction1_setup(pf)
    cfg = traction1_config(pf)
    prob = setup.problem
    nsteps_run = len(setup.schedule)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float64, device="cuda")

    def one_run(snap=0):
        return pf.run_quasistatic(setup, cfg, snapshot_stride=snap)

    for _ in range(args.warmup):
        one_run()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    sampler = ClockSampler(local)
    sampler.start()
    prob.call("pf_profile", 1)
    l0 = prob.launches()
    step_s = []
    its = []
    for _ in range(args.steps):
        flush_l2(flush)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        recs = one_run()
        e1.record()
        torch.cuda.synchronize()
        step_s.append(e0.elapsed_time(e1) * 1e-3)
        its.append(sum(r.report.am_iterations for r in recs))
    launches = prob.launches() - l0
    prof = read_profile(prob, None)
    prob.call("pf_profile", 0)
    clocks = sampler.stop()
    tot = sum(step_s)
    if dist:
        t = torch.tensor([tot], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot = float(t.item())
    # replicas: every rank runs its own replica concurrently; the job processed
    # world * steps * nsteps_run load steps in `tot` seconds (max over ranks)
    value = tot / (args.steps * nsteps_run * world)

    # e2e: same runs through the public API with host-resident state in / out each load step
    V = setup.mesh.n_vertices
    h2d = 0
    e2e_s = []
    for _ in range(max(1, args.steps)):
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        host_u = torch.zeros(2 * V, dtype=torch.float64).pin_memory()
        host_a = torch.zeros(V, dtype=torch.float64).pin_memory()
        st = pf.State(host_u.to("cuda", non_blocking=True), host_a.to("cuda", non_blocking=True),
                      host_a.to("cuda", non_blocking=True))
        recs = pf.run_quasistatic(setup, cfg, snapshot_stride=1, state=st)
        e1.record()
        torch.cuda.synchronize()
        e2e_s.append(e0.elapsed_time(e1) * 1e-3)
    h2d = (2 * V + 2 * V) * 8 / nsteps_run + sum(
        16 * len(setup.problem.bc.dofs) for _ in range(1))
    d2h = 3 * V * 8
    e2e = {"value": sum(e2e_s) / (len(e2e_s) * nsteps_run), "unit": "s/load-step",
           "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)}

    sweep = None
    if not args.no_sweep and rank == 0:
        sweep = operator_sweep(pf, torch, peak)

    cpu = None
    if rank == 0 and world == 1:
        t_cpu, n_cpu = run_oracle_traction1(1)
        cpu = {"value": t_cpu / n_cpu, "unit": "s/load-step", "cores": 1, "kind": "port",
               "sample": f"one full config-1 run ({n_cpu} load steps) of the oracle restatement "
                         "(SuperLU direct elastic solves, LU-based rsls) on this host"}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "s/load-step", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
                "higher_is_better": False, "scaling": "weak", "vs_baseline": None,
                "dtype": "f64", "data": "synthetic",
                "config": {"workload": "traction1: BASELINE config 1, 200x20 right-diagonal AT1 "
                           "bar (E=1, nu=0, Gc=1, ell=0.05, k=1e-6), t in linspace(0,1.5t_c,20), "
                           "AM omega=1, atol 1e-6; one step = one full 20-load-step run",
                           "parallelism": "replicas" if world > 1 else "single",
                           "l2": "flushed (512 MB write) between timed steps",
                           "am_iterations_per_run": its[-1] if its else None},
                "roofline": dominant_roofline(prof, peak, peak_kind),
                "kernel_profile": {k: {"launches": int(v["count"]), "ms": round(v["ms"], 3),
                                       "GB_s": round(v["bytes"] / max(v["ms"], 1e-9) / 1e6, 1)}
                                   for k, v in prof.items()},
                "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches),
                "clocks": clocks, "operator_sweep": sweep}
        print(json.dumps(line))
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
