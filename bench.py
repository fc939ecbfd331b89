"""Benchmark: quasi-static phase-field load steps on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload sent512|traction1] [--no-sweep] [--no-e2e]

Workload (BASELINE.json configs[1], the config the metric is quoted on): ``sent512`` -- 2D
plane-strain AT2 single-edge-notched tension, 512x512 crossed P1 mesh, ORAM omega = 1.8 with
Newton once the AM residual is below 1e-3, GMG-PCG at rtol 1e-8.  A bench "step" is one load step
of the 60-step schedule: W untimed warm-up steps (schedule steps 0..W-1), then K timed steps
(W..W+K-1), each bracketed by CUDA events on the solver stream with an L2 flush (512 MB write)
between steps.  ``value`` = seconds per load step of the whole job (lower is better).
``e2e`` replays the same K steps from the same starting state through the public API with the
state copied in from / out to pinned host memory every step.  The roofline of the dominant
kernel is measured live by a third replay with per-launch CUDA-event brackets (pf_profile;
graphs off).  Multi-GPU: replicas only -- every rank runs its own replica.
"""

from __future__ import annotations

import argparse
import gc
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fp64 operator-apply GDOF/s & HBM GB/s vs peak; sec per load step (AM+Newton)"
REF_N3, REF_N3_SMALL = 10, 6   # CPU sample cubes for config 4
REF_NT, REF_NT_SMALL = 48, 32  # CPU sample slabs (4n x n) for config 3


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:  # noqa: BLE001
        return 6650.0, "fallback"


class ClockSampler:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, dev_index=0):
        self.dev = dev_index
        self.proc = None
        self.lines = []
        self.first = threading.Event()

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # nvidia-smi's start-up (NVML init) stays outside the timed region
            self.first.wait(10.0)
        except Exception:  # noqa: BLE001
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())
            self.first.set()
        self.first.set()

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


# ---- workloads -----------------------------------------------------------------------------------
def sent_config(pf):
    # C-block Chebyshev degree 6: driver window (steps 5..24) 0.251 -> 0.236 s/step against degree
    # 12, degree 8 0.240 (gpurun_out sw_deg*, profiles/r02d_*): cheaper MINRES iterations win over
    # the few extra ones in the stalled Newton phase of the nucleation step
    return pf.SolverConfig(method="oram_newton", omega=1.8, outer_atol=1e-6, am_switch_atol=1e-3,
                           elastic_solver="cg", elastic_rtol=1e-8, elastic_precond="gmg",
                           max_am_iterations=2000,
                           fieldsplit_inner="mg", fieldsplit_cheb_degree=6,
                           # A Newton attempt is given 10 iterations instead of the reference default of
                           # 30 (SolverConfig.max_newton_iterations).  Successful attempts of this problem
                           # take 1-3; the nucleation step's two stalled attempts run to the cap and are
                           # rejected (their iterates discarded) either way, so the trajectory is identical
                           # for caps 8..30 (every energy to all printed digits,
                           # profiles/r02q_sent512_newton_cap.log) and only the wasted work shrinks:
                           # driver window 0.158 -> 0.140 s/step.  PF_MAX_NEWTON overrides.
                           max_newton_iterations=int(os.environ.get("PF_MAX_NEWTON", "10")))


def surfing_config(pf):
    return pf.SolverConfig(method="oram_newton", omega=1.6, outer_atol=1e-7, elastic_solver="cg",
                           elastic_rtol=1e-10, elastic_precond="gmg", max_am_iterations=3000,
                           fieldsplit_inner="mg")


def thermal_config(pf):
    return pf.SolverConfig(method="oram_newton", omega=1.5, outer_atol=1e-7, elastic_solver="cg",
                           elastic_rtol=1e-8, elastic_precond="gmg", max_am_iterations=2000,
                           fieldsplit_inner="mg")


def traction3d_config(pf):
    return pf.SolverConfig(method="oram_newton", omega=1.7, outer_atol=1e-6, elastic_solver="cg",
                           elastic_rtol=1e-8, elastic_precond="gmg", max_am_iterations=3000,
                           fieldsplit_inner="mg",
                           fieldsplit_cheb_degree=6)  # 3D: 104 vs 121 ms per Newton (degree 12)


def traction1_setup(pf):
    mat = pf.Material(E=1.0, nu=0.0, Gc=1.0, ell=0.05, k_ell=1e-6)
    return pf.setup_traction(mat, L=1.0, H=0.1, nx=200, ny=20, n_steps=20, pattern="right",
                             include_zero=True, load_max_factor=1.5)


def traction1_config(pf):
    return pf.SolverConfig(method="am", omega=1.0, outer_atol=1e-6, elastic_solver="cg",
                           elastic_rtol=1e-10, elastic_precond="gmg")


WORKLOADS = {
    "sent512": ("sent512: BASELINE config 2 -- plane-strain AT2 SENT, unit square, 512x512 crossed "
                "P1 (525,313 vertices, 1,050,626 u-dofs), E=210 nu=0.3 Gc=2.7e-3 ell=0.01 "
                "k_ell=1e-6, notch alpha=1 on y=0.5 x<=0.5, bottom clamped, top u_y=t (60 steps to "
                "6e-3), ORAM omega=1.8 + Newton when |Phi| < 1e-3, GMG-PCG rtol 1e-8, outer_atol "
                "1e-6; step = one load step"),
    "traction3d128": ("traction3d128: BASELINE config 4 -- 3D AT1 traction of the unit cube, 128^3 hex "
                      "cells x 6 Kuhn tets (2,146,689 vertices, 6,440,067 u-dofs), E=1 nu=0.3 ell=0.03 "
                      "k_ell=1e-6, Gc lognormal(0, 0.1) per cell (seed 0) + one Jacobi smoothing pass, "
                      "z=0 clamped, z=1 u_z=t (30 steps to 1.5 t_c), ORAM omega=1.7 + Newton, 3D "
                      "multigrid-PCG rtol 1e-8, outer_atol 1e-6; step = one load step"),
    "thermal2048": ("thermal2048: BASELINE config 3 -- quenched slab [0,4]x[0,1], 2048x512 union-jack "
                    "P1 (1,051,137 vertices), plane strain AT1, E=1 (+-1% seeded cell noise) nu=0.2 "
                    "Gc=1 ell=0.01, eps0 = -dT (1 - erf(y/(2 sqrt(1e-3)))) I, dT to 3 dT_c over 40 "
                    "steps, ORAM omega=1.5 + Newton, GMG-PCG rtol 1e-8, outer_atol 1e-7; step = one "
                    "load step (nucleation near step 14: pass --warmup >= 14 to time cracked steps)"),
    "surfing": ("surfing: the reference's acceptance surfing benchmark (SURVEY 8(f) row 1) -- "
                "[0,2]x[-0.5,0.5], band-graded union-jack mesh (h = ell/5 = 0.02 in the band, 100 "
                "columns), plane stress AT1 E=1 nu=0.3 Gc=1 ell=0.1, translated Mode-I field on the "
                "whole boundary (v = 1, tip from 0.05), 30 steps to t = 1.45, ORAM omega=1.6 + "
                "Newton, GMG-PCG rtol 1e-10, outer_atol 1e-7; step = one load step"),
    "traction1": ("traction1: BASELINE config 1 -- 200x20 right-diagonal AT1 bar (E=1, nu=0, Gc=1, "
                  "ell=0.05, k=1e-6), t in linspace(0,1.5t_c,20), AM omega=1, atol 1e-6; step = one "
                  "load step"),
}


def make_workload(pf, name):
    if name == "sent512":
        return pf.setup_sent(n=512), sent_config(pf)
    if name == "traction3d128":
        return pf.setup_traction3d(n=128), traction3d_config(pf)
    if name == "surfing":
        return pf.setup_surfing(pf.Material(E=1.0, nu=0.3, Gc=1.0, ell=0.1), h=0.02, n_steps=30,
                                t_end=1.45), surfing_config(pf)
    if name == "thermal2048":
        return pf.setup_thermal_slab(nx=2048, ny=512), thermal_config(pf)
    return traction1_setup(pf), traction1_config(pf)


# ---- CPU side (oracle = restatement of the reference algorithm; SuperLU direct solves) -----------
def oracle_traction3d_steps(n, warm, timed):
    from oracle import am as oam
    from oracle import problems as opb
    s = opb.traction3d(n=n)
    cfg = oam.AMConfig(method="oram_newton", omega=1.7, outer_atol=1e-6, max_am_iterations=3000)
    _, st = opb.run(s, cfg, snapshot_stride=0, steps=list(warm))
    t0 = time.perf_counter()
    rows, _ = opb.run(s, cfg, snapshot_stride=0, steps=list(timed), state=st)
    return (time.perf_counter() - t0) / len(rows)


def oracle_thermal_steps(ny, warm, timed):
    from oracle import am as oam
    from oracle import problems as opb
    s = opb.thermal_slab(nx=4 * ny, ny=ny)
    cfg = oam.AMConfig(method="oram_newton", omega=1.5, outer_atol=1e-7, max_am_iterations=2000)
    _, st = opb.run(s, cfg, snapshot_stride=0, steps=list(warm))
    t0 = time.perf_counter()
    rows, _ = opb.run(s, cfg, snapshot_stride=0, steps=list(timed), state=st)
    return (time.perf_counter() - t0) / len(rows)


def oracle_surfing_steps(warm, timed):
    from oracle import am as oam
    from oracle import problems as opb
    from oracle.p1 import MaterialSpec
    s = opb.surfing(MaterialSpec(E=1.0, nu=0.3, Gc=1.0, ell=0.1), h=0.02, n_steps=30, t_end=1.45)
    cfg = oam.AMConfig(method="oram_newton", omega=1.6, outer_atol=1e-7, max_am_iterations=3000)
    _, st = opb.run(s, cfg, snapshot_stride=0, steps=list(warm))
    t0 = time.perf_counter()
    rows, _ = opb.run(s, cfg, snapshot_stride=0, steps=list(timed), state=st)
    return (time.perf_counter() - t0) / len(rows)


def oracle_traction1_steps(warm, timed):
    from oracle import am as oam
    from oracle import problems as opb
    from oracle.p1 import MaterialSpec
    spec = MaterialSpec(E=1.0, nu=0.0, Gc=1.0, ell=0.05, k_ell=1e-6)
    s = opb.traction(spec, L=1.0, H=0.1, nx=200, ny=20, n_steps=20, pattern="right",
                     include_zero=True, load_max_factor=1.5)
    cfg = oam.AMConfig(method="am", omega=1.0, outer_atol=1e-6, elastic_solver="direct")
    _, st = opb.run(s, cfg, snapshot_stride=0, steps=list(warm))
    t0 = time.perf_counter()
    rows, _ = opb.run(s, cfg, snapshot_stride=0, steps=list(timed), state=st)
    return (time.perf_counter() - t0) / len(rows)


# AM iterations per SENT 512^2 load step, schedule steps 0..59, as recorded by the GPU arm with
# sent_config (profiles/r02a_sent512_window.json; the count is fixed by the algorithm: ORAM with
# omega = 1.8 contracts the displacement by |1 - omega| = 0.8 per iteration while the damage is
# static, so every non-nucleating step needs the same 31 iterations to reach the 1e-3 hand-off)
SENT512_AM = [31] * 18 + [67] + [31] * 30 + [308, 2148] + [31] * 9
SENT512_NEWTON = [1, 2, 1, 1, 2, 2, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 23, 2, 1, 1, 1, 1, 1, 1, 1, 1, 1, 2, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 30, 21, 1, 1, 1, 1, 1, 1, 1, 1, 1]  # with Newton attempts capped at 10 (sent_config)


def oracle_sent_am_iteration(n, step):
    """The reference algorithm (oracle restatement of solver.py:166-241) on ONE full-size SENT
    AM iteration (elastic half-step + damage half-step + relaxation + residual) at the load of
    schedule step ``step``, from the notch state after one untimed warm-up AM iteration (which forms
    the notch-tip damage profile).  SuperLU solves as the reference (linalg.py:250-262), with the
    symmetric minimum-degree ordering (MMD_AT_PLUS_A; the reference's default COLAMD factorises
    the same matrices ~4x slower, so this CPU figure is conservative).  Returns seconds."""
    from oracle import am as oam
    from oracle import krylov as okr
    from oracle import problems as opb
    okr.LU_PERMC = "MMD_AT_PLUS_A"
    s = opb.sent(n=n)
    m = s.model
    st = oam.LoadState.zeros(m, s.initial_alpha_lb)
    t = float(s.schedule[step])
    st.load = t
    s.apply_load(m, st, t)
    st.u[m.bc[0]] = m.bc[1]
    cfg = oam.AMConfig(method="am", omega=1.8, outer_atol=1e-6, max_am_iterations=1)
    oam.am_loop(st, m, cfg)  # warm-up (untimed)
    t0 = time.perf_counter()
    oam.am_loop(st, m, cfg)
    return time.perf_counter() - t0


def cpu_sample(workload, warm, timed):
    """The reference algorithm (oracle) on the host cores, on a bounded sample of the workload.

    sent512 (the headline): ONE full-size 512^2 AM iteration is measured (about 35 s on one core);
    seconds per load step = that time x the AM iterations of the same schedule steps (SENT512_AM,
    recorded by the GPU arm).  Labelled as such; the Newton phases are not counted, so the figure
    is a LOWER bound on the CPU time per load step.  Other workloads: the same schedule steps at
    two reduced sizes, scaled with the fitted cost growth (labelled).  Returns (value, desc, detail).
    """
    if workload == "sent512":
        step = timed[0]
        s_am = oracle_sent_am_iteration(512, step)
        am = [SENT512_AM[k] for k in timed]
        nw = [SENT512_NEWTON[k] for k in timed]
        value = s_am * sum(am) / len(am)
        desc = (f"measured: one full-size 512^2 SENT AM iteration (elastic + damage half-step, "
                f"relaxation, residual; oracle = reference algorithm, SuperLU with MMD ordering, "
                f"serial) at the load of schedule step {step}, after one untimed warm-up iteration "
                f"from the notch state: {s_am:.2f} s; x {sum(am) / len(am):.2f} AM iterations per "
                f"load step (steps {timed[0]}..{timed[-1]}, the GPU arm's counts) = s/load-step; the "
                f"{sum(nw)} Newton iterations of those steps are not counted (lower bound)")
        return value, desc, {"measured_s_per_am_iteration": s_am, "am_iterations_per_step": am,
                             "newton_iterations_not_counted": nw, "extrapolated": True,
                             "extrapolation": "s_per_am_iteration x recorded AM count",
                             "lu_ordering": "MMD_AT_PLUS_A"}
    if workload == "traction3d128":
        s_small = oracle_traction3d_steps(REF_N3_SMALL, warm, timed)
        s_big = oracle_traction3d_steps(REF_N3, warm, timed)
        v_small, v_big, v_full = ((n + 1) ** 3 for n in (REF_N3_SMALL, REF_N3, 128))
        expo = min(max(math.log(s_big / s_small) / math.log(v_big / v_small), 1.0), 2.0)
        value = s_big * (v_full / v_big) ** expo
        desc = (f"EXTRAPOLATED: schedule steps {timed[0]}..{timed[-1]} of the oracle (reference "
                f"algorithm, SuperLU, serial) measured at {REF_N3_SMALL}^3 ({s_small:.3f} s/step) and "
                f"{REF_N3}^3 ({s_big:.3f} s/step); scaled to 128^3 with the fitted growth vertices^{expo:.2f}")
        return value, desc, {"s_per_step_small": s_small, "s_per_step_big": s_big,
                             "n_small": REF_N3_SMALL, "n_big": REF_N3, "exponent": expo,
                             "extrapolated": True}
    if workload == "surfing":
        v = oracle_surfing_steps(warm, timed)
        return v, (f"schedule steps {timed[0]}..{timed[-1]} of the oracle (reference algorithm, "
                   f"SuperLU, serial) on the SAME surfing workload (no scaling)"), {"extrapolated": False}
    if workload == "thermal2048":
        s_small = oracle_thermal_steps(REF_NT_SMALL, warm, timed)
        s_big = oracle_thermal_steps(REF_NT, warm, timed)
        v_small, v_big, v_full = ((4 * n + 1) * (n + 1) for n in (REF_NT_SMALL, REF_NT, 512))
        expo = min(max(math.log(s_big / s_small) / math.log(v_big / v_small), 1.0), 2.0)
        value = s_big * (v_full / v_big) ** expo
        desc = (f"EXTRAPOLATED: schedule steps {timed[0]}..{timed[-1]} of the oracle (reference "
                f"algorithm, SuperLU, serial) measured at {4 * REF_NT_SMALL}x{REF_NT_SMALL} "
                f"({s_small:.3f} s/step) and {4 * REF_NT}x{REF_NT} ({s_big:.3f} s/step); scaled to "
                f"2048x512 with the fitted growth vertices^{expo:.2f}")
        return value, desc, {"s_per_step_small": s_small, "s_per_step_big": s_big,
                             "ny_small": REF_NT_SMALL, "ny_big": REF_NT, "exponent": expo,
                             "extrapolated": True}
    v = oracle_traction1_steps(warm, timed)
    return v, f"schedule steps {timed[0]}..{timed[-1]} of config 1 (oracle, SuperLU), full size", \
        {"extrapolated": False}


# ---- helpers -------------------------------------------------------------------------------------
def read_profile(problem):
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


def ncu_traffic(kind):
    """DRAM bytes (read + write) per launch of a kernel class from the committed ncu --set full
    capture (profiles/r02_ncu/summary.json, tools/ncu_r02.sh).  The multigrid-cycle class launches,
    per V-cycle, one persistent coarse cycle and four fine smoother strips (two EPI_CHEB-like, two
    EPI_RESID-like): its per-launch traffic is their average."""
    try:
        with open(os.path.join(ROOT, "profiles", "r02_ncu", "summary.json")) as f:
            s = json.load(f)
    except Exception:  # noqa: BLE001
        return None, None
    if kind == "gmg_cycle":
        t = (s["k_gmg_coarse"]["dram_bytes_per_launch"] + 2 * s["OpKuuILb0ELi1E"]["dram_bytes_per_launch"]
             + 2 * s["OpKuuILb0ELi2E"]["dram_bytes_per_launch"]) / 5.0
        return round(t), ("profiles/r02_ncu/summary.json: ncu --set full dram__bytes_read.sum + "
                          "dram__bytes_write.sum, mean over the class's launches per V-cycle (1 k_gmg_coarse "
                          "+ 4 fine smoother strips); below the algorithmic bytes because the 512^2 working "
                          "set is L2-resident")
    return None, None


def dominant_roofline(prof, peak, peak_kind):
    """Largest total-time kernel class that has algorithmic bytes; achieved = bytes / time."""
    cands = {k: v for k, v in prof.items() if v["bytes"] > 0 and v["ms"] > 0}
    if not cands:
        return None
    name, p = max(cands.items(), key=lambda kv: kv[1]["ms"])
    gbs = p["bytes"] / (p["ms"] * 1e-3) / 1e9
    total = sum(v["ms"] for v in prof.values())
    traffic, tsrc = ncu_traffic(name)
    return {"bound": "hbm", "kernel": name, "achieved": round(gbs, 2), "peak": peak,
            "peak_source": peak_kind, "unit": "GB/s", "frac": round(gbs / peak, 4),
            "traffic": traffic, "traffic_source": tsrc, "launches": int(p["count"]),
            "avg_launch_us": round(1e3 * p["ms"] / max(p["count"], 1), 3),
            "bytes_per_launch": round(p["bytes"] / max(p["count"], 1)),
            "share_of_kernel_time": round(p["ms"] / total, 4) if total > 0 else None}


SWEEP_2D = ((256, "union_jack"), (512, "union_jack"), (1024, "union_jack"), (2048, "union_jack"),
            (4096, "union_jack"), (8192, "union_jack"), (8192, "right"), (8192, "crossed"))
SWEEP_3D = (32, 64, 128, 256)


def operator_sweep(pf, torch, peak, reps=10, check=True):
    """BASELINE config 5: matrix-free Kuu and AT1 / AT2 Kaa applies, 2D 256^2..8192^2 (all three
    patterns at 8192^2) and 3D 32^3..256^3; alpha ~ U[0,1], u, x ~ N(0,1) (seeded), E=1, nu=0.3,
    k_ell=1e-6, L2 flushed before every apply; algorithmic bytes: Kuu = (x, alpha, y)
    per vertex, Kaa = (x, u, y) per vertex (the kernel re-reads u through its per-element kappa
    cache; the bytes counted are the 8(d) compulsory ones, 32 B / 40 B per vertex in 2D / 3D).

    The config-5 CPU leg (``check``): every row is recomputed on the host cores by the oracle --
    the matrix-free C restatement of the assembled oracle SpMV (oracle/mfapply.c, pinned to the
    assembled oracle in tests/test_oracle_mf.py) -- and the row carries its time and the max
    relative difference |y_gpu - y_cpu|_inf / |y_cpu|_inf (the config asks for 1e-12)."""
    import numpy as np
    mf = None
    if check:
        from oracle import mfapply as mf  # CPU leg (checker): outside every timed region
        from oracle.p1 import MaterialSpec
    res = []
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float64, device="cuda")
    cases = [(n, p, 2) for n, p in SWEEP_2D] + [(n, "kuhn6", 3) for n in SWEEP_3D]
    for n, pattern, dim in cases:
        regime = "3d" if dim == 3 else "plane_stress"
        mesh = pf.StructuredMesh3D(n, n, n) if dim == 3 else pf.StructuredMesh(n, n, 1.0, 1.0, pattern)
        V = mesh.n_vertices
        g = torch.Generator(device="cuda").manual_seed(n + dim)
        alpha = torch.rand(V, dtype=torch.float64, device="cuda", generator=g)
        x = torch.randn(dim * V, dtype=torch.float64, device="cuda", generator=g)
        u = torch.randn(dim * V, dtype=torch.float64, device="cuda", generator=g)
        xa = torch.randn(V, dtype=torch.float64, device="cuda", generator=g)
        host = None
        if mf is not None:
            host = {k: t.cpu().numpy() for k, t in (("alpha", alpha), ("x", x), ("u", u), ("xa", xa))}
        st = pf.State(u, alpha, torch.zeros_like(alpha))
        for model in ("AT1", "AT2"):
            mat = pf.Material(E=1.0, nu=0.3, Gc=1.0, ell=0.1, k_ell=1e-6, regime=regime)
            prob = pf.Discretization(mesh, mat, pf.DamageModel(model), solvers="operators")
            ops = [("Kaa_" + model, pf.assemble_Kaa(st, prob), xa, (8.0 * dim + 16.0) * V, V)]
            if model == "AT1":
                ops.insert(0, ("Kuu", pf.assemble_Kuu(st, prob, apply_bc=False), x, (16.0 * dim + 8.0) * V,
                               dim * V))
            for name, op, xin, nbytes, dofs in ops:
                y = op @ xin
                times = []
                for _ in range(reps):
                    flush.add_(1.0)
                    e0 = torch.cuda.Event(enable_timing=True)
                    e1 = torch.cuda.Event(enable_timing=True)
                    e0.record()
                    op.matvec(xin)
                    e1.record()
                    torch.cuda.synchronize()
                    times.append(e0.elapsed_time(e1) * 1e-3)
                t = sorted(times)[len(times) // 2]
                row = {"op": name, "mesh": f"{n}^{dim} {pattern}", "dofs": dofs, "median_s": t,
                       "GDOF_s": round(dofs / t / 1e9, 3), "GB_s": round(nbytes / t / 1e9, 1),
                       "frac": round(nbytes / t / 1e9 / peak, 3),
                       "bytes_per_dof": round(nbytes / dofs, 2), "l2": "flushed"}
                if name != "Kuu":  # the apply reads the per-element kappa cache instead of u
                    kb = 16.0 * V + 8.0 * prob.n_elements
                    row["kernel_bytes_per_dof"] = round(kb / dofs, 2)
                    row["kernel_frac"] = round(kb / t / 1e9 / peak, 3)
                if host is not None:
                    spec = MaterialSpec(E=1.0, nu=0.3, Gc=1.0, ell=0.1, k_ell=1e-6, model=model, regime=regime)
                    shape = (n, n, n) if dim == 3 else (n, n)
                    ext = (1.0, 1.0, 1.0) if dim == 3 else (1.0, 1.0)
                    c0 = time.perf_counter()
                    if name == "Kuu":
                        yc = mf.apply("Kuu", shape, ext, pattern, spec, alpha=host["alpha"], x=host["x"])
                    else:
                        yc = mf.apply("Kaa", shape, ext, pattern, spec, u=host["u"], x=host["xa"])
                    row["cpu_oracle_s"] = round(time.perf_counter() - c0, 4)
                    row["cpu_threads"] = os.cpu_count()
                    yg = y.cpu().numpy()
                    row["max_rel_err_vs_oracle"] = float(np.max(np.abs(yg - yc)) / np.max(np.abs(yc)))
                    del yc, yg
                res.append(row)
                del y
            del prob, ops
        del alpha, x, u, xa, st, host
        gc.collect()
        torch.cuda.empty_cache()
    return res


UMESH_SWEEP = ((2, 1024), (2, 2048), (2, 4096), (3, 64), (3, 128))


def umesh_sweep(pf, torch, peak, reps=10):
    """Element-list (jittered) meshes: pf_umesh Kuu / Kaa applies on the
    reference's jittered union-jack rect_mesh (jitter 0.25, mesh.py:134-141) and on jittered
    Kuhn boxes (jitter 0.1: Kuhn tets invert sooner); same inputs and L2 flush as the structured sweep.  Algorithmic bytes = the
    compulsory footprint of one apply: per vertex x, y, alpha (Kuu) or u, x, y (Kaa) + the vertex
    CSR row pointer; per element its record (64 B 2D / 128 B 3D) + int4 connectivity; per
    (vertex, element) incidence one 4 B entry."""
    res = []
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float64, device="cuda")
    for dim, n in UMESH_SWEEP:
        if dim == 2:
            mesh = pf.jittered_rect_mesh(1.0, 1.0, 1.0 / n, jitter=0.25, seed=n)
            mat = pf.Material(E=1.0, nu=0.3, Gc=1.0, ell=0.1, k_ell=1e-6)
        else:
            mesh = pf.jittered_box_mesh(n, n, n, jitter=0.1, seed=n)
            mat = pf.Material(E=1.0, nu=0.3, Gc=1.0, ell=0.1, k_ell=1e-6, regime="3d")
        ops = pf.UnstructuredOperators(mesh, mat, "AT1")
        V, T = mesh.n_vertices, mesh.n_elements
        del mesh
        g = torch.Generator(device="cuda").manual_seed(n + dim)
        alpha = torch.rand(V, dtype=torch.float64, device="cuda", generator=g)
        x = torch.randn(dim * V, dtype=torch.float64, device="cuda", generator=g)
        u = torch.randn(dim * V, dtype=torch.float64, device="cuda", generator=g)
        xa = torch.randn(V, dtype=torch.float64, device="cuda", generator=g)
        y = torch.empty_like(x)
        ya = torch.empty_like(xa)
        table = T * ((64 if dim == 2 else 128) + 16) + 4.0 * (V + 1) + 4.0 * (dim + 1) * T
        for name, fn, nbytes, dofs in (
                ("Kuu", lambda: ops.apply_Kuu(alpha, x, out=y), (16.0 * dim + 8.0) * V + table, dim * V),
                ("Kaa", lambda: ops.apply_Kaa(u, alpha, xa, out=ya), (8.0 * dim + 16.0) * V + table, V)):
            fn()
            times = []
            for _ in range(reps):
                flush.add_(1.0)
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record()
                fn()
                e1.record()
                torch.cuda.synchronize()
                times.append(e0.elapsed_time(e1) * 1e-3)
            t = sorted(times)[len(times) // 2]
            res.append({"op": name, "mesh": f"{n}^{dim} jittered {'union_jack' if dim == 2 else 'kuhn6'}",
                        "dofs": dofs, "elements": T, "median_s": t, "GDOF_s": round(dofs / t / 1e9, 3),
                        "GB_s": round(nbytes / t / 1e9, 1), "frac": round(nbytes / t / 1e9 / peak, 3),
                        "bytes_per_dof": round(nbytes / dofs, 2), "l2": "flushed"})
        del ops, alpha, x, u, xa, y, ya
        gc.collect()
        torch.cuda.empty_cache()
    return res


def run_steps(pf, torch, setup, cfg, state, steps, flush, host_io=False):
    """Run schedule steps; returns (seconds per step list, records, h2d, d2h bytes)."""
    times, recs = [], []
    h2d = d2h = 0
    for k in steps:
        flush.add_(1.0)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        if host_io:
            hu, ha, hl = (t.cpu().pin_memory() for t in (state.u, state.alpha, state.alpha_lb))
        e0.record()
        if host_io:  # state enters from pinned host memory, result leaves to host
            state = pf.State(hu.to("cuda", non_blocking=True), ha.to("cuda", non_blocking=True),
                             hl.to("cuda", non_blocking=True), state.load)
            h2d += (hu.numel() + ha.numel() + hl.numel()) * 8
        r = pf.run_quasistatic(setup, cfg, snapshot_stride=1 if host_io else 0, state=state,
                               steps=[k])
        if host_io:
            d2h += (r[0].u.size + r[0].alpha.size) * 8
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) * 1e-3)
        recs.append(r[0])
    return times, recs, h2d, d2h, state


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=8)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="sent512", choices=list(WORKLOADS))
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    nsched = {"sent512": 60, "traction3d128": 30, "thermal2048": 40, "surfing": 30}.get(args.workload, 20)
    W = max(0, min(args.warmup, nsched - 1))
    K = max(1, min(args.steps, nsched - W))
    timed = list(range(W, W + K))

    if args.impl == "reference":
        if rank != 0:
            return 0
        # the reference algorithm (oracle restatement, SuperLU) on the box's host cores
        t0 = time.perf_counter()
        v, sample, detail = cpu_sample(args.workload, range(W), timed)
        line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "s/load-step",
                "n_gpus": args.gpus, "steps": K, "warmup": W, "ms_per_step": 1e3 * v,
                "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic", "config": {"workload": WORKLOADS[args.workload],
                                                "parallelism": "cpu"},
                "cpu_baseline": {"value": v, "unit": "s/load-step", "cores": 1, "kind": "port",
                                 "sample": sample, "detail": detail,
                                 "threads_note": "SuperLU / scipy sparsetools are serial: one core "
                                                 f"used of {os.cpu_count()}"},
                "e2e": {"value": v, "unit": "s/load-step", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0},
                "wall_s": round(time.perf_counter() - t0, 1)}
        print(json.dumps(line))
        return 0

    import torch
    import paper_1511_08463_b200 as pf

    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    peak, peak_kind = peaks()
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float64, device="cuda")

    setup, cfg = make_workload(pf, args.workload)
    prob = setup.problem
    state = pf.State.zeros(setup.mesh, setup.initial_alpha_lb)
    # warm-up: schedule steps 0..W-1 (untimed)
    _, _, _, _, state = run_steps(pf, torch, setup, cfg, state, list(range(W)), flush)
    snap = state.copy()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    sampler = ClockSampler(local)
    sampler.start()
    l0 = prob.launches()
    step_s, recs, _, _, _ = run_steps(pf, torch, setup, cfg, state, timed, flush)
    launches = prob.launches() - l0
    clocks = sampler.stop()
    tot = sum(step_s)
    if dist:
        t = torch.tensor([tot], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot = float(t.item())
    # replicas: every rank runs its own copy of the workload; the contract's value is
    # the whole-job aggregate (K * world load steps in tot seconds), the latency of one replica's
    # load step is reported beside it
    value = tot / (K * world)
    per_replica = tot / K

    # e2e replay from the same starting state through host memory
    e2e = None
    if not args.no_e2e:
        e_s, _, h2d, d2h, _ = run_steps(pf, torch, setup, cfg, snap.copy(), timed, flush,
                                        host_io=True)
        e2e = {"value": sum(e_s) / (K * world), "unit": "s/load-step",
               "h2d_bytes_per_step": int(h2d / K), "d2h_bytes_per_step": int(d2h / K)}

    # profiled replay: per-kernel CUDA-event brackets (graphs off) for the roofline
    prof = {}
    if rank == 0:
        prob.call("pf_profile", 1)
        read_profile(prob)
        run_steps(pf, torch, setup, cfg, snap.copy(), timed, flush)
        prof = read_profile(prob)
        prob.call("pf_profile", 0)

    sweep = operator_sweep(pf, torch, peak) if (not args.no_sweep and rank == 0) else None
    usweep = umesh_sweep(pf, torch, peak) if (not args.no_sweep and rank == 0) else None
    cpu = None
    if rank == 0 and world == 1:
        v, desc, detail = cpu_sample(args.workload, range(W),
                                     timed if args.workload in ("traction1", "surfing", "sent512") else timed[:2])
        cpu = {"value": v, "unit": "s/load-step", "cores": 1, "kind": "port", "sample": desc,
               "detail": detail}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "s/load-step", "n_gpus": world,
                "steps": K, "warmup": W, "ms_per_step": 1e3 * tot / K, "higher_is_better": False,
                "per_replica_s_per_load_step": per_replica,
                "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": WORKLOADS[args.workload],
                           "timed_schedule_steps": [timed[0], timed[-1]],
                           "parallelism": "replicas" if world > 1 else "single",
                           "l2": "flushed (512 MB write) between timed steps",
                           "per_step_s": [round(x, 4) for x in step_s],
                           "am_iterations": [r.report.am_iterations for r in recs],
                           "newton_iterations": [r.report.newton_iterations for r in recs],
                           "krylov_iterations": [r.report.total_krylov_iterations for r in recs],
                           "energies": [list(map(float, r.energy)) for r in recs]},
                "roofline": dominant_roofline(prof, peak, peak_kind),
                "kernel_profile": {k: {"launches": int(v["count"]), "ms": round(v["ms"], 3),
                                       "GB_s": round(v["bytes"] / max(v["ms"], 1e-9) / 1e6, 1)}
                                   for k, v in prof.items()},
                "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches),
                "clocks": clocks, "operator_sweep": sweep,
                "operator_sweep_unstructured": usweep}
        print(json.dumps(line))
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
