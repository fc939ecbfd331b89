"""The reference's thermal-shock case on the element-list path: per-step device time (CUDA
events) and AM counts, 12 steps at 2 dT_c (the golden trajectory's settings)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1511_08463_b200 as pf
n = int(sys.argv[1]) if len(sys.argv) > 1 else 12
mg = len(sys.argv) > 2 and sys.argv[2] == "gmg"   # elastic PCG preconditioned by the structured twin's V-cycle
setup = pf.setup_thermal_shock(n_steps=n, dT_factor=2.0, multigrid=mg)
cfg = pf.SolverConfig(method="am", outer_atol=1e-8, elastic_precond="gmg" if mg else "jacobi")
V = setup.mesh.n_vertices
z = torch.zeros(V, dtype=torch.float64, device="cuda")
st = pf.State(u=torch.zeros(2 * V, dtype=torch.float64, device="cuda"), alpha=z.clone(), alpha_lb=z.clone())
tot = 0.0
for k in range(n):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    r = pf.run_quasistatic(setup, cfg, snapshot_stride=0, steps=[k], state=st)[0]
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1); tot += ms
    print(f"step {k:2d} tau={r.load:.3f} {ms:9.1f} ms AM={r.report.am_iterations:4d} "
          f"kry={r.report.total_krylov_iterations:7d} E={tuple(round(x, 6) for x in r.energy)}", flush=True)
print(f"total {tot/1e3:.2f} s, launches {setup.ops.launches}")
