"""Run the thermal-slab (config 3) schedule on the device; per-step timing and counts."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1511_08463_b200 as pf

nx = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
ny = int(sys.argv[2]) if len(sys.argv) > 2 else 512
nsteps = int(sys.argv[3]) if len(sys.argv) > 3 else 40
setup = pf.setup_thermal_slab(nx=nx, ny=ny)
cfg = pf.SolverConfig(method="oram_newton", omega=1.5, outer_atol=1e-7, elastic_solver="cg",
                      elastic_rtol=1e-8, elastic_precond="gmg", max_am_iterations=2000)
st = pf.State.zeros(setup.mesh)
t_all = time.perf_counter()
for k in range(min(nsteps, len(setup.schedule))):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    r = pf.run_quasistatic(setup, cfg, snapshot_stride=0, state=st, steps=[k])[0]
    torch.cuda.synchronize(); t1 = time.perf_counter()
    print(f"step {k:3d} dT={r.load:.4f} {1e3*(t1-t0):8.1f} ms AM={r.report.am_iterations:4d} "
          f"N={r.report.newton_iterations:3d}/{r.report.newton_attempts} kry={r.report.total_krylov_iterations:6d} "
          f"res={r.report.final_residual_norm:.2e} E=({r.energy.elastic:.6e},{r.energy.dissipated:.6e}) "
          f"amax={float(st.alpha.max()):.3f}", flush=True)
print(f"total {time.perf_counter()-t_all:.1f} s")
