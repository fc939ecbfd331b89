"""Element-list elastic solve on a jittered union-jack mesh: Jacobi-PCG (one persistent launch) vs
PCG preconditioned by the V-cycle of the un-jittered structured twin.  usage: umesh_gmg_time.py [h]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1511_08463_b200 as pf

h = float(sys.argv[1]) if len(sys.argv) > 1 else 0.0625
setup = pf.setup_thermal_shock(n_steps=4, h=h, multigrid=True)
ops, mesh = setup.ops, setup.mesh
dofs, vals = setup.apply_load(ops, float(setup.schedule[2]))
ops.set_dirichlet(np.asarray(dofs, dtype=np.int64))
rng = np.random.default_rng(0)
V = mesh.n_vertices
a = rng.uniform(0.0, 0.3, V)
a[np.abs(mesh.vertices[:, 0] - 10.0) < 2 * h] = 1.0
alpha = torch.as_tensor(a, device="cuda")
b = torch.as_tensor(rng.standard_normal(2 * V), device="cuda")
b[torch.as_tensor(dofs, device="cuda")] = 0.0
for pre in ("jacobi", "gmg"):
    ops.elastic_solve(alpha, b, rtol=1e-8, precond=pre)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    x, r = ops.elastic_solve(alpha, b, rtol=1e-8, precond=pre)
    torch.cuda.synchronize(); t = time.perf_counter() - t0
    print(f"h={h} V={V} {pre:7s}: {1e3*t:9.2f} ms, {r.iterations} iterations, converged={r.converged}")
