"""Elastic GMG-PCG solve on a loaded SENT state vs the Chebyshev smoother degree (graph mode,
hierarchy reused; best of 5 cold-start solves)."""
import os, sys, time, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1511_08463_b200 as pf
from paper_1511_08463_b200 import _lib

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
setup = pf.setup_sent(n=n)
prob = setup.problem
st = pf.State.zeros(setup.mesh, setup.initial_alpha_lb)
setup.apply_load(prob, st, 3e-3)
cfg = pf.SolverConfig(elastic_solver="cg", elastic_rtol=1e-8, elastic_precond="gmg", warm_start=False)
out = torch.empty_like(st.u)
for deg in [int(a) for a in sys.argv[2:]] or [1, 2, 3, 4]:
    opts = pf.solver._lin_opts(cfg, False)
    opts.cheb_degree = deg
    best = 1e9
    for rep in range(6):
        r = _lib.LinReport()
        torch.cuda.synchronize(); t0 = time.perf_counter()
        prob.call("pf_elastic_solve", _lib.ptr(st.alpha), _lib.ptr(st.u), _lib.ptr(out), C.byref(opts), C.byref(r), pf.fem._stream())
        torch.cuda.synchronize(); dt = time.perf_counter() - t0
        if rep > 0: best = min(best, dt)
    print(f"deg={deg} its={r.iterations} best wall={1e3*best:.3f} ms  per it={1e3*best/max(r.iterations,1):.3f} ms")
