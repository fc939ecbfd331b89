"""GMG vs Jacobi PCG on the SENT (config 2) elastic half-step: iterations and time."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1511_08463_b200 as pf

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
setup = pf.setup_sent(n=n)
prob = setup.problem
st = pf.State.zeros(setup.mesh, setup.initial_alpha_lb)
setup.apply_load(prob, st, 3e-3)
for precond, deg in (("jacobi", 2), ("gmg", 2), ("gmg", 3), ("gmg", 4)):
    cfg = pf.SolverConfig(elastic_solver="cg", elastic_rtol=1e-8, elastic_precond=precond, warm_start=False)
    opts = pf.solver._lin_opts(cfg, False)
    opts.cheb_degree = deg
    import ctypes as C
    from paper_1511_08463_b200 import _lib
    out = torch.empty_like(st.u)
    for rep in range(2):
        r = _lib.LinReport()
        torch.cuda.synchronize(); t0 = time.perf_counter()
        prob.call("pf_elastic_solve", _lib.ptr(st.alpha), _lib.ptr(st.u), _lib.ptr(out), C.byref(opts),
                  C.byref(r), pf.fem._stream())
        torch.cuda.synchronize(); t1 = time.perf_counter()
    print(f"n={n} {precond:6s} deg={deg}: its={r.iterations:5d} res={r.final_residual_norm:.3e} "
          f"b={r.b_norm:.3e} time={1e3*(t1-t0):.1f} ms launches={prob.launches()}")
