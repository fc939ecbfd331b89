"""Elastic GMG-PCG on a loaded SENT state: iterations and time vs Chebyshev degree."""
import os, sys, time, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1511_08463_b200 as pf
from paper_1511_08463_b200 import _lib, solver as S
n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
setup = pf.setup_sent(n=n)
prob = setup.problem
cfg = pf.SolverConfig(method="oram_newton", omega=1.8, outer_atol=1e-6, am_switch_atol=1e-3,
                      elastic_solver="cg", elastic_rtol=1e-8, elastic_precond="gmg")
st = pf.State.zeros(setup.mesh, setup.initial_alpha_lb)
pf.run_quasistatic(setup, cfg, snapshot_stride=0, state=st, steps=list(range(10)))
out = torch.empty_like(st.u)
for deg in [int(x) for x in os.environ.get('DEGS', '2,3,4,5').split(',')]:
    for reuse in (1,):
        opts = S._lin_opts(cfg, False)
        opts.cheb_degree = deg
        opts.gmg_reuse = reuse
        r = _lib.LinReport()
        prob.call("pf_elastic_solve", _lib.ptr(st.alpha), _lib.ptr(st.u), _lib.ptr(out), C.byref(opts), C.byref(r), pf.fem._stream())
        torch.cuda.synchronize(); t0 = time.perf_counter()
        for _ in range(5):
            prob.call("pf_elastic_solve", _lib.ptr(st.alpha), _lib.ptr(st.u), _lib.ptr(out), C.byref(opts), C.byref(r), pf.fem._stream())
        torch.cuda.synchronize()
        print(f"deg={deg} reuse={reuse} its={r.iterations} {1e3*(time.perf_counter()-t0)/5:.3f} ms")
