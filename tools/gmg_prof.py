"""Per-kernel-class GPU time of one GMG-PCG elastic solve on SENT (profiling on, eager)."""
import os, sys, time, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1511_08463_b200 as pf
from paper_1511_08463_b200 import _lib
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import read_profile

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
deg = int(sys.argv[2]) if len(sys.argv) > 2 else 3
setup = pf.setup_sent(n=n)
prob = setup.problem
st = pf.State.zeros(setup.mesh, setup.initial_alpha_lb)
setup.apply_load(prob, st, 3e-3)
cfg = pf.SolverConfig(elastic_solver="cg", elastic_rtol=1e-8, elastic_precond="gmg", warm_start=False)
opts = pf.solver._lin_opts(cfg, False)
opts.cheb_degree = deg
out = torch.empty_like(st.u)
for prof in (0, 1):
    prob.call("pf_profile", prof)
    r = _lib.LinReport()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    prob.call("pf_elastic_solve", _lib.ptr(st.alpha), _lib.ptr(st.u), _lib.ptr(out), C.byref(opts), C.byref(r), pf.fem._stream())
    torch.cuda.synchronize(); t1 = time.perf_counter()
    print(f"profile={prof} its={r.iterations} wall={1e3*(t1-t0):.2f} ms")
p = read_profile(prob)
tot = sum(v["ms"] for v in p.values())
for k, v in sorted(p.items(), key=lambda kv: -kv[1]["ms"]):
    print(f"  {k:10s} n={int(v['count']):5d} ms={v['ms']:8.3f} avg_us={1e3*v['ms']/v['count']:7.2f}")
print(f"  sum kernel ms={tot:.3f}")
