"""SENT (config 2): where the time of a load step goes -- wall time of every elastic_step,
damage_step and coupled_newton_solve call (synchronised), summed over one load step."""
import os, sys, time
from collections import defaultdict
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1511_08463_b200 as pf
from paper_1511_08463_b200 import solver as S

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
k = int(sys.argv[2]) if len(sys.argv) > 2 else 8
setup = pf.setup_sent(n=n)
cfg = pf.SolverConfig(method="oram_newton", omega=1.8, outer_atol=1e-6, am_switch_atol=1e-3,
                      elastic_solver="cg", elastic_rtol=1e-8, elastic_precond="gmg",
                      max_am_iterations=2000, fieldsplit_inner="mg",
                      gmg_degree=int(os.environ.get("DEG", "2")),
                      damage_forcing=bool(int(os.environ.get("FORCING", "1"))),
                      fieldsplit_rtol=float(os.environ.get("FSRTOL", "1e-6")))
st = pf.State.zeros(setup.mesh, setup.initial_alpha_lb)
pf.run_quasistatic(setup, cfg, snapshot_stride=0, state=st, steps=list(range(k)))
acc = defaultdict(lambda: [0, 0.0])
for name in ("elastic_step", "damage_step", "coupled_newton_solve"):
    f = getattr(S, name)
    def wrap(*a, _f=f, _n=name, **kw):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        r = _f(*a, **kw)
        torch.cuda.synchronize(); acc[_n][0] += 1; acc[_n][1] += time.perf_counter() - t0
        return r
    setattr(S, name, wrap)
torch.cuda.synchronize(); t0 = time.perf_counter()
pf.run_quasistatic(setup, cfg, snapshot_stride=0, state=st, steps=[k, k + 1])
torch.cuda.synchronize(); tot = time.perf_counter() - t0
print(f"2 load steps ({k},{k+1}): {1e3*tot:.1f} ms  E {st.alpha.sum().item():.12e}")
for name, (c, t) in acc.items():
    print(f"  {name:22s} calls={c:4d} total={1e3*t:8.1f} ms  per call={1e3*t/max(c,1):7.3f} ms")
