"""Config 4 (traction3d, 128^3): where the time of load steps goes -- wall time of every
elastic_step, damage_step and coupled_newton_solve (synchronised), per inner mode of Newton."""
import os, sys, time
from collections import defaultdict
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1511_08463_b200 as pf
from paper_1511_08463_b200 import solver as S

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
k = int(sys.argv[2]) if len(sys.argv) > 2 else 4
inner = sys.argv[3] if len(sys.argv) > 3 else "direct"
setup = pf.setup_traction3d(n=n)
cfg = pf.SolverConfig(method="oram_newton", omega=1.7, outer_atol=1e-6, elastic_solver="cg",
                      elastic_rtol=1e-8, elastic_precond="gmg", max_am_iterations=3000,
                      fieldsplit_inner=inner,
                      fieldsplit_additive=bool(int(os.environ.get("ADDITIVE", "1"))),
                      damage_forcing=bool(int(os.environ.get("FORCING", "1"))),
                      fieldsplit_cheb_degree=int(os.environ.get("CDEG", "6")),
                      gmg_degree=int(os.environ.get("DEG", "2")))
st = pf.State.zeros(setup.mesh)
pf.run_quasistatic(setup, cfg, snapshot_stride=0, state=st, steps=list(range(k)))
acc = defaultdict(lambda: [0, 0.0])
log = []
for name in ("elastic_step", "damage_step", "coupled_newton_solve"):
    f = getattr(S, name)
    def wrap(*a, _f=f, _n=name, **kw):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        r = _f(*a, **kw)
        torch.cuda.synchronize(); dt = time.perf_counter() - t0
        acc[_n][0] += 1; acc[_n][1] += dt
        if _n == "coupled_newton_solve":
            log.append((dt, r[1].iterations, r[1].total_krylov_iterations, r[1].converged, r[1].final_residual_norm))
        return r
    setattr(S, name, wrap)
torch.cuda.synchronize(); t0 = time.perf_counter()
try:
    pf.run_quasistatic(setup, cfg, snapshot_stride=0, state=st, steps=[k, k + 1])
except Exception as e:  # noqa: BLE001
    print("FAILED:", e)
torch.cuda.synchronize(); tot = time.perf_counter() - t0
print(f"deg={cfg.gmg_degree} inner={inner} add={cfg.fieldsplit_additive} forcing={cfg.damage_forcing} 2 load steps ({k},{k+1}): {1e3*tot:.1f} ms")
for name, (c, t) in acc.items():
    print(f"  {name:22s} calls={c:4d} total={1e3*t:8.1f} ms  per call={1e3*t/max(c,1):7.3f} ms")
for row in log:
    print("  newton: %.1f ms its=%d kry=%d conv=%s res=%.3e" % (1e3 * row[0], *row[1:]))
