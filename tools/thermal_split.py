"""Config 3 (thermal slab 2048x512): time split of the cracked load steps (elastic / damage /
Newton calls, synchronised) and the Newton attempts of ORAM-N."""
import os, sys, time
from collections import defaultdict
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1511_08463_b200 as pf
from paper_1511_08463_b200 import solver as S
import bench

k0 = int(sys.argv[1]) if len(sys.argv) > 1 else 16
setup, cfg = pf.setup_thermal_slab(nx=2048, ny=512), bench.thermal_config(pf)
cfg.damage_forcing = bool(int(os.environ.get("FORCING", "1")))
st = pf.State.zeros(setup.mesh, setup.initial_alpha_lb)
pf.run_quasistatic(setup, cfg, snapshot_stride=0, state=st, steps=list(range(k0)))
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
            log.append((dt, r[1].iterations, r[1].total_krylov_iterations, r[1].converged))
        return r
    setattr(S, name, wrap)
torch.cuda.synchronize(); t0 = time.perf_counter()
recs = pf.run_quasistatic(setup, cfg, snapshot_stride=0, state=st, steps=[k0])
torch.cuda.synchronize(); tot = time.perf_counter() - t0
r = recs[0].report
print(f"forcing={cfg.damage_forcing} E={recs[0].energy.total:.12e} step {k0}: {1e3*tot:.1f} ms  AM its {r.am_iterations} newton its {r.newton_iterations} attempts {r.newton_attempts}")
for name, (c, t) in acc.items():
    print(f"  {name:22s} calls={c:4d} total={1e3*t:8.1f} ms  per call={1e3*t/max(c,1):7.3f} ms")
for row in log:
    print("  newton: %.1f ms its=%d kry=%d conv=%s" % (1e3 * row[0], *row[1:]))
