"""Multigrid-PCG convergence on SENT-like states for each 2D pattern (cold starts, rtol 1e-8)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1511_08463_b200 as pf
from paper_1511_08463_b200 import solver as S
n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
for pattern in ("crossed", "union_jack", "right"):
    setup = pf.setup_sent(n=n, pattern=pattern)
    prob = setup.problem
    cfg = pf.SolverConfig(method="oram_newton", omega=1.8, outer_atol=1e-6, am_switch_atol=1e-3,
                          elastic_solver="cg", elastic_rtol=1e-8, elastic_precond="gmg")
    st = pf.State.zeros(setup.mesh, setup.initial_alpha_lb)
    pf.run_quasistatic(setup, cfg, snapshot_stride=0, state=st, steps=list(range(8)))
    c2 = pf.SolverConfig(**{**cfg.__dict__, "warm_start": False, "gmg_reuse": False})
    _, kit = S.elastic_step(st, prob, c2)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    _, kit = S.elastic_step(st, prob, c2)
    torch.cuda.synchronize()
    print(f"{pattern:10s} its={kit} rho={1e-8 ** (1.0 / kit):.3f} {1e3 * (time.perf_counter() - t0):.2f} ms", flush=True)
