"""Golden trajectories of BASELINE config 2 (SENT) at reduced size, from the CPU oracle.

The reference package has no AT2, plane strain or crossed mesh, so config 2 cannot be run on the
reference itself; the oracle restates it (oracle/problems.py:85 ``sent``) and is pinned to the
reference by tests/test_oracle_golden.py (shared union-jack AT1 paths to 1e-12) and
tests/test_oracle_fd.py (AT2 / plane strain / crossed by finite differences).

Same physics as config 2 at a coarser mesh: n x n crossed P1, AT2 plane strain, E=210, nu=0.3,
Gc=2.7e-3, k_ell=1e-6, notch alpha_lb=1 on y=0.5, x<=0.5, bottom clamped, top u_y=t; the length
scale is scaled with the mesh (ell = 5 h, so ell/h = 5 as at 512^2 with ell = 0.01) and the load
ramp with sqrt(ell / 0.01) (the AT2 critical load scales as ell^-1/2) so the notch-tip damage grows
and the crack runs through inside the schedule.  ORAM omega=1.8 with the Newton hand-off at
|Phi| < 1e-3 (config 2), oracle solves direct (SuperLU, the reference default).

Two tolerance settings: parity (outer_atol 1e-9, the rule for comparing energies at
1e-6) and config-literal (outer_atol 1e-6, what bench.py runs).

    python tests/golden/make_sent_golden.py        # writes tests/golden/oracle_sent64.npz (~5 min)
"""

from __future__ import annotations

import math
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import am as oam  # noqa: E402
from oracle import problems as opb  # noqa: E402
from oracle.p1 import MaterialSpec  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
N, STEPS = 64, 20


def sent_params(n=N):
    ell = 5.0 / n
    return ell, 6e-3 * math.sqrt(ell / 0.01)


def run(atol):
    ell, t_max = sent_params()
    spec = MaterialSpec(E=210.0, nu=0.3, Gc=2.7e-3, ell=ell, k_ell=1e-6, model="AT2",
                        regime="plane_strain")
    s = opb.sent(n=N, spec=spec, n_steps=STEPS, t_max=t_max)
    cfg = oam.AMConfig(method="oram_newton", omega=1.8, outer_atol=atol, am_switch_atol=1e-3,
                       max_am_iterations=3000)
    t0 = time.perf_counter()
    rows, _ = opb.run(s, cfg, snapshot_stride=1)
    print(f"atol {atol:g}: {time.perf_counter() - t0:.1f} s", flush=True)
    return {"load": np.array([r.load for r in rows]),
            "energy": np.array([[r.energy.elastic, r.energy.dissipated, r.energy.total] for r in rows]),
            "alpha": np.array([r.alpha for r in rows]),
            "am": np.array([r.stats.am_iterations for r in rows]),
            "newton": np.array([r.stats.newton_iterations for r in rows])}


def main():
    out = {"n": N, "steps": STEPS, "ell": sent_params()[0], "t_max": sent_params()[1]}
    for tag, atol in (("parity", 1e-9), ("literal", 1e-6)):
        for k, v in run(atol).items():
            out[f"{tag}_{k}"] = v
    np.savez_compressed(os.path.join(OUT, f"oracle_sent{N}.npz"), **out)


if __name__ == "__main__":
    main()
