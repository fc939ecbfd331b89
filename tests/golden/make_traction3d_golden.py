"""Golden trajectories of BASELINE config 4 (3D traction, lognormal Gc) at reduced size, from the
CPU oracle (oracle/problems.py ``traction3d``; the reference package is 2D-only, so the oracle's 3D
Kuhn path is pinned by finite differences in tests/test_oracle_fd.py and shares every formula with
the reference-pinned 2D path).

Same physics as config 4 at 12^3 hex cells x 6 Kuhn tets: AT1, E=1, nu=0.3, Gc lognormal(0, 0.1)
per cell (seed 0) + one Jacobi smoothing pass, z=0 clamped, z=1 u_z = t with t over 12 steps up to
1.5 t_c; the length scale is scaled with the mesh (ell = 0.03 * 128 / 12, ell/h = 3.84 as at 128^3).
ORAM omega = 1.7 + Newton, oracle solves direct (SuperLU).  The crack runs through at step 7.
Two tolerance settings: parity (outer_atol 1e-9) and config-literal (1e-6).

    python tests/golden/make_traction3d_golden.py   # writes tests/golden/oracle_traction3d12.npz (~5 min)
"""

from __future__ import annotations

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
N, STEPS = 12, 12
ELL = 0.03 * 128 / N


def run(atol):
    spec = MaterialSpec(E=1.0, nu=0.3, Gc=1.0, ell=ELL, k_ell=1e-6, model="AT1", regime="3d")
    s = opb.traction3d(n=N, spec=spec, n_steps=STEPS)
    cfg = oam.AMConfig(method="oram_newton", omega=1.7, outer_atol=atol, max_am_iterations=3000)
    t0 = time.perf_counter()
    rows, _ = opb.run(s, cfg, snapshot_stride=1)
    print(f"atol {atol:g}: {time.perf_counter() - t0:.1f} s", flush=True)
    return {"load": np.array([r.load for r in rows]),
            "energy": np.array([[r.energy.elastic, r.energy.dissipated, r.energy.total] for r in rows]),
            "alpha": np.array([r.alpha for r in rows]),
            "am": np.array([r.stats.am_iterations for r in rows]),
            "newton": np.array([r.stats.newton_iterations for r in rows])}


def main():
    out = {"n": N, "steps": STEPS, "ell": ELL}
    for tag, atol in (("parity", 1e-9), ("literal", 1e-6)):
        for k, v in run(atol).items():
            out[f"{tag}_{k}"] = v
    np.savez_compressed(os.path.join(OUT, f"oracle_traction3d{N}.npz"), **out)


if __name__ == "__main__":
    main()
