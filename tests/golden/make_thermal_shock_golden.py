"""Golden trajectory of the reference's own thermal-shock case (cases.py:195-235), produced by
running the REFERENCE package itself (the element-list path's parity target).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_thermal_shock_golden.py

Case defaults (L = 20, H = 10, ell = 1, h = ell/4: the jittered 80 x 40 union-jack rect_mesh,
plane-stress AT1), a 12-step geometric tau schedule, dT = 2 dT_c so that the periodic crack
pattern forms inside the schedule; alternate minimisation (method am, omega = 1, direct solves) at
outer_atol 1e-8 (the SURVEY 8(c) parity setting).  Writes tests/golden/ref_thermal_shock.npz.
"""

import os
import sys
import time

import numpy as np

REF = os.environ.get("PHASEFRAC_REF", "/root/reference/pkg/src")
sys.path.insert(0, REF)

from phasefrac import cases, solver  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
STEPS, DT_FACTOR, ATOL = 12, 2.0, 1e-8


def main():
    s = cases.setup_thermal_shock(n_steps=STEPS, dT_factor=DT_FACTOR)
    cfg = solver.SolverConfig(method="am", outer_atol=ATOL)
    t0 = time.perf_counter()
    recs = cases.run_quasistatic(s, cfg)
    print(f"{time.perf_counter() - t0:.1f} s")
    np.savez_compressed(os.path.join(OUT, "ref_thermal_shock.npz"), steps=STEPS, dT_factor=DT_FACTOR, atol=ATOL,
                        load=np.array([r.load for r in recs]),
                        energy=np.array([[r.energy.elastic, r.energy.dissipated, r.energy.total] for r in recs]),
                        alpha=np.array([r.alpha for r in recs]),
                        am=np.array([r.report.am_iterations for r in recs]),
                        vertices=s.problem.mesh.vertices)


if __name__ == "__main__":
    main()
