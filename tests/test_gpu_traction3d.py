"""Config 4 (3D traction, lognormal Gc) parity: bench.py's traction3d configuration on the device
against the oracle at reduced size.

bench.py runs BASELINE config 4 at 128^3 with ``bench.traction3d_config`` (ORAM omega = 1.7 +
Newton, 3D multigrid PCG, multigrid field split with a degree-6 C block).  These tests run exactly
that configuration (``setup_traction3d`` + ``traction3d_config``) at 12^3 hex cells with ell scaled
to keep ell/h = 3.84, through nucleation and the crack running through (step 7 of 12), and compare
every step with the oracle trajectory in tests/golden/oracle_traction3d12.npz
(tests/golden/make_traction3d_golden.py; the reference's ORAM-N semantics, solver.py:333-387).
The lognormal Gc field breaks the cube's symmetry, so alpha is compared directly.
"""

import os

import numpy as np
import pytest

from conftest import GOLDEN, ROOT

pytestmark = pytest.mark.gpu


def _run(tag):
    import sys
    sys.path.insert(0, ROOT)
    import bench
    import paper_1511_08463_b200 as pf
    g = np.load(os.path.join(GOLDEN, "oracle_traction3d12.npz"))
    mat = pf.Material(E=1.0, nu=0.3, Gc=1.0, ell=float(g["ell"]), k_ell=1e-6, regime="3d")
    setup = pf.setup_traction3d(n=int(g["n"]), material=mat, n_steps=int(g["steps"]))
    cfg = bench.traction3d_config(pf)
    if tag == "parity":
        cfg.outer_atol = 1e-9
        cfg.elastic_rtol = 1e-12
    recs = pf.run_quasistatic(setup, cfg)
    E = np.array([tuple(r.energy) for r in recs])
    Eo = g[f"{tag}_energy"]
    A = np.array([r.alpha for r in recs])
    return g, E, Eo, np.max(np.abs(A - g[f"{tag}_alpha"]), axis=1)


def test_traction3d12_trajectory_parity():
    g, E, Eo, da = _run("parity")
    assert Eo[:, 1].max() > 0.1 * Eo[:, 2].max()  # the crack runs through inside the schedule
    rel = np.abs(E - Eo) / np.maximum(np.abs(Eo), 1e-300)
    for k in range(E.shape[0]):
        for q in range(3):
            if Eo[k, q] == 0.0:  # undamaged steps: no dissipation on either side
                assert abs(E[k, q]) <= 1e-12
            else:
                assert rel[k, q] <= 1e-6, f"step {k}: energy {q} rel diff {rel[k, q]:.3e}"
        assert da[k] <= 1e-4, f"step {k}: max |d alpha| {da[k]:.3e}"


def test_traction3d12_trajectory_config_literal():
    g, E, Eo, da = _run("literal")
    for k in range(E.shape[0]):
        assert abs(E[k, 2] - Eo[k, 2]) <= 1e-4 * abs(Eo[k, 2]), f"step {k}: total energy"
        assert abs(E[k, 1] - Eo[k, 1]) <= 1e-4 * abs(Eo[k, 2]), f"step {k}: dissipated energy"
        assert da[k] <= 1e-3, f"step {k}: max |d alpha| {da[k]:.3e}"
