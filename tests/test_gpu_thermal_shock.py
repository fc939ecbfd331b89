"""The reference's own thermal-shock case (cases.py:195-235) on the element-list path, against the
golden trajectory the reference itself produced (tests/golden/make_thermal_shock_golden.py):
the jittered 80 x 40 union-jack rect_mesh (reproduced bit for bit), the erfc inelastic strain at
the element centroids, 12 geometric tau steps at dT = 2 dT_c while the periodic crack pattern
forms, alternate minimisation (method am) at outer_atol 1e-8.  North-star bars at every step:
energies within 1e-6 relative, alpha within 1e-4 (the jitter breaks every symmetry).  Also the
INI front end: ``[case] name = thermal_shock`` now runs (runio.py) and writes its artifacts."""

import os

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu


def test_thermal_shock_matches_reference_trajectory():
    import paper_1511_08463_b200 as pf
    g = np.load(os.path.join(GOLDEN, "ref_thermal_shock.npz"))
    setup = pf.setup_thermal_shock(n_steps=int(g["steps"]), dT_factor=float(g["dT_factor"]))
    assert np.array_equal(setup.mesh.vertices, g["vertices"])  # the reference's jittered mesh
    cfg = pf.SolverConfig(method="am", outer_atol=float(g["atol"]))
    recs = pf.run_quasistatic(setup, cfg)
    E = np.array([tuple(r.energy) for r in recs])
    Eo = g["energy"]
    assert Eo[-1, 1] > 0.5 * Eo[-1, 2]  # the crack pattern formed inside the schedule
    for k in range(E.shape[0]):
        for q in range(3):
            if Eo[k, q] == 0.0:
                assert abs(E[k, q]) <= 1e-12
            else:
                assert abs(E[k, q] - Eo[k, q]) <= 1e-6 * abs(Eo[k, q]), f"step {k} energy {q}"
        assert np.max(np.abs(recs[k].alpha - g["alpha"][k])) <= 1e-4, f"step {k} alpha"


def test_thermal_shock_ini_runs_on_the_device(tmp_path):
    from paper_1511_08463_b200 import runio
    cfg = runio.parse_config("[case]\nname = thermal_shock\nn_steps = 4\nL = 8.0\nH = 4.0\n"
                             "[solver]\nmethod = oram\nomega = 1.4\n")
    rc = runio.run(cfg, output_dir=str(tmp_path))
    assert rc == 0
    assert (tmp_path / "energies.csv").exists() and (tmp_path / "iterations.csv").exists()
    assert sorted(p.name for p in tmp_path.glob("step_*.vtk"))
    text = (tmp_path / "iterations.csv").read_text().splitlines()
    assert len(text) > 4
