"""INI front end on the device path (reference runio.py / cli.py): grammar, validation, echo,
artifact formats against the reference's own outputs (tests/golden/cli, made by
make_cli_golden.sh from the reference CLI), device-to-GPU mapping of sweep workers, and GPU runs
whose energies match the reference's."""

import filecmp
import os

import numpy as np
import pytest

from conftest import GOLDEN
from paper_1511_08463_b200 import runio

CLI = os.path.join(GOLDEN, "cli")


def read(name):
    with open(os.path.join(CLI, name)) as fh:
        return fh.read()


def csv_rows(path):
    with open(path) as fh:
        head = fh.readline().strip().split(",")
        return head, [dict(zip(head, line.strip().split(","))) for line in fh if line.strip()]


@pytest.mark.parametrize("name", ["traction", "surfing"])
def test_validate_echo_matches_reference(name):
    cfg = runio.parse_config(read(f"{name}.ini"))
    assert runio.echo_config(cfg) == read(f"ref_{name}_echo.ini")
    assert runio.parse_config(runio.echo_config(cfg)) == cfg


def test_defaults_follow_the_reference_rules():
    c = runio.parse_config("[case]\nname = surfing\nell = 0.2\n")
    assert (c.L, c.H, c.n_steps, c.h) == (2.0, 1.0, 25, 0.2 / 5.0)
    t = runio.parse_config("[case]\nname = thermal_shock\n")
    assert (t.ell, t.h, t.L) == (1.0, 0.2, 20.0)
    assert runio.parse_config("").case == "traction"


@pytest.mark.parametrize("text", [
    "[nope]\nx = 1\n",
    "[case]\nwidth = 1\n",
    "[case]\nell = abc\n",
    "[solver]\nmethod = am\nomega = 1.5\n",
    "[solver]\nmethod = oram\nomega = 2.0\n",
    "[case]\nnu = 0.5\n",
    "[case]\ntau_min = 5\ntau_max = 1\n",
    "[linear]\nelastic = lu\n",
    "[linear]\nfieldsplit_inner = mg\n",  # the device-only choice is not part of the INI grammar
    "[output]\nsnapshot_stride = -1\n",
    "[case\nname = traction\n",
])
def test_invalid_configs_raise_config_error(text):
    with pytest.raises(runio.ConfigError):
        runio.parse_config(text)


def test_sweep_grammar():
    spec = runio.parse_sweep(read("omega_sweep.ini"))
    assert spec.parameter == "omega" and spec.values == [1.0, 1.5]
    for bad in ("[case]\nname = traction\n", "[sweep]\nvalues = 1\n",
                "[sweep]\nparameter = E\nvalues = 1\n", "[sweep]\nparameter = omega\nvalues =\n",
                "[sweep]\nparameter = omega\nvalues = 1\nstep = 2\n"):
        with pytest.raises(runio.ConfigError):
            runio.parse_sweep(bad)


def test_no_device_form_is_a_config_error():
    with pytest.raises(runio.ConfigError):
        runio.build_solver_config(runio.parse_config("[linear]\nelastic = cg\nelastic_precond = ssor\n"))
    # thermal_shock runs on the element-list path (alternate minimisation only): Newton methods
    # are a configuration error before any device work
    with pytest.raises(runio.ConfigError):
        runio.build_setup(runio.parse_config("[case]\nname = thermal_shock\n[solver]\nmethod = oram_n\n"))
    s = runio.build_solver_config(runio.parse_config("[solver]\nmethod = oram_n\nomega = 1.3\n"))
    assert (s.method, s.omega) == ("oram_newton", 1.3)


@pytest.mark.parametrize("pattern", ["union_jack", "right", "crossed"])
def test_vtk_triangles_follow_the_reference_element_order(pattern):
    from oracle.meshgen import grid_mesh
    from paper_1511_08463_b200 import StructuredMesh
    m = StructuredMesh(5, 3, 1.0, 0.6, pattern)
    assert np.array_equal(runio.triangles(m), grid_mesh(5, 3, 1.0, 0.6, pattern).elements)


def test_summary_reduction_and_worker_devices():
    rows = [dict(value=1.5, status="ok", total_am_iters=140), dict(value=1.0, status="ok", total_am_iters=40),
            dict(value=1.8, status="failed", total_am_iters=0)]
    out = runio.summarise("omega", rows)
    assert [r["reduction"] for r in out] == [1.0 - 140 / 40, 0.0, 0.0]
    out = runio.summarise("ell", [dict(value=0.1, status="ok", total_am_iters=10),
                                  dict(value=0.2, status="ok", total_am_iters=5)])
    assert [r["reduction"] for r in out] == [0.0, 0.5]
    assert [runio.device_for_worker(w, 8) for w in range(10)] == [0, 1, 2, 3, 4, 5, 6, 7, 0, 1]


def test_cli_exit_codes(tmp_path, capsys):
    assert runio.main(["validate", os.path.join(CLI, "traction.ini")]) == 0
    assert capsys.readouterr().out == read("ref_traction_echo.ini")
    bad = tmp_path / "bad.ini"
    bad.write_text("[case]\nname = cube\n")
    assert runio.main(["run", str(bad)]) == 2
    assert runio.main(["run", str(tmp_path / "missing.ini")]) == 4


# ---- GPU: runs through the device solvers vs the reference's own outputs ----------------------

def _close(a, b, rtol, atol):
    return abs(float(a) - float(b)) <= atol + rtol * abs(float(b))


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["traction", "surfing"])
def test_run_matches_reference_outputs(name, tmp_path):
    out = tmp_path / name
    assert runio.main(["run", os.path.join(CLI, f"{name}.ini"), "--output-dir", str(out)]) == 0
    head, rows = csv_rows(out / "energies.csv")
    rhead, ref = csv_rows(os.path.join(CLI, f"ref_{name}_energies.csv"))
    assert head == rhead and len(rows) == len(ref)
    for r, o in zip(rows, ref):
        assert r["step"] == o["step"] and float(r["load"]) == float(o["load"])
        for k in ("elastic", "dissipated", "total"):
            # north-star energy tolerance (1e-6 relative); energies that vanish: absolute floor
            assert _close(r[k], o[k], 1e-6, 1e-12), (name, r["step"], k, r[k], o[k])
        assert r["newton_iters"] == o["newton_iters"]
        # AM counts at crack nucleation depend on where each solver stops inside outer_atol
        assert abs(int(r["am_iters"]) - int(o["am_iters"])) <= max(2, 0.15 * int(o["am_iters"]))
    ih, _ = csv_rows(out / "iterations.csv")
    assert ih == csv_rows(os.path.join(CLI, f"ref_{name}_iterations.csv"))[0]
    assert (out / "provenance.txt").read_text().count("--- config echo ---") == 1
    snaps = sorted(p.name for p in out.glob("step_*.vtk"))
    stride = runio.parse_config(read(f"{name}.ini")).snapshot_stride
    n = len(ref)
    assert snaps == [f"step_{k:04d}.vtk" for k in range(n) if k % stride == 0 or k == n - 1]


@pytest.mark.gpu
def test_vtk_snapshot_matches_reference(tmp_path):
    out = tmp_path / "t"
    assert runio.main(["run", os.path.join(CLI, "traction.ini"), "--output-dir", str(out)]) == 0
    mine = (out / "step_0004.vtk").read_text().splitlines()
    ref = read("ref_traction_step_0004.vtk").splitlines()
    assert len(mine) == len(ref)
    k = ref.index("SCALARS alpha double 1")
    assert mine[:k] == ref[:k]  # header, points and connectivity are identical text
    a = np.array([float(x) for x in mine[k + 2:k + 2 + 533]])
    b = np.array([float(x) for x in ref[k + 2:k + 2 + 533]])
    assert np.max(np.abs(a - b)) < 1e-4


@pytest.mark.gpu
def test_reruns_are_bitwise_identical(tmp_path):
    for d in ("a", "b"):
        assert runio.main(["run", os.path.join(CLI, "surfing.ini"), "--output-dir", str(tmp_path / d)]) == 0
    for f in ("energies.csv", "iterations.csv", "step_0003.vtk"):
        assert filecmp.cmp(tmp_path / "a" / f, tmp_path / "b" / f, shallow=False), f


@pytest.mark.gpu
def test_omega_sweep_summary(tmp_path):
    assert runio.main(["sweep", os.path.join(CLI, "omega_sweep.ini"), "--output-dir", str(tmp_path)]) == 0
    head, rows = csv_rows(tmp_path / "summary.csv")
    rhead, ref = csv_rows(os.path.join(CLI, "ref_omega_sweep_summary.csv"))
    assert head == rhead
    for r, o in zip(rows, ref):
        assert r["status"] == o["status"] == "ok" and float(r["value"]) == float(o["value"])
        assert abs(int(r["total_am_iters"]) - int(o["total_am_iters"])) <= max(3, 0.15 * int(o["total_am_iters"]))
    assert float(rows[0]["reduction"]) == 0.0
    assert (tmp_path / "omega_1.5" / "energies.csv").exists()


@pytest.mark.gpu
def test_sweep_rows_in_spawned_gpu_workers(tmp_path):
    """--threads 2: rows run in spawned worker processes pinned to GPUs (replicas)."""
    assert runio.main(["sweep", os.path.join(CLI, "omega_sweep.ini"), "--threads", "2",
                       "--output-dir", str(tmp_path)]) == 0
    head, rows = csv_rows(tmp_path / "summary.csv")
    assert [r["status"] for r in rows] == ["ok", "ok"]
    _, ref = csv_rows(os.path.join(CLI, "ref_omega_sweep_summary.csv"))
    for r, o in zip(rows, ref):
        assert abs(int(r["total_am_iters"]) - int(o["total_am_iters"])) <= max(3, 0.15 * int(o["total_am_iters"]))
