"""The v2 2D strip engine (two vertex columns per lane, TMA row tiles; csrc/pf_strip2.cu) forced on
(PF_STRIP2=1) at test sizes -- by default it only takes meshes of 0.55M vertices and more.

Shapes are chosen so that every form of the row step runs: windows that touch the mesh boundary
(general step), interior windows (fast step: ny >= 126 gives a window with no boundary column),
strips of one row, odd row pitches (8-byte rows starting one item early, byte rows up to 15), both
union-jack parities at a strip start, per-cell fields, thermal rows and Dirichlet rows."""

import numpy as np
import pytest
import torch

import test_gpu_ops as ops
import test_gpu_solvers as sol
from gpu_util import make_pair, random_fields, rel

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _force_v2(monkeypatch):
    monkeypatch.setenv("PF_STRIP2", "1")


WIDE = [
    # pattern, regime, model, nx, ny, hetero, eps0
    ("union_jack", "plane_strain", "AT2", 37, 200, True, True),
    ("union_jack", "plane_stress", "AT1", 66, 129, False, False),
    ("right", "plane_strain", "AT1", 33, 190, True, False),
    ("crossed", "plane_stress", "AT2", 21, 150, True, True),
    ("crossed", "plane_strain", "AT1", 70, 127, False, False),
]


@pytest.mark.parametrize("case", ops.CASES + WIDE, ids=lambda c: f"{c[0]}-{c[1]}-{c[2]}-{c[3]}x{c[4]}")
def test_operator_parity_v2(case):
    ops.test_operator_parity(case)


@pytest.mark.parametrize("pattern", ["union_jack", "right", "crossed"])
def test_v2_equals_v1_bitwise_on_wide_meshes(pattern, monkeypatch):
    """Both engines form every sum in the same order: the Kuu apply is bitwise equal, the Kaa apply
    equal to round-off (the fast step's compile-time parity lets the compiler contract differently)."""
    import paper_1511_08463_b200 as pf
    out = {}
    for eng in ("0", "1"):
        monkeypatch.setenv("PF_STRIP2", eng)
        prob, om, rng = make_pair(pattern, "plane_strain", "AT2", 150, 260, hetero=True)
        u, a, lb = random_fields(om, rng)
        xu, xa = rng.standard_normal(om.nu_dofs), rng.standard_normal(om.nv)
        st = pf.State(ops.dev(u), ops.dev(a), ops.dev(lb))
        out[eng] = (ops.host(pf.assemble_Kuu(st, prob, apply_bc=True) @ ops.dev(xu)),
                    ops.host(pf.assemble_Kaa(st, prob) @ ops.dev(xa)))
    assert np.array_equal(out["0"][0], out["1"][0])
    assert rel(out["1"][1], out["0"][1]) < 1e-14


@pytest.mark.parametrize("pattern", ["union_jack", "crossed"])
def test_elastic_multigrid_solve_v2(pattern):
    """PCG with the fused CG step and the smoother epilogues on the v2 engine, wide cracked mesh."""
    import paper_1511_08463_b200 as pf
    from oracle import am as oam
    nx, ny = 60, 140
    prob, om, rng = make_pair(pattern, "plane_strain", "AT2", nx, ny, lx=1.0, ly=ny / nx, hetero=True)
    v = om.mesh.vertices
    a = np.where(np.abs(v[:, 0] - 0.5) < 1.5 / nx, 1.0, rng.uniform(0, 0.2, om.nv))
    u = np.zeros(om.nu_dofs)
    st = pf.State(ops.dev(u), ops.dev(a), ops.dev(np.zeros(om.nv)))
    ref, _ = oam.elastic_half_step(oam.LoadState(u, a, 0 * a), om, oam.AMConfig())
    for precond in ("jacobi", "gmg"):
        cfg = pf.SolverConfig(elastic_solver="cg", elastic_rtol=1e-12, elastic_precond=precond, warm_start=False)
        us, its = pf.elastic_step(st, prob, cfg)
        assert rel(ops.host(us), ref) < 1e-7, precond


@pytest.mark.parametrize("pattern,model", [("union_jack", "AT1"), ("crossed", "AT2"), ("right", "AT1")])
def test_damage_step_v2(pattern, model, monkeypatch):
    """The damage VI with its masked Kaa applies, trial evaluations and (graph-loop) PCG on v2."""
    monkeypatch.setenv("PF_PCG_GRAPH", "1")
    sol.test_damage_step_matches_oracle_rsls(pattern, model)


@pytest.mark.parametrize("pattern,model", [("union_jack", "AT2"), ("crossed", "AT1")])
def test_damage_step_v2_wide(pattern, model, monkeypatch):
    """Interior windows: masked applies read the TMA-staged active bytes in the fast row step."""
    import paper_1511_08463_b200 as pf
    from oracle import am as oam
    monkeypatch.setenv("PF_PCG_GRAPH", "1")
    prob, om, rng = make_pair(pattern, "plane_stress", model, 30, 141, hetero=True, eps0=True)
    u, a, lb = random_fields(om, rng, u_scale=0.4)
    st = pf.State(ops.dev(u), ops.dev(a), ops.dev(lb))
    ad, rep = pf.damage_step(st, prob, pf.SolverConfig(outer_atol=1e-9))
    ao, orep = oam.damage_half_step(oam.LoadState(u, a, lb), om, oam.AMConfig(outer_atol=1e-9))
    assert rep.converged and orep.converged
    assert np.max(np.abs(ops.host(ad) - ao)) < 1e-9


def test_quasistatic_run_v2():
    sol.test_quasistatic_run_matches_reference_golden()


def test_newton_v2():
    sol.test_coupled_newton_matches_oracle("crossed", "AT2")
