"""Host-side logic of the drop-in package (no device calls).  CPU only."""

import numpy as np
import pytest

from oracle.meshgen import grid_mesh
from oracle.p1 import MaterialSpec
from oracle.problems import critical_shock_plane_strain
from paper_1511_08463_b200 import (DamageModel, DirichletBC, Material, SolverConfig,
                                   StructuredMesh, boundary_dofs, combine_bcs, critical_shock,
                                   critical_traction, rect_mesh)


@pytest.mark.parametrize("omega", [0.0, 2.0, 2.5, -1.0])
def test_omega_outside_open_interval_rejected(omega):
    with pytest.raises(ValueError):
        SolverConfig(omega=omega)


def test_unknown_choices_rejected():
    with pytest.raises(ValueError):
        SolverConfig(method="fancy")
    with pytest.raises(ValueError):
        SolverConfig(elastic_solver="lu")
    with pytest.raises(ValueError):
        SolverConfig(coupled_solver="amg")
    with pytest.raises(ValueError):
        Material(nu=0.5)
    with pytest.raises(ValueError):
        DamageModel("AT3")


def test_dirichlet_merge_rules():
    bc = combine_bcs(DirichletBC([4, 2], [1.0, 0.0]), DirichletBC([2, 7], [0.0, 3.0]))
    assert list(bc.dofs) == [2, 4, 7] and list(bc.values) == [0.0, 1.0, 3.0]
    with pytest.raises(ValueError):
        combine_bcs(DirichletBC([2], [0.0]), DirichletBC([2], [1.0]))


@pytest.mark.parametrize("pattern", ["union_jack", "right", "crossed"])
def test_mesh_layout_matches_oracle(pattern):
    m = StructuredMesh(7, 5, 1.4, 0.5, pattern)
    o = grid_mesh(7, 5, 1.4, 0.5, pattern)
    assert m.n_vertices == o.n_vertices and m.n_triangles == o.n_elements
    assert np.allclose(m.vertices, o.vertices, rtol=0, atol=1e-15)
    for tag in ("left", "right", "bottom", "top"):
        assert np.array_equal(np.sort(m.boundary_vertices(tag)), o.boundary[tag])


@pytest.mark.parametrize("pattern", ["union_jack", "right", "crossed"])
def test_eps0_row_table_is_element_centroid(pattern):
    """The per-(type, row) centroid table used for eps0 equals the oracle's element centroids."""
    m = StructuredMesh(6, 4, 1.0, 0.8, pattern)
    o = grid_mesh(6, 4, 1.0, 0.8, pattern)
    yc = o.vertices[o.elements].mean(axis=1)[:, 1]
    tab = m.cell_row_centroid_y()
    ncell = 24
    J = np.tile(np.arange(4), 6)
    I = np.repeat(np.arange(6), 4)
    for slot in range(o.n_elements // ncell):
        for cell in range(ncell):
            if pattern == "union_jack":
                t = slot + 2 * ((I[cell] + J[cell]) % 2)
            else:
                t = slot
            assert abs(tab[t, J[cell]] - yc[slot * ncell + cell]) < 1e-15


def test_rect_mesh_and_boundary_dofs_like_reference():
    m = rect_mesh(1.0, 0.3, 0.05)
    assert (m.nx, m.ny) == (20, 6)
    d = boundary_dofs(m, "right", "displacement_x1")
    assert list(d[:2]) == [2 * 20 * 7, 2 * (20 * 7 + 1)]
    assert list(boundary_dofs(m, "left", "displacement_x2")[:2]) == [1, 3]


def test_critical_loads():
    assert np.isclose(critical_traction(Material(ell=0.1)), np.sqrt(3.75))
    mat = Material(E=1.0, nu=0.2, Gc=1.0, ell=0.01, regime="plane_strain")
    spec = MaterialSpec(E=1.0, nu=0.2, Gc=1.0, ell=0.01, regime="plane_strain")
    assert np.isclose(critical_shock(mat), critical_shock_plane_strain(spec), rtol=1e-15)
    # reference value (tests/test_model.py:102-107)
    assert np.isclose(critical_shock(Material(E=1.0, nu=0.3, Gc=1.0, ell=1.0, beta=1.0)),
                      0.6123724356957945, rtol=1e-15)


def test_stiffness_matches_oracle():
    for regime in ("plane_stress", "plane_strain"):
        mat = Material(E=2.1, nu=0.27, regime=regime)
        spec = MaterialSpec(E=2.1, nu=0.27, regime=regime)
        assert np.allclose(mat.stiffness_matrix(), spec.stiffness(), rtol=1e-15)


def test_option_structs_built_from_config():
    """SolverConfig -> pf_lin_opts / pf_vi_opts marshalling (no device needed)."""
    from paper_1511_08463_b200 import solver as S
    for reuse in (True, False):
        cfg = S.SolverConfig(elastic_solver="cg", elastic_precond="gmg", elastic_rtol=1e-9, gmg_reuse=reuse)
        o = S._lin_opts(cfg, True)
        assert o.precond == 1 and o.warm_start == 1 and o.rtol == 1e-9 and o.gmg_reuse == int(reuse)
    o = S._lin_opts(S.SolverConfig(), False)
    assert o.rtol == S.SolverConfig().direct_rtol and o.warm_start == 0


def test_reference_solver_choices_map_to_device_options():
    """coupled_solver / fieldsplit_inner / elastic_precond keep the reference meaning
    (solver.py:58-64, 251-263) on the device path, or fail loudly."""
    from paper_1511_08463_b200 import solver as S
    import pytest as _pt
    with _pt.raises(ValueError, match="not available on the B200 path"):
        S._lin_opts(S.SolverConfig(elastic_solver="cg", elastic_precond="ssor"), False)
    with _pt.raises(ValueError, match="not available on the B200 path"):
        S._lin_opts(S.SolverConfig(elastic_solver="cg", elastic_precond="chebyshev"), False)
    o = S._lin_opts(S.SolverConfig(elastic_solver="direct", elastic_precond="ssor"), False)
    assert o.precond == 1 and o.rtol == 1e-12      # reference default precond: multigrid at direct_rtol
    o = S._lin_opts(S.SolverConfig(elastic_solver="direct"), False)
    assert o.precond == 0                            # configured Jacobi kept


def test_fieldsplit_inner_choices_map_onto_the_c_options():
    """fieldsplit_inner: 'direct' (blocks solved to a tolerance), 'cg' (fixed PCG budget, the
    reference inner_cg) and 'mg' (device: one V-cycle for A, Chebyshev-Jacobi for C) map onto
    pf_vi_opts.inner_mode / inner_cycles; anything else is rejected like the reference."""
    from paper_1511_08463_b200 import solver as S
    from paper_1511_08463_b200.vi import VIConfig
    with pytest.raises(ValueError):
        SolverConfig(fieldsplit_inner="amg")
    captured = {}

    class Stop(Exception):
        pass

    class FakeProblem:
        def call(self, name, *args):
            captured["opts"] = args[5]._obj
            raise Stop

    class FakeState:
        u = alpha = alpha_lb = None

        def copy(self):
            return self

    orig, orig_stream = S._lib.ptr, S._stream
    S._lib.ptr = lambda t: 0
    S._stream = lambda: None
    try:
        for inner, mode, cycles in [("direct", 0, 0), ("cg", 0, 5), ("mg", 2, 12)]:
            with pytest.raises(Stop):
                S.coupled_newton_solve(FakeState(), FakeProblem(), SolverConfig(fieldsplit_inner=inner))
            o = captured["opts"]
            assert (o.inner_mode & 3, o.inner_cycles) == (mode, cycles), inner
            assert o.inner_mode & 4                      # newton_forcing (default): inexact Newton bit
        with pytest.raises(Stop):
            S.coupled_newton_solve(FakeState(), FakeProblem(),
                                   SolverConfig(fieldsplit_inner="mg", fieldsplit_cheb_degree=7))
        assert captured["opts"].inner_cycles == 7
        with pytest.raises(Stop):
            S.coupled_newton_solve(FakeState(), FakeProblem(),
                                   SolverConfig(fieldsplit_inner="mg", fieldsplit_additive=False))
        assert captured["opts"].inner_mode & 3 == 1
        with pytest.raises(Stop):
            S.coupled_newton_solve(FakeState(), FakeProblem(),
                                   SolverConfig(fieldsplit_inner="mg", newton_forcing=False))
        assert captured["opts"].inner_mode == 2          # the reference's fixed fieldsplit_rtol
    finally:
        S._lib.ptr, S._stream = orig, orig_stream
    assert VIConfig(inner_mode=1).to_c().inner_mode == 1
