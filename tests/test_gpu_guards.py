"""Bounds checks of the native library (compute-sanitizer is not available on this pool).

Every workspace buffer of a context created with PF_WS_GUARD=1 is followed by a 16 KB guard zone
filled with 0xA5 (pf_check_guards counts overwritten guard bytes), and every caller-owned field or
vector passed in is a view into a NaN-filled tensor with 4096 guard elements on each side:
* an out-of-bounds WRITE past any workspace buffer, multigrid-level buffer or caller tensor changes
  a guard byte / a guard NaN pattern -> caught bitwise;
* an out-of-bounds READ of a caller tensor pulls a NaN into the result -> caught by the finiteness
  and oracle-parity checks.
The sizes are odd and tiny (1 x 3, 13 x 7, 3 x 4 x 5) so strip, tile and block boundaries fall
everywhere, plus one wide mesh (5 x 131) with interior windows of the TMA engine; the 2D cases run on
both strip engines (the TMA engine cannot read outside a caller tensor by construction -- its tensor
maps carry the extents and the hardware zero-fills -- so for it the checks are about writes); every kernel family on the load-step path runs: operators, physics, load, the elastic
PCG (Jacobi and multigrid), the damage VI (persistent PCG), the relaxation, Newton (device MINRES).
"""

import ctypes as C

import numpy as np
import pytest
import torch

from gpu_util import make_pair, random_fields

pytestmark = pytest.mark.gpu
PAD = 4096


class Padded:
    """A device vector inside NaN guards (a bit pattern, compared bitwise)."""

    def __init__(self, host):
        host = np.ascontiguousarray(host, dtype=np.float64)
        self.n = host.size
        self.buf = torch.full((self.n + 2 * PAD,), float("nan"), dtype=torch.float64, device="cuda")
        self.v = self.buf[PAD:PAD + self.n]
        self.v.copy_(torch.as_tensor(host, device="cuda"))
        self.pattern = torch.full((PAD,), float("nan"), dtype=torch.float64, device="cuda").view(torch.int64)

    def intact(self):
        b = self.buf.view(torch.int64)
        return bool(torch.equal(b[:PAD], self.pattern) and torch.equal(b[PAD + self.n:], self.pattern))


def _ptr(t):
    return t.v.data_ptr() if isinstance(t, Padded) else (None if t is None else t.data_ptr())


def _guard_bytes(prob):
    from paper_1511_08463_b200.fem import _stream
    bad = C.c_int64(-1)
    prob.call("pf_check_guards", C.byref(bad), _stream())
    return bad.value


def _exercise(prob, om, rng, dim):
    import paper_1511_08463_b200 as pf
    from paper_1511_08463_b200 import _lib
    from paper_1511_08463_b200.fem import _stream
    from paper_1511_08463_b200.vi import VIConfig
    s = _stream()
    u, a, lb = random_fields(om, rng, u_scale=0.3)
    nu, na = om.nu_dofs, om.nv
    U, A, LB = Padded(u), Padded(a), Padded(lb)
    X, XA = Padded(rng.standard_normal(nu)), Padded(rng.standard_normal(na))
    outs = []

    def out(n):
        p = Padded(np.zeros(n))
        outs.append(p)
        return p

    Y = out(nu)
    prob.call("pf_apply_Kuu", _ptr(A), _ptr(X), _ptr(Y), _lib.BC_NONE, s)
    ref = om.Kuu(a, eliminate=False) @ X.v.cpu().numpy()
    assert np.max(np.abs(Y.v.cpu().numpy() - ref)) <= 1e-12 * np.max(np.abs(ref))
    YA = out(na)
    prob.call("pf_apply_Kaa", _ptr(U), _ptr(A), _ptr(XA), _ptr(YA), s)
    ref = om.Kaa(u, a) @ XA.v.cpu().numpy()
    assert np.max(np.abs(YA.v.cpu().numpy() - ref)) <= 1e-12 * np.max(np.abs(ref))
    prob.call("pf_apply_Kua", _ptr(U), _ptr(A), _ptr(XA), _ptr(out(nu)), _lib.BC_ELIMINATE, s)
    prob.call("pf_apply_Kau", _ptr(U), _ptr(A), _ptr(X), _ptr(out(na)), _lib.BC_ELIMINATE, s)
    res = (C.c_double * 8)()
    prob.call("pf_physics", _ptr(U), _ptr(A), _ptr(LB), _ptr(out(nu)), _ptr(out(na)), _ptr(out(na)),
              _lib.ROWS_ZERO, res, s)
    assert all(np.isfinite(list(res)))
    prob.call("pf_load_u", _ptr(A), _ptr(out(nu)), s)
    for prec in (_lib.PREC["jacobi"], _lib.PREC["gmg"]):
        opts = _lib.LinOpts(precond=prec, warm_start=1, maxit=0, rtol=1e-10, atol=0.0, check_every=4,
                            gmg_levels=0, cheb_degree=2, gmg_reuse=0)
        rep = _lib.LinReport()
        prob.call("pf_elastic_solve", _ptr(A), _ptr(U), _ptr(out(nu)), C.byref(opts), C.byref(rep), s)
        assert rep.converged
    vic = VIConfig(abs_tol=1e-9, inner_rtol=1e-12)
    vrep = _lib.VIReport()
    AD = out(na)
    prob.call("pf_damage_solve", _ptr(U), _ptr(LB), _ptr(A), _ptr(AD), C.byref(vic.to_c()), C.byref(vrep), s)
    assert vrep.converged
    ph, rx = (C.c_double * 8)(), (C.c_double * 3)()
    prob.call("pf_relax_alpha_physics", _ptr(U), _ptr(A), _ptr(AD), _ptr(LB), 1.5, _ptr(out(na)), ph, rx, s)
    prob.call("pf_relax_u", _ptr(U), _ptr(X), 1.5, _ptr(out(nu)), s)
    prob.call("pf_snap_bc", _ptr(out(nu)), s)
    # Newton with the device MINRES (multigrid field split) from a damaged state
    cfg = pf.SolverConfig(outer_atol=1e-8, fieldsplit_inner="mg", max_newton_iterations=6)
    vn = VIConfig(abs_tol=1e-8, max_iterations=6, fieldsplit_rtol=1e-6, inner_cycles=6, inner_mode=2)
    nrep = _lib.VIReport()
    prob.call("pf_newton", _ptr(U), _ptr(A), _ptr(LB), _ptr(out(nu)), _ptr(out(na)), C.byref(vn.to_c()),
              C.byref(nrep), s)
    del cfg
    torch.cuda.synchronize()
    for p in [U, A, LB, X, XA] + outs:
        assert p.intact(), "a kernel wrote outside a caller buffer"
    for p in outs:
        assert bool(torch.isfinite(p.v).all()), "a kernel read outside a caller buffer (NaN in the result)"
    assert _guard_bytes(prob) == 0, "a kernel wrote past a workspace buffer"


@pytest.mark.parametrize("engine", ["0", "1"])  # one-column cp.async engine / two-column TMA engine
@pytest.mark.parametrize("pattern", ["union_jack", "right", "crossed"])
@pytest.mark.parametrize("shape", [(13, 7), (1, 3), (33, 2), (5, 131)])
def test_bounds_2d(pattern, shape, engine, monkeypatch):
    monkeypatch.setenv("PF_WS_GUARD", "1")
    monkeypatch.setenv("PF_STRIP2", engine)
    prob, om, rng = make_pair(pattern, "plane_strain", "AT2", shape[0], shape[1], hetero=True, eps0=True)
    assert prob.ws_guarded()
    _exercise(prob, om, rng, 2)


@pytest.mark.parametrize("shape", [(3, 4, 5), (1, 1, 2), (9, 2, 7)])
def test_bounds_3d(shape, monkeypatch):
    import paper_1511_08463_b200 as pf
    from oracle.meshgen import kuhn_mesh
    from oracle.p1 import MaterialSpec, P1Model
    monkeypatch.setenv("PF_WS_GUARD", "1")
    nx, ny, nz = shape
    rng = np.random.default_rng(nx + ny + nz)
    mat = pf.Material(E=1.0, nu=0.3, Gc=1.0, ell=0.1, k_ell=1e-6, regime="3d")
    prob = pf.Discretization(pf.StructuredMesh3D(nx, ny, nz), mat, pf.DamageModel("AT1"))
    om = P1Model(kuhn_mesh(nx, ny, nz), MaterialSpec(E=1.0, nu=0.3, Gc=1.0, ell=0.1, k_ell=1e-6,
                                                     model="AT1", regime="3d"))
    z0 = om.mesh.boundary["z0"]
    dofs = np.concatenate([3 * z0, 3 * z0 + 1, 3 * z0 + 2])
    prob.bc = pf.DirichletBC(np.sort(dofs), np.zeros(dofs.size))
    assert prob.ws_guarded()
    _exercise(prob, om, rng, 3)


def test_guards_catch_an_out_of_bounds_write(monkeypatch):
    """Positive control: a caller buffer 10 entries too short is overrun by the apply, and the NaN
    guard after it records the overrun."""
    from paper_1511_08463_b200 import _lib
    from paper_1511_08463_b200.fem import _stream
    monkeypatch.setenv("PF_WS_GUARD", "1")
    prob, om, rng = make_pair("crossed", "plane_strain", "AT2", 13, 7)
    u, a, lb = random_fields(om, rng)
    A, X = Padded(a), Padded(rng.standard_normal(om.nu_dofs))
    short = Padded(np.zeros(om.nu_dofs - 10))
    prob.call("pf_apply_Kuu", _ptr(A), _ptr(X), _ptr(short), _lib.BC_NONE, _stream())
    torch.cuda.synchronize()
    assert not short.intact()
    assert A.intact() and X.intact() and _guard_bytes(prob) == 0
