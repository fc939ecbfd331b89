"""Shared builders for the GPU parity tests: one device Discretization and one oracle
P1Model on byte-identical inputs (host-generated with numpy default_rng)."""

import numpy as np

from oracle.meshgen import grid_mesh
from oracle.p1 import MaterialSpec, P1Model


def element_type_and_row(nx, ny, pattern):
    """(type, J) of every oracle element (type-major storage, I-major cells)."""
    ncell = nx * ny
    npc = 4 if pattern == "crossed" else 2
    cell = np.tile(np.arange(ncell), npc)
    slot = np.repeat(np.arange(npc), ncell)
    I, J = cell // ny, cell % ny
    if pattern == "union_jack":
        t = slot + 2 * ((I + J) % 2)
    else:
        t = slot
    return t, J, cell


def make_pair(pattern="union_jack", regime="plane_stress", model="AT1", nx=13, ny=9, lx=1.3,
              ly=0.9, hetero=False, eps0=False, bc=True, seed=0, E=1.7, nu=0.27, Gc=1.3,
              ell=0.1, k_ell=1e-6):
    import paper_1511_08463_b200 as pf
    rng = np.random.default_rng(seed)
    mat = pf.Material(E=E, nu=nu, Gc=Gc, ell=ell, k_ell=k_ell, regime=regime)
    spec = MaterialSpec(E=E, nu=nu, Gc=Gc, ell=ell, k_ell=k_ell, model=model, regime=regime)
    mesh = pf.StructuredMesh(nx, ny, lx, ly, pattern)
    ncell = nx * ny
    E_cell = E * (1 + 0.2 * rng.uniform(-1, 1, ncell)) if hetero else None
    Gc_cell = Gc * np.exp(0.2 * rng.standard_normal(ncell)) if hetero else None
    prob = pf.Discretization(mesh, mat, pf.DamageModel(model), E_cell=E_cell, Gc_cell=Gc_cell)
    om_mesh = grid_mesh(nx, ny, lx, ly, pattern)
    t, J, cell = element_type_and_row(nx, ny, pattern)
    om = P1Model(om_mesh, spec, E_elem=None if E_cell is None else E_cell[cell],
                 Gc_elem=None if Gc_cell is None else Gc_cell[cell])
    if eps0:
        tab = 0.01 * rng.standard_normal((4, ny))
        prob.eps0_rows = tab
        e = tab[t, J]
        om.eps0 = np.column_stack([e, e, np.zeros_like(e)])
    if bc:
        left = 2 * om_mesh.boundary["left"]
        right = 2 * om_mesh.boundary["right"]
        top = 2 * om_mesh.boundary["top"] + 1
        dofs = np.concatenate([left, right, top, [1]])
        vals = np.concatenate([np.zeros(left.size), np.full(right.size, 0.07),
                               np.full(top.size, -0.01), [0.0]])
        b = pf.DirichletBC(dofs, vals)
        prob.bc = b
        om.bc = (b.dofs.astype(np.intp), b.values)
    return prob, om, rng


def random_fields(om, rng, lb_scale=0.3, u_scale=0.1):
    nv = om.nv
    lb = rng.uniform(0.0, lb_scale, nv)
    alpha = lb + rng.uniform(0.0, 1.0, nv) * (1.0 - lb)
    u = rng.standard_normal(om.nu_dofs) * u_scale
    return u, alpha, lb


def rel(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


def symmetric_alpha_distance(alpha, ref, nx, ny):
    """max|alpha - g(ref)| minimised over the symmetries of the structured bar problems
    (identity, x-mirror, y-mirror, 180-degree rotation; corner vertices).  Crack nucleation
    at a symmetric seed is a pitchfork bifurcation: which of the mirror-image branches the
    iteration follows is decided by round-off, and both branches have identical energies
    (the union-jack mesh is mirror symmetric, the right-diagonal mesh is 180-degree symmetric)."""
    a = np.asarray(alpha)[: (nx + 1) * (ny + 1)].reshape(nx + 1, ny + 1)
    r = np.asarray(ref)[: (nx + 1) * (ny + 1)].reshape(nx + 1, ny + 1)
    cands = [r, r[::-1, :], r[:, ::-1], r[::-1, ::-1]]
    return float(min(np.max(np.abs(a - c)) for c in cands))
