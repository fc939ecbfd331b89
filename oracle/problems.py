"""Benchmark setups and the quasi-static driver -- oracle (test infrastructure only).

``traction`` restates the reference's ``setup_traction`` (``cases.py:154-192``);
``run`` restates ``run_quasistatic`` (``cases.py:268-306``).  The other setups
are the BASELINE.json configs the reference does not implement (SENT,
erf-profile thermal slab with E noise, 3D traction with a lognormal Gc
field); every choice a config leaves open is fixed here and documented in
DESIGN.md ("Config choices").
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Callable, Optional

import numpy as np
from scipy.special import erf

from .am import AMConfig, LoadState, StepStats, load_step
from .meshgen import SimplexMesh, banded_rows, grid_mesh, kuhn_mesh
from .p1 import EnergyParts, MaterialSpec, P1Model, merge_bcs


def critical_traction(spec: MaterialSpec) -> float:
    """sqrt(3 Gc / (8 E ell)) (model.py:84-91; AT1 uniaxial onset)."""
    return math.sqrt(3.0 * spec.Gc / (8.0 * spec.E * spec.ell))


def critical_shock_plane_strain(spec: MaterialSpec) -> float:
    """AT1 onset of an in-plane isotropic shock at a laterally constrained,
    traction-free plane-strain face: surface stress E dT/(1-nu^2), energy
    density E dT^2/(1-nu^2) = 3 Gc/(8 ell)  =>  dT_c = sqrt(3 Gc (1-nu^2)/(8 E ell)).
    (Reference critical_shock, model.py:94-104, is the plane-stress analogue.)"""
    return math.sqrt(3.0 * spec.Gc * (1.0 - spec.nu ** 2) / (8.0 * spec.E * spec.ell)) / spec.beta


@dataclass
class Setup:
    name: str
    model: P1Model
    schedule: np.ndarray
    apply_load: Callable[[P1Model, LoadState, float], None]
    initial_alpha_lb: Optional[np.ndarray] = None
    seed_threshold: Optional[float] = None
    seed_alpha: Optional[np.ndarray] = None
    params: dict = field(default_factory=dict)


def comp_dofs(verts, comp, d):
    return (d * np.asarray(verts) + comp).astype(np.intp)


def traction(spec: MaterialSpec, L=1.0, H=0.3, nx=None, ny=None, pattern="union_jack",
             n_steps=30, load_max_factor=1.5, seed_level=0.05, include_zero=False) -> Setup:
    """Bar on [0,L]x[0,H]: u1=0 left, u1=t L right, u2=0 at vertex 0 (cases.py:154-192).

    ``include_zero`` selects linspace(0, f t_c, n) (BASELINE config 1) instead of the
    reference's linspace(0, f t_c, n+1)[1:]."""
    h = spec.ell / 5.0
    nx = max(1, round(L / h)) if nx is None else nx
    ny = max(1, round(H / h)) if ny is None else ny
    mesh = grid_mesh(nx, ny, L, H, pattern)
    model = P1Model(mesh, spec)
    tc = critical_traction(spec)
    sched = (np.linspace(0.0, load_max_factor * tc, n_steps) if include_zero
             else np.linspace(0.0, load_max_factor * tc, n_steps + 1)[1:])
    left = comp_dofs(mesh.boundary["left"], 0, 2)
    right = comp_dofs(mesh.boundary["right"], 0, 2)
    pin = np.array([1], dtype=np.intp)   # u2 of vertex 0 (nearest the origin)

    def apply_load(m: P1Model, st: LoadState, t: float):
        m.bc = merge_bcs((left, np.zeros(left.size)), (right, np.full(right.size, t * L)),
                         (pin, np.zeros(1)))

    x = mesh.vertices[:, 0]
    cols = np.unique(mesh.vertices[: (nx + 1) * (ny + 1), 0])
    xs = cols[np.argmin(np.abs(cols - 0.5 * L))]
    hx = L / nx
    seed = np.where(np.abs(x - xs) < 0.5 * hx, seed_level, 0.0)
    return Setup("traction", model, sched, apply_load, seed_threshold=tc, seed_alpha=seed,
                 params={"critical_traction": tc, "L": L})


def sent(n=512, spec: Optional[MaterialSpec] = None, n_steps=60, t_max=6e-3,
         pattern="crossed") -> Setup:
    """Single-edge-notched tension on the unit square (BASELINE config 2)."""
    spec = spec or MaterialSpec(E=210.0, nu=0.3, Gc=2.7e-3, ell=0.01, k_ell=1e-6,
                                model="AT2", regime="plane_strain")
    mesh = grid_mesh(n, n, 1.0, 1.0, pattern)
    model = P1Model(mesh, spec)
    v = mesh.vertices
    notch = (np.abs(v[:, 1] - 0.5) < 1e-12) & (v[:, 0] <= 0.5 + 1e-12)
    lb = np.where(notch, 1.0, 0.0)
    bot = mesh.boundary["bottom"]
    top = mesh.boundary["top"]
    fixed = np.concatenate([comp_dofs(bot, 0, 2), comp_dofs(bot, 1, 2)])
    topy = comp_dofs(top, 1, 2)
    sched = t_max * np.arange(1, n_steps + 1) / n_steps

    def apply_load(m, st, t):
        m.bc = merge_bcs((fixed, np.zeros(fixed.size)), (topy, np.full(topy.size, t)))

    return Setup("sent", model, sched, apply_load, initial_alpha_lb=lb,
                 params={"notch_vertices": int(notch.sum())})


def thermal_slab(nx=2048, ny=512, spec: Optional[MaterialSpec] = None, n_steps=40,
                 dT_factor=3.0, tau=1e-3, noise=0.01, seed=0, pattern="union_jack") -> Setup:
    """Quenched slab [0,4]x[0,1] (BASELINE config 3): eps0 = -dT (1 - erf(y / (2 sqrt tau))) I."""
    spec = spec or MaterialSpec(E=1.0, nu=0.2, Gc=1.0, ell=0.01, model="AT1",
                                regime="plane_strain")
    mesh = grid_mesh(nx, ny, 4.0, 1.0, pattern)
    rng = np.random.default_rng(seed)
    E_cell = spec.E * (1.0 + noise * rng.uniform(-1.0, 1.0, nx * ny))
    model = P1Model(mesh, spec, E_elem=E_cell[mesh.element_cell()])
    dTc = critical_shock_plane_strain(spec)
    sched = dT_factor * dTc * np.arange(1, n_steps + 1) / n_steps
    yc = mesh.vertices[mesh.elements].mean(axis=1)[:, 1]
    prof = 1.0 - erf(yc / (2.0 * math.sqrt(tau)))
    bot = comp_dofs(mesh.boundary["bottom"], 1, 2)
    pin = np.array([0], dtype=np.intp)   # u1 of the bottom-left vertex

    def apply_load(m, st, dT):
        m.bc = merge_bcs((bot, np.zeros(bot.size)), (pin, np.zeros(1)))
        e = -spec.beta * dT * prof
        m.eps0 = np.zeros((mesh.n_elements, 3))
        m.eps0[:, 0] = e
        m.eps0[:, 1] = e

    return Setup("thermal_slab", model, sched, apply_load,
                 params={"critical_shock": dTc, "tau": tau, "E_cell": E_cell})


def surfing_displacement(points, t, spec: MaterialSpec, K_I=None, v=1.0, L_c=0.05):
    """Asymptotic Mode-I displacement about a tip at (L_c + v t, 0), theta in (-pi, pi] from +x,
    plane-stress Kolosov constant (3 - nu)/(1 + nu) (cases.py:42-63)."""
    pts = np.atleast_2d(np.asarray(points, dtype=float))
    K = math.sqrt(spec.Gc * spec.E) if K_I is None else K_I
    kappa = (3.0 - spec.nu) / (1.0 + spec.nu)
    mu = spec.E / (2.0 * (1.0 + spec.nu))
    dx = pts[:, 0] - (L_c + v * t)
    dy = pts[:, 1]
    r = np.hypot(dx, dy)
    th = np.arctan2(dy, dx)
    amp = (K / (2.0 * mu)) * np.sqrt(r / (2.0 * np.pi)) * (kappa - np.cos(th))
    return np.stack([amp * np.cos(0.5 * th), amp * np.sin(0.5 * th)], axis=1)


def surfing(spec: Optional[MaterialSpec] = None, L=2.0, H=1.0, h=None, h_coarse=None,
            band_halfwidth=None, K_I=None, v=1.0, L_c=0.05, n_steps=25, t_end=1.0) -> Setup:
    """Steady crack propagation on [0,L]x[-H/2,H/2] driven by the translated Mode-I field on the
    whole boundary, pre-crack alpha_lb = 1 within h of {y=0, 0<=x<=L_c}, mesh refined in a band
    around y = 0 (cases.py:110-150, banded_rect_mesh mesh.py:163-190)."""
    spec = spec or MaterialSpec(ell=0.1)
    h = spec.ell / 5.0 if h is None else h
    h_coarse = 5.0 * h if h_coarse is None else h_coarse
    band_halfwidth = 2.0 * spec.ell if band_halfwidth is None else band_halfwidth
    nx, ys = banded_rows(L, H, h, h_coarse, band_halfwidth)
    mesh = grid_mesh(nx, len(ys) - 1, L, H, "union_jack", 0.0, -H / 2, ys=ys)
    model = P1Model(mesh, spec)
    b = mesh.boundary
    bverts = np.unique(np.concatenate([b["left"], b["right"], b["bottom"], b["top"]]))
    bdofs = np.column_stack([2 * bverts, 2 * bverts + 1]).ravel().astype(np.intp)
    bxy = mesh.vertices[bverts]

    def apply_load(m, st, t):
        vals = surfing_displacement(bxy, t, spec, K_I=K_I, v=v, L_c=L_c)
        m.bc = merge_bcs((bdofs, vals.ravel()))

    xy = mesh.vertices
    near = np.clip(xy[:, 0], 0.0, L_c)
    lb = np.where(np.hypot(xy[:, 0] - near, xy[:, 1]) <= h * (1.0 + 1e-9), 1.0, 0.0)
    sched = np.linspace(0.0, t_end, n_steps)
    return Setup("surfing", model, sched, apply_load, initial_alpha_lb=lb,
                 params={"L_c": L_c, "v": v, "h": h, "ys": ys, "nx": nx})


def lognormal_gc(n, sigma=0.1, seed=0, Gc=1.0):
    """Per-hex-cell Gc*exp(N(0, sigma^2)), then one Jacobi pass (mean with face neighbours)."""
    rng = np.random.default_rng(seed)
    g = Gc * np.exp(rng.normal(0.0, sigma, (n, n, n)))
    s = g.copy()
    c = np.ones_like(g)
    for ax in range(3):
        for sh in (1, -1):
            r = np.roll(g, sh, axis=ax)
            valid = np.ones_like(g, dtype=bool)
            idx = [slice(None)] * 3
            idx[ax] = 0 if sh == 1 else -1
            valid[tuple(idx)] = False
            s += np.where(valid, r, 0.0)
            c += valid
    return (s / c).ravel()


def traction3d(n=128, spec: Optional[MaterialSpec] = None, n_steps=30, load_max_factor=1.5,
               sigma=0.1, seed=0) -> Setup:
    """3D AT1 traction of the unit cube with lognormal Gc (BASELINE config 4)."""
    spec = spec or MaterialSpec(E=1.0, nu=0.3, Gc=1.0, ell=0.03, model="AT1", regime="3d")
    mesh = kuhn_mesh(n, n, n)
    Gc_cell = lognormal_gc(n, sigma, seed, spec.Gc)
    model = P1Model(mesh, spec, Gc_elem=Gc_cell[mesh.element_cell()])
    tc = critical_traction(spec)
    sched = np.linspace(0.0, load_max_factor * tc, n_steps + 1)[1:]
    z0 = mesh.boundary["z0"]
    z1 = mesh.boundary["z1"]
    clamp = np.concatenate([comp_dofs(z0, c, 3) for c in range(3)])
    pull = comp_dofs(z1, 2, 3)

    def apply_load(m, st, t):
        m.bc = merge_bcs((clamp, np.zeros(clamp.size)), (pull, np.full(pull.size, t)))

    return Setup("traction3d", model, sched, apply_load,
                 params={"critical_traction": tc, "Gc_cell": Gc_cell})


@dataclass
class StepRow:
    step: int
    load: float
    energy: EnergyParts
    stats: StepStats
    u: Optional[np.ndarray] = None
    alpha: Optional[np.ndarray] = None


def run(setup: Setup, cfg: AMConfig, snapshot_stride=1, steps=None,
        state: Optional[LoadState] = None):
    """March through the schedule (cases.py:268-306); returns (rows, final state)."""
    m = setup.model
    st = LoadState.zeros(m, setup.initial_alpha_lb) if state is None else state
    rows = []
    seeded = False
    n = setup.schedule.shape[0]
    rng = range(n) if steps is None else steps
    for k in rng:
        t = float(setup.schedule[k])
        st.load = t
        st.alpha_lb = st.alpha.copy()
        setup.apply_load(m, st, t)
        if m.bc is not None:
            st.u[m.bc[0]] = m.bc[1]
        if (setup.seed_threshold is not None and not seeded
                and t > setup.seed_threshold * (1.0 + 1e-12)):
            st.alpha = np.maximum(st.alpha, setup.seed_alpha)
            seeded = True
        rep = load_step(st, m, cfg)
        en = m.energy(st.u, st.alpha)
        snap = snapshot_stride > 0 and (k % snapshot_stride == 0 or k == n - 1)
        rows.append(StepRow(k, t, en, rep, st.u.copy() if snap else None,
                            st.alpha.copy() if snap else None))
        if not rep.converged:
            raise RuntimeError(f"oracle: no convergence at step {k} (load {t:g})")
    return rows, st
