"""Benchmark setups and the quasi-static driver (reference cases.py).

``setup_traction`` and ``run_quasistatic`` keep the reference semantics
(cases.py:154-192, 268-306).  ``setup_sent``, ``setup_thermal_slab`` are the
BASELINE.json configs 2 and 3 the reference lacks; every open choice is the
one documented in DESIGN.md ("Config choices") and restated by the oracle
(oracle/problems.py) so both sides consume byte-identical inputs.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Callable, Optional

import numpy as np
import torch
from scipy.special import erf

from .fem import (Discretization, DirichletBC, EnergyBreakdown, State, assemble_energy,
                  combine_bcs)
from .mesh import StructuredMesh, StructuredMesh3D, banded_rect_mesh, boundary_dofs, rect_mesh
from .model import DamageModel, Material, critical_shock, critical_traction
from .solver import NonlinearReport, SolverConfig, solve_load_step


@dataclass
class ProblemSetup:
    """A benchmark: mesh, discretisation, loading program, optional seeding (cases.py:83-109)."""

    name: str
    mesh: StructuredMesh
    problem: Discretization
    schedule: np.ndarray
    apply_load: Callable[[Discretization, State, float], None]
    initial_alpha_lb: Optional[np.ndarray] = None
    seed_threshold: Optional[float] = None
    seed_alpha: Optional[np.ndarray] = None
    params: dict = field(default_factory=dict)

    def __post_init__(self):
        self.schedule = np.asarray(self.schedule, dtype=float)
        if self.schedule.ndim != 1:
            raise ValueError("schedule must be a 1D array of load values")
        if np.any(np.diff(self.schedule) <= 0.0):
            raise ValueError("schedule must be strictly increasing")


def setup_traction(material: Optional[Material] = None, L: float = 1.0, H: float = 0.3,
                   h: Optional[float] = None, n_steps: int = 30, load_max_factor: float = 1.5,
                   seed_level: float = 0.05, pattern: str = "union_jack",
                   nx: Optional[int] = None, ny: Optional[int] = None,
                   include_zero: bool = False) -> ProblemSetup:
    """Bar on [0,L]x[0,H]: u1=0 left, u1=t L right, u2 pinned at vertex 0 (cases.py:154-192).

    ``include_zero=True`` gives the schedule linspace(0, f t_c, n_steps) of BASELINE
    config 1; the default is the reference's linspace(0, f t_c, n+1)[1:]."""
    material = material or Material(ell=0.1)
    h = material.ell / 5.0 if h is None else h
    if nx is None or ny is None:
        mesh = rect_mesh(L, H, h, pattern=pattern)
    else:
        mesh = StructuredMesh(nx, ny, L, H, pattern)
    problem = Discretization(mesh, material)
    tc = critical_traction(material)
    schedule = (np.linspace(0.0, load_max_factor * tc, n_steps) if include_zero
                else np.linspace(0.0, load_max_factor * tc, n_steps + 1)[1:])
    left = boundary_dofs(mesh, "left", "displacement_x1")
    right = boundary_dofs(mesh, "right", "displacement_x1")
    pin = np.array([1], dtype=np.intp)  # u2 at vertex 0, the vertex nearest the origin

    def apply_load(problem: Discretization, state: State, t: float) -> None:
        problem.bc = combine_bcs(DirichletBC(left, np.zeros(left.size)),
                                 DirichletBC(right, np.full(right.size, t * L)),
                                 DirichletBC(pin, np.zeros(1)))

    x = mesh.vertices[:, 0]
    cols = np.linspace(0.0, L, mesh.nx + 1)
    xstar = cols[np.argmin(np.abs(cols - 0.5 * L))]
    seed = np.where(np.abs(x - xstar) < 0.5 * mesh.hx, seed_level, 0.0)
    return ProblemSetup("traction", mesh, problem, schedule, apply_load,
                        seed_threshold=tc, seed_alpha=seed,
                        params={"critical_traction": tc, "h": h, "L": L})


def setup_sent(n: int = 512, material: Optional[Material] = None, n_steps: int = 60,
               t_max: float = 6e-3, pattern: str = "crossed") -> ProblemSetup:
    """Single-edge-notched tension (BASELINE config 2): unit square, AT2, plane strain,
    notch alpha = 1 (as alpha_lb, reference convention cases.py:143-146) on y = 0.5,
    x <= 0.5; bottom clamped, top u2 = t with t_k = t_max k / n_steps, k = 1..n_steps."""
    material = material or Material(E=210.0, nu=0.3, Gc=2.7e-3, ell=0.01, k_ell=1e-6,
                                    regime="plane_strain")
    mesh = StructuredMesh(n, n, 1.0, 1.0, pattern)
    problem = Discretization(mesh, material, DamageModel("AT2"))
    v = mesh.vertices
    notch = (np.abs(v[:, 1] - 0.5) < 1e-12) & (v[:, 0] <= 0.5 + 1e-12)
    lb = np.where(notch, 1.0, 0.0)
    bot = np.sort(mesh.boundary_vertices("bottom"))
    top = np.sort(mesh.boundary_vertices("top"))
    fixed = np.concatenate([2 * bot, 2 * bot + 1])
    topy = 2 * top + 1
    schedule = t_max * np.arange(1, n_steps + 1) / n_steps

    def apply_load(problem, state, t):
        problem.bc = combine_bcs(DirichletBC(fixed, np.zeros(fixed.size)),
                                 DirichletBC(topy, np.full(topy.size, t)))

    return ProblemSetup("sent", mesh, problem, schedule, apply_load, initial_alpha_lb=lb,
                        params={"notch_vertices": int(notch.sum())})


def setup_thermal_slab(nx: int = 2048, ny: int = 512, material: Optional[Material] = None,
                       n_steps: int = 40, dT_factor: float = 3.0, tau: float = 1e-3,
                       noise: float = 0.01, seed: int = 0,
                       pattern: str = "union_jack") -> ProblemSetup:
    """Quenched slab [0,4]x[0,1] (BASELINE config 3): eps0 = -dT (1 - erf(y/(2 sqrt tau))) I,
    dT_k = dT_factor dT_c k / n_steps, E (1 + noise U[-1,1]) per cell (default_rng(seed)),
    bottom u2 = 0, bottom-left u1 = 0, plane strain AT1."""
    material = material or Material(E=1.0, nu=0.2, Gc=1.0, ell=0.01, regime="plane_strain")
    mesh = StructuredMesh(nx, ny, 4.0, 1.0, pattern)
    rng = np.random.default_rng(seed)
    E_cell = material.E * (1.0 + noise * rng.uniform(-1.0, 1.0, nx * ny))
    problem = Discretization(mesh, material, DamageModel("AT1"), E_cell=E_cell)
    dTc = critical_shock(material)
    schedule = dT_factor * dTc * np.arange(1, n_steps + 1) / n_steps
    prof = 1.0 - erf(mesh.cell_row_centroid_y() / (2.0 * math.sqrt(tau)))
    bot = 2 * np.sort(mesh.boundary_vertices("bottom")) + 1
    pin = np.array([0], dtype=np.intp)

    bc = combine_bcs(DirichletBC(bot, np.zeros(bot.size)), DirichletBC(pin, np.zeros(1)))

    def apply_load(problem, state, dT):
        problem.bc = bc
        problem.eps0_rows = -material.beta * dT * prof

    return ProblemSetup("thermal_slab", mesh, problem, schedule, apply_load,
                        params={"critical_shock": dTc, "tau": tau, "E_cell": E_cell})


def lognormal_gc(n, sigma=0.1, seed=0, Gc=1.0):
    """Per-hex Gc exp(N(0, sigma^2)) (default_rng(seed)), then one Jacobi pass: the mean of each
    cell with its face neighbours (config 4)."""
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


def setup_traction3d(n: int = 128, material: Optional[Material] = None, n_steps: int = 30,
                     load_max_factor: float = 1.5, sigma: float = 0.1, seed: int = 0) -> ProblemSetup:
    """3D AT1 traction of the unit cube with a lognormal Gc field (BASELINE config 4): z=0 face
    clamped, z=1 face u_z = t, t in linspace(0, f t_c, n+1)[1:]."""
    material = material or Material(E=1.0, nu=0.3, Gc=1.0, ell=0.03, k_ell=1e-6, regime="3d")
    mesh = StructuredMesh3D(n, n, n)
    Gc_cell = lognormal_gc(n, sigma, seed, material.Gc)
    problem = Discretization(mesh, material, DamageModel("AT1"), Gc_cell=Gc_cell)
    tc = critical_traction(material)
    schedule = np.linspace(0.0, load_max_factor * tc, n_steps + 1)[1:]
    z0 = mesh.face_vertices("z0")
    z1 = mesh.face_vertices("z1")
    clamp = np.concatenate([3 * z0, 3 * z0 + 1, 3 * z0 + 2])
    pull = 3 * z1 + 2
    def apply_load(problem, state, t):
        problem.bc = combine_bcs(DirichletBC(clamp, np.zeros(clamp.size)),
                                 DirichletBC(pull, np.full(pull.size, t)))
    return ProblemSetup("traction3d", mesh, problem, schedule, apply_load,
                        params={"critical_traction": tc, "Gc_cell": Gc_cell})


def surfing_displacement(points, t: float, material: Material, K_I: Optional[float] = None,
                         v: float = 1.0, L_c: float = 0.05) -> np.ndarray:
    """Asymptotic Mode-I displacement about a tip at (L_c + v t, 0) (cases.py:42-63): polar
    angle in (-pi, pi] from +x, plane-stress Kolosov constant (3 - nu)/(1 + nu), 0 at r = 0."""
    pts = np.atleast_2d(np.asarray(points, dtype=float))
    K = math.sqrt(material.Gc * material.E) if K_I is None else K_I
    kappa = (3.0 - material.nu) / (1.0 + material.nu)
    mu = material.E / (2.0 * (1.0 + material.nu))
    dx = pts[:, 0] - (L_c + v * t)
    dy = pts[:, 1]
    r = np.hypot(dx, dy)
    th = np.arctan2(dy, dx)
    amp = (K / (2.0 * mu)) * np.sqrt(r / (2.0 * np.pi)) * (kappa - np.cos(th))
    out = np.stack([amp * np.cos(0.5 * th), amp * np.sin(0.5 * th)], axis=1)
    return out[0] if np.asarray(points).ndim == 1 else out


def setup_surfing(material: Optional[Material] = None, L: float = 2.0, H: float = 1.0,
                  h: Optional[float] = None, h_coarse: Optional[float] = None,
                  band_halfwidth: Optional[float] = None, K_I: Optional[float] = None,
                  v: float = 1.0, L_c: float = 0.05, n_steps: int = 25,
                  t_end: float = 1.0) -> ProblemSetup:
    """Boundary-driven steady crack propagation on [0, L] x [-H/2, H/2] (cases.py:110-150): the
    translated Mode-I field on every boundary vertex, pre-crack alpha_lb = 1 within h of
    {y = 0, 0 <= x <= L_c}, graded mesh refined in a band of half-width ~2 ell."""
    material = material or Material(ell=0.1)
    h = material.ell / 5.0 if h is None else h
    h_coarse = 5.0 * h if h_coarse is None else h_coarse
    band_halfwidth = 2.0 * material.ell if band_halfwidth is None else band_halfwidth
    mesh = banded_rect_mesh(L, H, h, h_coarse, band_halfwidth)
    problem = Discretization(mesh, material)
    bverts = mesh.all_boundary_vertices()
    bdofs = np.column_stack([2 * bverts, 2 * bverts + 1]).ravel()
    bxy = mesh.vertices[bverts]

    def apply_load(problem: Discretization, state: State, t: float) -> None:
        vals = surfing_displacement(bxy, t, material, K_I=K_I, v=v, L_c=L_c)
        problem.bc = DirichletBC(bdofs, vals.ravel())

    xy = mesh.vertices
    near = np.clip(xy[:, 0], 0.0, L_c)
    lb = np.where(np.hypot(xy[:, 0] - near, xy[:, 1]) <= h * (1.0 + 1e-9), 1.0, 0.0)
    schedule = np.linspace(0.0, t_end, n_steps)
    return ProblemSetup("surfing", mesh, problem, schedule, apply_load, initial_alpha_lb=lb,
                        params={"L_c": L_c, "v": v, "h": h})


# -- quasi-static driver (cases.py:241-306) ---------------------------------------------------------

@dataclass
class StepRecord:
    step: int
    load: float
    energy: EnergyBreakdown
    report: NonlinearReport
    u: Optional[np.ndarray] = None
    alpha: Optional[np.ndarray] = None


class StepFailureError(RuntimeError):
    """Nonlinear solve failed at one load step; carries the partial run (cases.py:253-265)."""

    def __init__(self, step, load, records, state, report):
        super().__init__(f"solver did not converge at step {step} (load {load:g}); "
                         f"final residual {report.final_residual_norm:.3e}")
        self.step, self.load, self.records, self.state, self.report = step, load, records, state, report


def _to_host(problem, t) -> np.ndarray:
    """Device field -> fresh host array through a pinned staging buffer kept on the problem
    (a pageable .cpu() of a 128^3 snapshot ran at ~2.5 GB/s: 27 ms of a 0.2 s load step)."""
    if not t.is_cuda:
        return t.numpy().copy()
    n = t.numel()
    buf = getattr(problem, "_pinned_stage", None)
    if buf is None or buf.numel() < n:
        buf = torch.empty(n, dtype=t.dtype, pin_memory=True)
        problem._pinned_stage = buf
    v = buf[:n]
    v.copy_(t.reshape(-1))
    return v.numpy().copy().reshape(tuple(t.shape))


def run_quasistatic(setup, config: SolverConfig, snapshot_stride: int = 1,
                    state: Optional[State] = None, steps=None) -> list:
    """March a state through the loading schedule (cases.py:268-306).

    Fields stay on the device; snapshots are copied to the host every
    ``snapshot_stride`` steps (and on the final step).  An ``UnstructuredSetup`` (element-list
    mesh, e.g. the thermal-shock case) runs on the element-list path."""
    if isinstance(setup, UnstructuredSetup):
        return run_quasistatic_unstructured(setup, config, snapshot_stride, state, steps)
    problem = setup.problem
    state = State.zeros(setup.mesh, setup.initial_alpha_lb, device=problem.device) \
        if state is None else state
    records = []
    seeded = False
    n = setup.schedule.shape[0]
    for k in (range(n) if steps is None else steps):
        t = float(setup.schedule[k])
        state.load = t
        state.alpha_lb = state.alpha.clone()
        setup.apply_load(problem, state, t)
        if problem.bc is not None:
            state.u[problem._bc_dofs_dev] = problem._bc_vals_dev
        if (setup.seed_threshold is not None and not seeded
                and t > setup.seed_threshold * (1.0 + 1e-12)):
            seed = torch.as_tensor(setup.seed_alpha, dtype=torch.float64, device=problem.device)
            state.alpha = torch.maximum(state.alpha, seed)
            seeded = True
        report = solve_load_step(state, problem, config)
        energy = assemble_energy(state, problem)
        snap = snapshot_stride > 0 and (k % snapshot_stride == 0 or k == n - 1)
        records.append(StepRecord(step=k, load=t, energy=energy, report=report,
                                  u=_to_host(problem, state.u) if snap else None,
                                  alpha=_to_host(problem, state.alpha) if snap else None))
        if not report.converged:
            raise StepFailureError(k, t, records, state, report)
    return records


# -- element-list meshes: the reference's thermal-shock case -------------------

@dataclass
class UnstructuredSetup:
    """A benchmark on an element-list mesh (the ProblemSetup of cases.py:83-109).  ``apply_load(ops,
    t)`` installs the inelastic strain for load value t and returns the Dirichlet data (dofs,
    values)."""

    name: str
    mesh: object
    ops: object
    schedule: np.ndarray
    apply_load: Callable
    initial_alpha_lb: Optional[np.ndarray] = None
    params: dict = field(default_factory=dict)

    def __post_init__(self):
        self.schedule = np.asarray(self.schedule, dtype=float)
        if self.schedule.ndim != 1 or np.any(np.diff(self.schedule) <= 0.0):
            raise ValueError("schedule must be a strictly increasing 1D array of load values")


def thermal_strain(x2, tau: float, material: Material, delta_T: float) -> np.ndarray:
    """(e, e, 0) Voigt with e = -beta dT erfc(x2 / (ell tau)) (the reference's thermal_strain,
    cases.py:66-80)."""
    from scipy.special import erfc
    if tau <= 0.0:
        raise ValueError(f"tau must be positive, got {tau}")
    x2 = np.asarray(x2, dtype=float)
    e = -material.beta * delta_T * erfc(x2 / (material.ell * tau))
    out = np.zeros(x2.shape + (3,))
    out[..., 0] = e
    out[..., 1] = e
    return out


def setup_thermal_shock(material: Optional[Material] = None, L: float = 20.0, H: float = 10.0,
                        h: Optional[float] = None, dT_factor: float = 1.0, n_steps: int = 40,
                        tau_min: float = 0.05, tau_max: float = 3.0, jitter: float = 0.25,
                        model: str = "AT1", multigrid: bool = False) -> UnstructuredSetup:
    """Quench of [0, L] x [0, H] from its bottom surface (the reference's setup_thermal_shock,
    cases.py:195-235) on the element-list path: the jittered union-jack rect_mesh (mesh.py:112-142,
    seed 0), the erfc inelastic strain at the element centroids, u1 = 0 on the lateral sides,
    u2 = 0 on the top, tau in geomspace(tau_min, tau_max, n_steps), dT = dT_factor dT_c."""
    from .umesh import UnstructuredOperators, jittered_rect_mesh
    material = material or Material(ell=1.0)
    h = material.ell / 4.0 if h is None else h
    mesh = jittered_rect_mesh(L, H, h, jitter=jitter)
    ops = UnstructuredOperators(mesh, material, model)
    dTc = critical_shock(material)
    dT = dT_factor * dTc
    b = mesh.boundary
    dofs = np.unique(np.concatenate([2 * b["left"], 2 * b["right"], 2 * b["top"] + 1])).astype(np.int64)
    vals = np.zeros(dofs.size)
    depth = mesh.vertices[mesh.elements].mean(axis=1)[:, 1]

    def apply_load(ops, tau):
        ops.set_eps0(thermal_strain(depth, tau, material, dT))
        return dofs, vals

    schedule = np.geomspace(tau_min, tau_max, n_steps)
    if multigrid:
        # the same grid without the jitter: its multigrid V-cycle preconditions the elastic PCG
        # (SolverConfig.elastic_precond = "gmg")
        nx, ny = max(1, round(L / h)), max(1, round(H / h))
        twin = Discretization(StructuredMesh(nx, ny, L, H, "union_jack"), material, DamageModel(model))
        twin.bc = DirichletBC(dofs, vals)
        ops.attach_structured_twin(twin)
    return UnstructuredSetup("thermal_shock", mesh, ops, schedule, apply_load,
                             params={"delta_T": dT, "critical_shock": dTc, "h": h})


def run_quasistatic_unstructured(setup: UnstructuredSetup, config: SolverConfig, snapshot_stride: int = 1,
                                 state: Optional[State] = None, steps=None) -> list:
    """run_quasistatic (cases.py:268-306) on an element-list mesh: per load step the alternate
    minimisation of UnstructuredOperators.am_load_step (elastic Jacobi-PCG half-step, damage VI,
    over-relaxation with the midpoint rule).  There is no Newton phase on this path: methods other
    than "am" (= the INI's am / oram) are a ValueError."""
    import torch
    from .vi import ActiveSetReport  # noqa: F401  (report types shared with the structured path)
    if config.method != "am":
        raise ValueError(f"method {config.method!r} needs the coupled Newton step, which the element-list "
                         "path does not have; use method 'am' (am / oram in the INI)")
    ops, mesh = setup.ops, setup.mesh
    d = mesh.dim
    if state is None:
        lb = np.zeros(mesh.n_vertices) if setup.initial_alpha_lb is None else setup.initial_alpha_lb
        state = State(u=torch.zeros(d * mesh.n_vertices, dtype=torch.float64, device=ops.device),
                      alpha=torch.as_tensor(lb, dtype=torch.float64, device=ops.device).clone(),
                      alpha_lb=torch.as_tensor(lb, dtype=torch.float64, device=ops.device).clone())
    rtol = config.direct_rtol if config.elastic_solver == "direct" else config.elastic_rtol
    # elastic_precond="gmg": the V-cycle of the structured twin (jittered structured meshes only)
    precond = "gmg" if (config.elastic_precond == "gmg" and getattr(ops, "_twin", None) is not None) else "jacobi"
    records = []
    n = setup.schedule.shape[0]
    for k in (range(n) if steps is None else steps):
        t = float(setup.schedule[k])
        state.load = t
        state.alpha_lb = state.alpha.clone()
        dofs, vals = setup.apply_load(ops, t)
        st = ops.am_load_step(state.u, state.alpha, state.alpha_lb, dofs, vals, omega=config.omega,
                              outer_atol=config.outer_atol, max_am_iterations=config.max_am_iterations,
                              elastic_rtol=rtol, damage_atol_factor=config.damage_atol_factor,
                              max_vi_iterations=config.max_vi_iterations, log_callback=config.log_callback,
                              elastic_precond=precond)
        en = st["energy_history"][-1]
        energy = EnergyBreakdown(*en)
        report = NonlinearReport(converged=bool(st["converged"]), final_residual_norm=st["final_residual_norm"],
                                 am_iterations=st["am_iterations"], total_krylov_iterations=st["krylov_iterations"],
                                 omega_bar_min=st["omega_bar_min"],
                                 energy_history=[EnergyBreakdown(*e) for e in st["energy_history"]],
                                 residual_history=list(st["residual_history"]))
        snap = snapshot_stride > 0 and (k % snapshot_stride == 0 or k == n - 1)
        records.append(StepRecord(step=k, load=t, energy=energy, report=report,
                                  u=state.u.cpu().numpy() if snap else None,
                                  alpha=state.alpha.cpu().numpy() if snap else None))
        if not report.converged:
            raise StepFailureError(k, t, records, state, report)
    return records
