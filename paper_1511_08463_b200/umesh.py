"""Element-list (unstructured / jittered) P1 meshes on the device (first step).

The structured path (``fem.Discretization``) keeps geometry implicit.  The reference's
thermal-shock case builds its mesh by jittering the interior vertices of a union-jack grid
(``rect_mesh(..., jitter, seed)``, mesh.py:112-142; cases.py:195-234), after which every
element has its own shape.  ``UnstructuredOperators`` holds such a mesh (or any positively
oriented triangle / tetrahedron mesh) as element lists in a PyTorch-owned device workspace and
applies the reference's Hessian blocks through the C ABI (``pf_umesh_*``,
include/phasefrac_b200.h):

* ``apply_Kuu(alpha, x)``  = ``assemble_Kuu(state, problem, apply_bc) @ x``  (fem.py:233-244)
* ``apply_Kaa(u, alpha, x)`` = ``assemble_Kaa(state, problem) @ x``           (fem.py:266-282)
* ``elastic_solve`` / ``physics`` / ``damage_solve``: the elastic CG, energies and gradients, and
  the damage box QP (damage_step, solver.py:160-191) on the same mesh

No CPU fallback: without the CUDA library every call raises.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from itertools import permutations
from typing import Optional

import numpy as np

from . import _lib
from .linalg import BreakdownError, LinearSolveReport, LinearSolverError
from .model import DamageModel, Material

_REGIME = {"plane_stress": 0, "plane_strain": 1, "3d": 2}


@dataclass
class UnstructuredMesh:
    """Vertices (V, d) and positively oriented elements (T, d+1); boundary tag -> vertex ids."""
    vertices: np.ndarray
    elements: np.ndarray
    boundary: dict = field(default_factory=dict)

    def __post_init__(self):
        self.vertices = np.ascontiguousarray(self.vertices, dtype=np.float64)
        self.elements = np.ascontiguousarray(self.elements, dtype=np.int64)
        d = self.vertices.shape[1]
        if d not in (2, 3) or self.elements.ndim != 2 or self.elements.shape[1] != d + 1:
            raise ValueError("UnstructuredMesh needs (V, 2) + (T, 3) or (V, 3) + (T, 4) arrays")

    @property
    def dim(self) -> int:
        return self.vertices.shape[1]

    @property
    def n_vertices(self) -> int:
        return self.vertices.shape[0]

    @property
    def n_elements(self) -> int:
        return self.elements.shape[0]


def _jitter(v, lo, hi, h, jitter, seed):
    """mesh.py:134-141: seeded uniform offsets of up to ``jitter`` cell sizes on the strictly
    interior vertices, in vertex-index order."""
    if not 0.0 <= jitter <= 0.4:
        raise ValueError(f"jitter must lie in [0, 0.4]; got {jitter}")
    if jitter > 0.0:
        interior = np.all((v > lo) & (v < hi), axis=1)
        rng = np.random.default_rng(seed)
        v[interior] += rng.uniform(-jitter, jitter, size=(int(interior.sum()), v.shape[1])) * h
    return v


def jittered_rect_mesh(L: float, H: float, h: float, jitter: float = 0.0, seed: int = 0,
                       origin_x2: float = 0.0) -> UnstructuredMesh:
    """The reference's ``rect_mesh(L, H, h, origin_x2, jitter, seed)`` (mesh.py:112-142): a
    union-jack grid (vertex (i, j) = i*(ny+1)+j, triangles as ``_grid`` mesh.py:88-99) whose
    interior vertices are jittered."""
    if L <= 0 or H <= 0 or h <= 0:
        raise ValueError(f"rect_mesh needs positive L, H, h; got L={L}, H={H}, h={h}")
    nx, ny = max(1, round(L / h)), max(1, round(H / h))
    xs = np.linspace(0.0, L, nx + 1)
    ys = np.linspace(origin_x2, origin_x2 + H, ny + 1)
    X, Y = np.meshgrid(xs, ys, indexing="ij")
    v = np.column_stack([X.ravel(), Y.ravel()])
    I, J = (a.ravel() for a in np.meshgrid(np.arange(nx), np.arange(ny), indexing="ij"))
    v00, v10, v11, v01 = I * (ny + 1) + J, (I + 1) * (ny + 1) + J, (I + 1) * (ny + 1) + J + 1, I * (ny + 1) + J + 1
    even = ((I + J) % 2 == 0)[:, None]
    t1 = np.where(even, np.column_stack([v00, v10, v11]), np.column_stack([v00, v10, v01]))
    t2 = np.where(even, np.column_stack([v00, v11, v01]), np.column_stack([v10, v11, v01]))
    v = _jitter(v, np.array([xs[0], ys[0]]), np.array([xs[-1], ys[-1]]), np.array([L / nx, H / ny]),
                jitter, seed)
    jj, ii = np.arange(ny + 1), np.arange(nx + 1)
    bnd = {"left": jj, "right": nx * (ny + 1) + jj, "bottom": ii * (ny + 1), "top": ii * (ny + 1) + ny}
    return UnstructuredMesh(v, np.vstack([t1, t2]), bnd)


def jittered_box_mesh(nx: int, ny: int, nz: int, lx: float = 1.0, ly: float = 1.0, lz: float = 1.0,
                      jitter: float = 0.0, seed: int = 0) -> UnstructuredMesh:
    """Hex grid split into 6 Kuhn tetrahedra (the structured 3D layout, vertex (i, j, k) =
    (i*(ny+1)+j)*(nz+1)+k) with the rect_mesh jitter applied to its interior vertices."""
    xs, ys, zs = (np.linspace(0.0, l, n + 1) for l, n in ((lx, nx), (ly, ny), (lz, nz)))
    X, Y, Z = np.meshgrid(xs, ys, zs, indexing="ij")
    v = np.column_stack([X.ravel(), Y.ravel(), Z.ravel()])
    I, J, K = (a.ravel() for a in np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij"))

    def vid(i, j, k):
        return (i * (ny + 1) + j) * (nz + 1) + k

    blocks = []
    for perm in permutations((0, 1, 2)):
        cur, path = [0, 0, 0], [(0, 0, 0)]
        for ax in perm:
            cur[ax] = 1
            path.append(tuple(cur))
        blocks.append(np.column_stack([vid(I + p[0], J + p[1], K + p[2]) for p in path]))
    el = np.vstack(blocks)
    p = v[el]
    neg = np.einsum("ti,ti->t", np.cross(p[:, 1] - p[:, 0], p[:, 2] - p[:, 0]), p[:, 3] - p[:, 0]) < 0
    el[neg] = el[neg][:, [0, 2, 1, 3]]
    v = _jitter(v, np.zeros(3), np.array([lx, ly, lz]), np.array([lx / nx, ly / ny, lz / nz]), jitter, seed)
    return UnstructuredMesh(v, el)


class _UDesc(C.Structure):
    _fields_ = [("dim", C.c_int32), ("regime", C.c_int32), ("model", C.c_int32), ("reserved", C.c_int32),
                ("n_vertices", C.c_int64), ("n_elements", C.c_int64),
                ("vertices", C.c_void_p), ("elements", C.c_void_p), ("E_elem", C.c_void_p),
                ("Gc_elem", C.c_void_p), ("E", C.c_double), ("nu", C.c_double), ("Gc", C.c_double),
                ("ell", C.c_double), ("k_ell", C.c_double)]


def _raise(code, handle):
    if code == _lib.PF_OK:
        return
    msg = _lib.load().pf_umesh_last_error(handle).decode(errors="replace") or f"status {code}"
    if code == _lib.PF_EBREAKDOWN:
        raise BreakdownError(msg)
    if code in (_lib.PF_EINVAL, _lib.PF_ENOWS):
        raise ValueError(msg)
    raise RuntimeError(f"CUDA failure in libphasefrac_b200: {msg}")


class UnstructuredOperators:
    """Matrix-free Kuu / Kaa on an element-list mesh (the structured ``Discretization``'s
    operators, fem.py:233-282, for meshes whose geometry is not implicit).

    ``E_elem`` / ``Gc_elem``: optional per-element absolute values (override the scalars)."""

    def __init__(self, mesh: UnstructuredMesh, material: Material,
                 damage_model: DamageModel | str = "AT1", E_elem=None, Gc_elem=None, device=None):
        import torch

        if not torch.cuda.is_available():
            raise RuntimeError("UnstructuredOperators needs a CUDA device (no CPU fallback)")
        dm = damage_model if isinstance(damage_model, DamageModel) else DamageModel(damage_model)
        if (mesh.dim == 3) != (material.regime == "3d"):
            raise ValueError(f"regime {material.regime!r} does not match a {mesh.dim}D mesh")
        self.mesh, self.material, self.damage_model = mesh, material, dm
        dev = torch.device(device or "cuda")
        self.device = dev if dev.index is not None else torch.device("cuda", torch.cuda.current_device())
        lib = _lib.load()
        Ee = None if E_elem is None else np.ascontiguousarray(E_elem, dtype=np.float64)
        Ge = None if Gc_elem is None else np.ascontiguousarray(Gc_elem, dtype=np.float64)
        for a in (Ee, Ge):
            if a is not None and a.shape != (mesh.n_elements,):
                raise ValueError("per-element fields need one value per element")
        d = _UDesc(mesh.dim, _REGIME[material.regime], 0 if dm.kind == "AT1" else 1, 0,
                   mesh.n_vertices, mesh.n_elements, mesh.vertices.ctypes.data, mesh.elements.ctypes.data,
                   None if Ee is None else Ee.ctypes.data, None if Ge is None else Ge.ctypes.data,
                   material.E, material.nu, material.Gc, material.ell, material.k_ell)
        h = C.c_void_p()
        _raise(lib.pf_umesh_create(C.byref(d), C.byref(h)), None)
        self._h = h
        nbytes = lib.pf_umesh_workspace_bytes(h)
        with torch.cuda.device(self.device):
            self._ws = torch.empty(nbytes + 256, dtype=torch.uint8, device=self.device)
            base = self._ws.data_ptr()
            self._check(lib.pf_umesh_bind_workspace(h, C.c_void_p((base + 255) & ~255), nbytes, self._stream()))
        self.workspace_bytes = int(nbytes)

    # ---- plumbing ---------------------------------------------------------------------------
    @staticmethod
    def _stream():
        import torch
        return C.c_void_p(torch.cuda.current_stream().cuda_stream)

    def _check(self, code):
        _raise(code, self._h)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and _lib._lib is not None:
            _lib._lib.pf_umesh_destroy(h)
            self._h = None

    @property
    def n_vertices(self) -> int:
        return self.mesh.n_vertices

    @property
    def n_udofs(self) -> int:
        return self.mesh.dim * self.mesh.n_vertices

    @property
    def launches(self) -> int:
        return int(_lib.load().pf_umesh_launch_count(self._h))

    def _vec(self, t, n, name):
        import torch
        if t.device != self.device or t.dtype != torch.float64 or t.numel() != n:
            raise ValueError(f"{name} must be a float64 tensor of {n} entries on {self.device}")
        return _lib.ptr(t)

    # ---- API ----------------------------------------------------------------------------------
    def set_dirichlet(self, dofs) -> None:
        """Dirichlet dofs (interleaved indices) for ``apply_Kuu(..., apply_bc=True)``."""
        d = np.ascontiguousarray(np.unique(np.asarray(dofs, dtype=np.int64)))
        self._check(_lib.load().pf_umesh_set_dirichlet(self._h, d.ctypes.data if d.size else None, d.size,
                                                        self._stream()))

    def set_eps0(self, eps0) -> None:
        """Inelastic strain per element (T x 3 Voigt in 2D, T x 6 in 3D; fem.py eps0, cases.py
        thermal_strain) as a host array or device tensor, or None: every strain of u becomes
        B u - eps0 (energies, residuals, the damage Hessian's coupling).  Kept on the device."""
        import torch
        if eps0 is None:
            self._eps0 = None
            self._check(_lib.load().pf_umesh_set_eps0(self._h, None, self._stream()))
            return
        nv = 3 if self.mesh.dim == 2 else 6
        t = torch.as_tensor(np.asarray(eps0, dtype=np.float64) if not torch.is_tensor(eps0) else eps0,
                            dtype=torch.float64, device=self.device).reshape(-1).contiguous()
        if t.numel() != nv * self.mesh.n_elements:
            raise ValueError(f"eps0 needs {nv} Voigt components per element")
        self._eps0 = t  # the library keeps the pointer: keep the tensor alive
        self._check(_lib.load().pf_umesh_set_eps0(self._h, _lib.ptr(t), self._stream()))

    def apply_Kuu(self, alpha, x, out=None, apply_bc: bool = False):
        import torch
        out = torch.empty_like(x) if out is None else out
        self._check(_lib.load().pf_umesh_apply_Kuu(
            self._h, self._vec(alpha, self.n_vertices, "alpha"), self._vec(x, self.n_udofs, "x"),
            self._vec(out, self.n_udofs, "out"), 1 if apply_bc else 0, self._stream()))
        return out

    def apply_Kaa(self, u, alpha, x, out=None):
        import torch
        out = torch.empty_like(x) if out is None else out
        self._check(_lib.load().pf_umesh_apply_Kaa(
            self._h, self._vec(u, self.n_udofs, "u"), self._vec(alpha, self.n_vertices, "alpha"),
            self._vec(x, self.n_vertices, "x"), self._vec(out, self.n_vertices, "out"), self._stream()))
        return out

    def attach_structured_twin(self, twin) -> None:
        """Use the multigrid V-cycle of a structured Discretization on the SAME grid (same vertex
        numbering, cells and Dirichlet dofs; vertices at their un-jittered positions) as the
        preconditioner of this mesh's elastic PCG (elastic_solve(precond="gmg")).  The reference's
        jitter (mesh.py:134-141) moves interior vertices by a fraction of h and keeps the union-jack
        connectivity, so the two stiffness operators are spectrally equivalent."""
        if twin.mesh.n_vertices != self.n_vertices or twin.mesh.dim != self.mesh.dim:
            raise ValueError("the structured twin must have the same vertices as the element-list mesh")
        self._twin = twin

    def _elastic_solve_gmg(self, alpha, b, out, rtol, atol, maxit):
        """PCG (cg_solve, linalg.py:106-152: x0 = 0, stop at |r| <= max(rtol |b|, atol), breakdown on
        p.Ap <= 0 or r.z <= 0) on this mesh's Kuu with z = V-cycle(structured twin) r.  Vectors and
        scalars stay on the device; one host read of |r| per iteration."""
        import torch
        from .fem import _stream
        from .linalg import BreakdownError
        twin = self._twin
        twin.call("pf_gmg_prepare", _lib.ptr(alpha), _stream())
        n = self.n_udofs
        x = out.zero_()
        r = b.clone()
        z, q = torch.empty_like(b), torch.empty_like(b)
        bnorm = float(torch.linalg.vector_norm(b))
        tol = max(rtol * bnorm, atol)
        rn = bnorm
        its = 0
        maxit = int(maxit) if maxit else 10 * n
        if rn <= tol:
            return x, LinearSolveReport(0, rn, True)
        twin.call("pf_gmg_apply", _lib.ptr(r), _lib.ptr(z), _stream())
        p = z.clone()
        rz = torch.dot(r, z)
        while its < maxit:
            self.apply_Kuu(alpha, p, out=q, apply_bc=True)
            pq = torch.dot(p, q)
            gamma = rz / pq
            x.addcmul_(p, gamma)
            r.addcmul_(q, gamma, value=-1.0)
            its += 1
            rn, pqh, rzh = (float(v) for v in torch.stack([torch.linalg.vector_norm(r), pq, rz]).tolist())
            if not pqh > 0.0 or not rzh > 0.0:
                raise BreakdownError(f"elastic PCG breakdown (p.Ap = {pqh:.3e}, r.z = {rzh:.3e})")
            if rn <= tol:
                break
            twin.call("pf_gmg_apply", _lib.ptr(r), _lib.ptr(z), _stream())
            rz_new = torch.dot(r, z)
            p.mul_(rz_new / rz).add_(z)
            rz = rz_new
        return x, LinearSolveReport(its, rn, rn <= tol)

    def elastic_solve(self, alpha, b, out=None, rtol: float = 1e-8, atol: float = 0.0, maxit: int = 0,
                      check_every: int = 10, raise_on_failure: bool = True, precond: str = "jacobi"):
        """x with Kuu(alpha) x = b, Dirichlet rows/cols eliminated, by device Jacobi PCG from
        x0 = 0 (cg_solve, linalg.py:106-152).  Returns (x, LinearSolveReport); non-convergence
        raises LinearSolverError "elastic CG stalled" as solver.py:139-141 unless
        raise_on_failure is False.  ``precond="gmg"``: the V-cycle of an attached structured twin
        (attach_structured_twin) instead of Jacobi."""
        import torch
        out = torch.empty_like(b) if out is None else out
        if precond == "gmg":
            if getattr(self, "_twin", None) is None:
                raise ValueError("precond='gmg' needs attach_structured_twin() first")
            x, report = self._elastic_solve_gmg(alpha, b, out, float(rtol), float(atol), maxit)
            if raise_on_failure and not report.converged:
                raise LinearSolverError(f"elastic CG stalled after {report.iterations} iterations "
                                        f"(|r| = {report.final_residual_norm:.3e})")
            return x, report
        if precond != "jacobi":
            raise ValueError(f"unknown preconditioner {precond!r}")
        o = _lib.LinOpts(precond=_lib.PREC["jacobi"], warm_start=0, maxit=int(maxit), rtol=float(rtol),
                         atol=float(atol), check_every=int(check_every))
        rep = _lib.LinReport()
        self._check(_lib.load().pf_umesh_elastic_solve(
            self._h, self._vec(alpha, self.n_vertices, "alpha"), self._vec(b, self.n_udofs, "b"),
            self._vec(out, self.n_udofs, "out"), C.byref(o), C.byref(rep), self._stream()))
        report = LinearSolveReport(int(rep.iterations), float(rep.final_residual_norm), bool(rep.converged))
        if raise_on_failure and not rep.converged:
            raise LinearSolverError(f"elastic CG stalled after {rep.iterations} iterations "
                                    f"(|r| = {rep.final_residual_norm:.3e})")
        return out, report

    def physics(self, u, alpha, want_residuals: bool = True):
        """(EnergyBreakdown-like (elastic, surface, total), r_u raw, r_alpha) at (u, alpha):
        assemble_energy / assemble_residual_u(apply_bc=False) / assemble_residual_alpha
        (fem.py:162-218) on the element-list mesh."""
        import torch
        ru = torch.empty_like(u) if want_residuals else None
        ra = torch.empty_like(alpha) if want_residuals else None
        en = (C.c_double * 3)()
        self._check(_lib.load().pf_umesh_physics(
            self._h, self._vec(u, self.n_udofs, "u"), self._vec(alpha, self.n_vertices, "alpha"),
            None if ru is None else _lib.ptr(ru), None if ra is None else _lib.ptr(ra), en, self._stream()))
        return (float(en[0]), float(en[1]), float(en[2])), ru, ra

    def damage_solve(self, u, alpha_lb, alpha, out=None, config=None, raise_on_failure: bool = True):
        """alpha_out = rsls solution of the damage box QP at fixed u (damage_step, solver.py:160-191;
        rsls vi.py:187-264): min E(u, a) over alpha_lb <= a <= 1 from clip(alpha).  Reduced-space
        active set with a device Jacobi-PCG inner solve.  Returns (alpha_out, ActiveSetReport);
        non-convergence raises VISolverError-like RuntimeError unless raise_on_failure is False."""
        import torch
        from .vi import ActiveSetReport, VIConfig
        cfg = config or VIConfig()
        out = torch.empty_like(alpha) if out is None else out
        o = cfg.to_c()
        rep = _lib.VIReport()
        self._check(_lib.load().pf_umesh_damage_solve(
            self._h, self._vec(u, self.n_udofs, "u"), self._vec(alpha_lb, self.n_vertices, "alpha_lb"),
            self._vec(alpha, self.n_vertices, "alpha"), self._vec(out, self.n_vertices, "out"),
            C.byref(o), C.byref(rep), self._stream()))
        report = ActiveSetReport.from_c(rep)
        if raise_on_failure and not report.converged:
            raise RuntimeError(f"damage VI did not converge in {report.iterations} iterations "
                               f"(|Phi| = {report.final_residual_norm:.3e})")
        return out, report

    def am_load_step(self, u, alpha, alpha_lb, bc_dofs, bc_values, omega: float = 1.0,
                     outer_atol: float = 1e-7, max_am_iterations: int = 1000,
                     elastic_rtol: float = 1e-10, damage_atol_factor: float = 0.1,
                     max_vi_iterations: int = 200, log_callback=None, elastic_precond: str = "jacobi"):
        """One load step of alternate minimisation on the element-list mesh (am_loop with an
        absolute target, solver.py:129-241; oracle/am.py am_loop): elastic half-step (device PCG on
        the Dirichlet-lifted Kuu), over-relaxed update u0 + omega (u* - u0), damage half-step
        (``damage_solve``), relaxed damage with midpoint backtracking (relax_damage,
        solver.py:202-215), until |(r_u with Dirichlet rows zero, Phi_FB(alpha, r_alpha))| <=
        outer_atol.  Updates u and alpha in place; returns a dict of step statistics.  No body
        force / inelastic strain on this path."""
        import torch
        from .vi import VIConfig
        dofs = torch.as_tensor(np.asarray(bc_dofs, dtype=np.int64), device=u.device)
        vals = torch.as_tensor(np.asarray(bc_values, dtype=np.float64), device=u.device)
        self.set_dirichlet(np.asarray(bc_dofs, dtype=np.int64))
        g = torch.zeros_like(u)
        g[dofs] = vals
        u[dofs] = vals
        one = torch.ones_like(alpha)
        vcfg = VIConfig(abs_tol=damage_atol_factor * outer_atol, max_iterations=max_vi_iterations)

        def residual():
            en, ru, ra = self.physics(u, alpha)
            ru[dofs] = 0.0
            x = alpha - alpha_lb
            y = one - alpha
            inner = torch.hypot(y, ra) - y + ra          # fb(hi - x, -F)
            phi = torch.hypot(x, inner) - x - inner      # fb(x - lo, inner)
            return float(torch.sqrt(torch.sum(ru * ru) + torch.sum(phi * phi))), en

        res, en = residual()
        stats = {"converged": False, "am_iterations": 0, "krylov_iterations": 0,
                 "omega_bar_min": omega, "residual_history": [res], "energy_history": [en],
                 "vi_unconverged": 0, "vi_steepest_descent_steps": 0}
        # at least one AM iteration, as the reference loop (solver.py:186-241; oracle am_loop)
        while stats["am_iterations"] < max_am_iterations:
            stats["am_iterations"] += 1
            # lifted right-hand side -r_u(g) = f - K g (f: the inelastic-strain load,
            # assemble_load_u fem.py:192-199), Dirichlet rows = the prescribed values
            _, b, _ = self.physics(g, alpha)
            b.neg_()
            b[dofs] = vals
            us, lrep = self.elastic_solve(alpha, b, rtol=elastic_rtol, precond=elastic_precond)
            stats["krylov_iterations"] += lrep.iterations
            u.add_(omega * (us - u))
            u[dofs] = vals
            a0 = alpha.clone()
            # an unconverged damage VI returns its iterate and the AM loop carries on, as the
            # reference damage_step (solver.py:145-160)
            a_star, vrep = self.damage_solve(u, alpha_lb, alpha, config=vcfg, raise_on_failure=False)
            stats["krylov_iterations"] += vrep.total_krylov_iterations
            stats["vi_unconverged"] += 0 if vrep.converged else 1
            stats["vi_steepest_descent_steps"] += vrep.steepest_descent_steps
            wb, cand, k = omega, a_star, 0
            if wb != 1.0:
                cand = a0 + wb * (a_star - a0)
                while bool(torch.any(cand < alpha_lb)) or bool(torch.any(cand > 1.0)):
                    wb = 0.5 * (1.0 + wb)
                    k += 1
                    if k >= 60 or wb == 1.0:
                        wb, cand = 1.0, a_star
                        break
                    cand = a0 + wb * (a_star - a0)
            alpha.copy_(torch.minimum(torch.maximum(cand, alpha_lb), one))
            stats["omega_bar_min"] = min(stats["omega_bar_min"], wb)
            res, en = residual()
            stats["residual_history"].append(res)
            stats["energy_history"].append(en)
            if log_callback is not None:  # the AM log record of solver.py:226-233
                log_callback({"phase": "am", "cycle": 0, "iteration": stats["am_iterations"], "residual": res,
                              "omega_bar": wb, "elastic": en[0], "dissipated": en[1], "total": en[2]})
            stats["converged"] = res <= outer_atol
            if stats["converged"]:
                break
        stats["final_residual_norm"] = stats["residual_history"][-1]
        return stats
