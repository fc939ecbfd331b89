"""Device-resident P1 discretisation (reference fem.py), backed by libphasefrac_b200.so.

``Discretization`` owns one C-ABI context plus its PyTorch-allocated workspace; all
fields are ``torch.float64`` CUDA tensors in the reference layout (fem.py:35-55,
mesh.py:3-10).  The assembly functions keep the reference names and signatures but
are matrix-free: ``assemble_Kuu`` & co. return operator objects whose ``matvec`` /
``@`` runs the sm_100a kernels, instead of scipy CSR matrices.
"""

from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import NamedTuple, Optional

import numpy as np
import torch

from . import _lib
from .mesh import StructuredMesh
from .model import DamageModel, Material


class EnergyBreakdown(NamedTuple):
    elastic: float
    dissipated: float
    total: float


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


@dataclass
class State:
    """Solution fields plus the irreversibility floor and the current load (fem.py:35-55)."""

    u: torch.Tensor
    alpha: torch.Tensor
    alpha_lb: torch.Tensor
    load: float = 0.0

    @classmethod
    def zeros(cls, mesh, alpha_lb=None, device="cuda") -> "State":
        n = mesh.n_vertices
        d = getattr(mesh, "dim", 2)
        if alpha_lb is None:
            lb = torch.zeros(n, dtype=torch.float64, device=device)
        else:
            lb = torch.as_tensor(np.asarray(alpha_lb, dtype=float), dtype=torch.float64,
                                 device=device).clone()
        return cls(u=torch.zeros(d * n, dtype=torch.float64, device=device), alpha=lb.clone(),
                   alpha_lb=lb, load=0.0)

    @classmethod
    def from_numpy(cls, u, alpha, alpha_lb, load=0.0, device="cuda") -> "State":
        t = lambda a: torch.as_tensor(np.ascontiguousarray(a, dtype=float), device=device).clone()
        return cls(t(u), t(alpha), t(alpha_lb), load)

    def copy(self) -> "State":
        return State(self.u.clone(), self.alpha.clone(), self.alpha_lb.clone(), self.load)

    def numpy(self):
        return (self.u.cpu().numpy(), self.alpha.cpu().numpy(), self.alpha_lb.cpu().numpy())

    def check_feasible(self, tol: float = 1e-12) -> None:
        bad = bool(((self.alpha < self.alpha_lb - tol) | (self.alpha > 1.0 + tol)).any())
        if bad:
            raise ValueError("state violates alpha_lb <= alpha <= 1")


@dataclass
class DirichletBC:
    """Prescribed values on displacement dofs (fem.py:58-90); host arrays, uploaded on
    assignment to ``Discretization.bc``."""

    dofs: np.ndarray
    values: np.ndarray

    def __post_init__(self):
        dofs = np.asarray(self.dofs, dtype=np.int64).ravel()
        values = np.asarray(self.values, dtype=float).ravel()
        if dofs.shape != values.shape:
            raise ValueError("dofs and values must have matching shapes")
        order = np.argsort(dofs, kind="stable")
        dofs, values = dofs[order], values[order]
        dup = dofs[1:] == dofs[:-1]
        if np.any(dup):
            bad = dup & (values[1:] != values[:-1])
            if np.any(bad):
                raise ValueError(f"conflicting Dirichlet values on dof {dofs[1:][bad][0]}")
            keep = np.concatenate([[True], ~dup])
            dofs, values = dofs[keep], values[keep]
        self.dofs, self.values = dofs, values


def combine_bcs(*bcs: DirichletBC) -> DirichletBC:
    return DirichletBC(np.concatenate([b.dofs for b in bcs]), np.concatenate([b.values for b in bcs]))


class Discretization:
    """Mesh + material bound to a device context (fem.py:93-156).

    ``bc`` and ``eps0_rows`` are the mutable per-load-step inputs.  ``E_cell`` /
    ``Gc_cell`` are optional per-cell fields (n_cells, I-major).  ``solvers="operators"`` plans
    no multigrid hierarchy and no Newton vectors (operator applies and the Jacobi/VI solvers only).
    """

    def __init__(self, mesh: StructuredMesh, material: Material,
                 damage: Optional[DamageModel] = None, E_cell=None, Gc_cell=None,
                 device: str = "cuda", solvers: str = "all"):
        self.lib = _lib.load()
        self.mesh = mesh
        self.material = material
        self.damage = damage or DamageModel()
        self.device = torch.device(device)
        dim = getattr(mesh, "dim", 2)
        if (material.regime == "3d") != (dim == 3):
            raise ValueError("3D meshes need Material(regime='3d') and vice versa")
        d = _lib.PfDesc(dim=dim, pattern=_lib.PATTERNS[mesh.pattern],
                        regime=_lib.REGIMES[material.regime], model=_lib.MODELS[self.damage.kind],
                        nx=mesh.nx, ny=mesh.ny, nz=getattr(mesh, "nz", 0), lx=mesh.lx, ly=mesh.ly,
                        lz=getattr(mesh, "lz", 0.0), E=material.E, nu=material.nu, Gc=material.Gc,
                        ell=material.ell, k_ell=material.k_ell,
                        skip=0 if solvers == "all" else _lib.SKIP_GMG | _lib.SKIP_NEWTON)
        if solvers not in ("all", "operators"):
            raise ValueError("solvers must be 'all' or 'operators'")
        self.dim = dim
        ctx = C.c_void_p()
        _lib.raise_for(self.lib.pf_ctx_create(C.byref(d), C.byref(ctx)), None)
        self._ctx = ctx
        q = (C.c_int64 * 8)()
        self.lib.pf_query(ctx, q)
        self.n_vertices, self.n_udofs, self.n_elements, self.n_cells = q[0], q[1], q[2], q[3]
        nbytes = int(self.lib.pf_workspace_bytes(ctx))
        self._ws = torch.empty(nbytes + 512, dtype=torch.uint8, device=self.device)
        base = (self._ws.data_ptr() + 255) & ~255
        _lib.raise_for(self.lib.pf_bind_workspace(ctx, C.c_void_p(base), nbytes), ctx)
        self._E = self._field(E_cell)
        self._Gc = self._field(Gc_cell)
        _lib.raise_for(self.lib.pf_set_cell_fields(ctx, _lib.ptr(self._E), _lib.ptr(self._Gc)), ctx)
        rows = getattr(mesh, "row_heights", None)
        if rows is not None:  # graded rows (banded_rect_mesh)
            hy = np.ascontiguousarray(rows, dtype=np.float64)
            _lib.raise_for(self.lib.pf_set_row_heights(ctx, hy.ctypes.data_as(C.c_void_p), _stream()), ctx)
        self._bc: Optional[DirichletBC] = None
        self._eps0_rows: Optional[np.ndarray] = None
        self._guarded = bool(os.environ.get("PF_WS_GUARD"))  # read by pf_ctx_create as well

    def ws_guarded(self) -> bool:
        """True when the context was created with workspace guard zones (PF_WS_GUARD=1, a
        bounds-check aid; pf_check_guards counts overwritten guard bytes)."""
        return self._guarded

    def _field(self, f):
        if f is None:
            return None
        t = torch.as_tensor(np.asarray(f, dtype=float), dtype=torch.float64, device=self.device)
        if t.numel() != self.mesh.n_cells:
            raise ValueError("per-cell fields need n_cells entries")
        return t.contiguous()

    def __del__(self):
        try:
            if getattr(self, "_ctx", None):
                self.lib.pf_ctx_destroy(self._ctx)
                self._ctx = None
        except Exception:  # noqa: BLE001
            pass

    @property
    def ctx(self):
        return self._ctx

    def call(self, name, *args):
        _lib.raise_for(getattr(self.lib, name)(self._ctx, *args), self._ctx)

    # per-step data -------------------------------------------------------------------
    @property
    def bc(self) -> Optional[DirichletBC]:
        return self._bc

    @bc.setter
    def bc(self, bc: Optional[DirichletBC]):
        if bc is None:
            self.call("pf_set_dirichlet", None, None, 0, _stream())
            self._bc = None
            return
        dofs = np.ascontiguousarray(bc.dofs, dtype=np.int64)
        vals = np.ascontiguousarray(bc.values, dtype=np.float64)
        self.call("pf_set_dirichlet", dofs.ctypes.data_as(C.c_void_p),
                  vals.ctypes.data_as(C.c_void_p), int(dofs.size), _stream())
        self._bc = bc
        self._bc_dofs_dev = torch.as_tensor(dofs, device=self.device)
        self._bc_vals_dev = torch.as_tensor(vals, device=self.device)

    @property
    def eps0_rows(self) -> Optional[np.ndarray]:
        return self._eps0_rows

    @eps0_rows.setter
    def eps0_rows(self, table):
        """Isotropic inelastic strain e per (element type, cell row): eps0 = e (1, 1, 0)."""
        if table is None:
            self.call("pf_set_eps0_rows", None, _stream())
            self._eps0_rows = None
            return
        t = np.zeros((4, self.mesh.ny))
        a = np.asarray(table, dtype=float)
        t[: a.shape[0]] = a
        t = np.ascontiguousarray(t)
        self.call("pf_set_eps0_rows", t.ctypes.data_as(C.c_void_p), _stream())
        self._eps0_rows = a

    def launches(self) -> int:
        return int(self.lib.pf_launch_count(self._ctx))


def _empty(problem, n):
    return torch.empty(n, dtype=torch.float64, device=problem.device)


def physics(state: State, problem: Discretization, rows: int = _lib.ROWS_ZERO,
            want_ru=False, want_ra=False, want_phi=False):
    """One fused pass: energies, r_u, r_alpha, Phi and their norms (host floats)."""
    ru = _empty(problem, problem.n_udofs) if want_ru else None
    ra = _empty(problem, problem.n_vertices) if want_ra else None
    ph = _empty(problem, problem.n_vertices) if want_phi else None
    out = (C.c_double * 8)()
    problem.call("pf_physics", _lib.ptr(state.u), _lib.ptr(state.alpha), _lib.ptr(state.alpha_lb),
                 _lib.ptr(ru), _lib.ptr(ra), _lib.ptr(ph), rows, out, _stream())
    return list(out), ru, ra, ph


def assemble_energy(state: State, problem: Discretization) -> EnergyBreakdown:
    """Elastic / dissipated / total energy (fem.py:162-174)."""
    out, *_ = physics(state, problem)
    return EnergyBreakdown(out[0], out[1], out[2])


def assemble_residual_u(state: State, problem: Discretization, apply_bc: bool = True):
    """dE/du; Dirichlet rows replaced by u - ubar when apply_bc (fem.py:177-189)."""
    _, ru, _, _ = physics(state, problem, _lib.ROWS_VALUE if apply_bc else _lib.ROWS_RAW,
                          want_ru=True)
    return ru


def assemble_residual_alpha(state: State, problem: Discretization):
    """dE/dalpha (fem.py:202-218)."""
    _, _, ra, _ = physics(state, problem, _lib.ROWS_RAW, want_ra=True)
    return ra


def assemble_load_u(state: State, problem: Discretization):
    """Inelastic-strain load vector f (fem.py:192-199)."""
    f = _empty(problem, problem.n_udofs)
    problem.call("pf_load_u", _lib.ptr(state.alpha), _lib.ptr(f), _stream())
    return f


class DeviceOperator:
    """Matrix-free stand-in for an assembled block: ``op @ x`` / ``op.matvec(x)``."""

    def __init__(self, problem, shape, fn):
        self.problem, self.shape, self._fn = problem, shape, fn

    def matvec(self, x):
        x = x.contiguous()
        y = _empty(self.problem, self.shape[0])
        self._fn(x, y)
        return y

    __matmul__ = matvec


def assemble_Kuu(state: State, problem: Discretization, apply_bc: bool = True) -> DeviceOperator:
    """Degraded elasticity operator, Dirichlet rows/cols eliminated when apply_bc (fem.py:233-243)."""
    a = state.alpha.clone()
    mode = _lib.BC_ELIMINATE if (apply_bc and problem.bc is not None) else _lib.BC_NONE
    n = problem.n_udofs
    return DeviceOperator(problem, (n, n), lambda x, y: problem.call(
        "pf_apply_Kuu", _lib.ptr(a), _lib.ptr(x), _lib.ptr(y), mode, _stream()))


def assemble_Kua(state: State, problem: Discretization, apply_bc: bool = True) -> DeviceOperator:
    """Mixed block d r_u / d alpha, Dirichlet rows zeroed (fem.py:246-263)."""
    u, a = state.u.clone(), state.alpha.clone()
    mode = _lib.BC_ELIMINATE if (apply_bc and problem.bc is not None) else _lib.BC_NONE
    op = DeviceOperator(problem, (problem.n_udofs, problem.n_vertices), lambda x, y: problem.call(
        "pf_apply_Kua", _lib.ptr(u), _lib.ptr(a), _lib.ptr(x), _lib.ptr(y), mode, _stream()))
    op.T = DeviceOperator(problem, (problem.n_vertices, problem.n_udofs), lambda x, y: problem.call(
        "pf_apply_Kau", _lib.ptr(u), _lib.ptr(a), _lib.ptr(x), _lib.ptr(y), mode, _stream()))
    return op


def assemble_Kaa(state: State, problem: Discretization) -> DeviceOperator:
    """Damage block (fem.py:266-276; AT2 adds the w'' reaction).  The "assembly" is one pass
    computing the per-element reaction coefficients at the current u (the block does not
    depend on alpha); applies then read only x and those coefficients."""
    kappa = _empty(problem, problem.n_elements)
    problem.call("pf_kaa_coefficients", _lib.ptr(state.u), _lib.ptr(kappa), None, _stream())
    n = problem.n_vertices
    return DeviceOperator(problem, (n, n), lambda x, y: problem.call(
        "pf_apply_Kaa_coef", _lib.ptr(kappa), _lib.ptr(x), _lib.ptr(y), _stream()))
