"""ctypes binding of libphasefrac_b200.so (the C ABI in include/phasefrac_b200.h).

The product path has no CPU fallback: if the shared library is missing or fails to
load, every entry point raises.  Status codes map to the reference exception classes
(linalg.py:21-43, solver.py:139-141).
"""

from __future__ import annotations

import ctypes as C
import os

from .linalg import (BreakdownError, InnerSolverError, LinearSolverError)

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libphasefrac_b200.so")

PF_OK, PF_EINVAL, PF_ECUDA, PF_EBREAKDOWN, PF_ESTALL, PF_EINNER, PF_ENOWS = range(7)
PATTERNS = {"union_jack": 0, "right": 1, "crossed": 2, "kuhn6": 3}
REGIMES = {"plane_stress": 0, "plane_strain": 1, "3d": 2}
MODELS = {"AT1": 0, "AT2": 1}
BC_NONE, BC_ELIMINATE = 0, 1
ROWS_RAW, ROWS_ZERO, ROWS_VALUE = 0, 1, 2
PREC = {"jacobi": 0, "gmg": 1}


class PfDesc(C.Structure):
    _fields_ = [("dim", C.c_int32), ("pattern", C.c_int32), ("regime", C.c_int32),
                ("model", C.c_int32), ("nx", C.c_int64), ("ny", C.c_int64), ("nz", C.c_int64),
                ("lx", C.c_double), ("ly", C.c_double), ("lz", C.c_double),
                ("E", C.c_double), ("nu", C.c_double), ("Gc", C.c_double), ("ell", C.c_double),
                ("k_ell", C.c_double), ("skip", C.c_int32), ("reserved", C.c_int32)]

SKIP_GMG, SKIP_NEWTON = 1, 2


class LinOpts(C.Structure):
    _fields_ = [("precond", C.c_int32), ("warm_start", C.c_int32), ("maxit", C.c_int64),
                ("rtol", C.c_double), ("atol", C.c_double), ("check_every", C.c_int32),
                ("gmg_levels", C.c_int32), ("cheb_degree", C.c_int32), ("gmg_reuse", C.c_int32)]


class LinReport(C.Structure):
    _fields_ = [("iterations", C.c_int64), ("final_residual_norm", C.c_double),
                ("b_norm", C.c_double), ("converged", C.c_int32), ("status", C.c_int32)]


class VIOpts(C.Structure):
    _fields_ = [("abs_tol", C.c_double), ("max_iterations", C.c_int32), ("precond", C.c_int32),
                ("ls_backtrack", C.c_double), ("ls_min_step", C.c_double), ("armijo", C.c_double),
                ("inner_rtol", C.c_double), ("inner_maxit", C.c_int64), ("zero_tol", C.c_double),
                ("fieldsplit_rtol", C.c_double), ("inner_cycles", C.c_int32),
                ("inner_mode", C.c_int32)]


class VIReport(C.Structure):
    _fields_ = [("iterations", C.c_int32), ("converged", C.c_int32),
                ("final_residual_norm", C.c_double), ("total_krylov_iterations", C.c_int64),
                ("steepest_descent_steps", C.c_int32), ("linear_failures", C.c_int32),
                ("status", C.c_int32), ("n_history", C.c_int32), ("history", C.c_double * 64)]


EXPORTS = {
    # name: (restype, argtypes)
    "pf_ctx_create": (C.c_int, [C.POINTER(PfDesc), C.POINTER(C.c_void_p)]),
    "pf_ctx_destroy": (None, [C.c_void_p]),
    "pf_last_error": (C.c_char_p, [C.c_void_p]),
    "pf_query": (C.c_int, [C.c_void_p, C.POINTER(C.c_int64)]),
    "pf_workspace_bytes": (C.c_int64, [C.c_void_p]),
    "pf_bind_workspace": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64]),
    "pf_set_cell_fields": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "pf_set_dirichlet": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]),
    "pf_set_eps0_rows": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "pf_set_row_heights": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "pf_apply_Kuu": (C.c_int, [C.c_void_p] * 4 + [C.c_int32, C.c_void_p]),
    "pf_apply_Kaa": (C.c_int, [C.c_void_p] * 5 + [C.c_void_p]),
    "pf_kaa_coefficients": (C.c_int, [C.c_void_p] * 5),
    "pf_apply_Kaa_coef": (C.c_int, [C.c_void_p] * 5),
    "pf_apply_Kua": (C.c_int, [C.c_void_p] * 5 + [C.c_int32, C.c_void_p]),
    "pf_apply_Kau": (C.c_int, [C.c_void_p] * 5 + [C.c_int32, C.c_void_p]),
    "pf_physics": (C.c_int, [C.c_void_p] * 7 + [C.c_int32, C.c_void_p, C.c_void_p]),
    "pf_load_u": (C.c_int, [C.c_void_p] * 3 + [C.c_void_p]),
    "pf_elastic_solve": (C.c_int, [C.c_void_p] * 4 + [C.POINTER(LinOpts), C.POINTER(LinReport),
                                                       C.c_void_p]),
    "pf_gmg_prepare": (C.c_int, [C.c_void_p] * 3),
    "pf_gmg_apply": (C.c_int, [C.c_void_p] * 4),
    "pf_damage_solve": (C.c_int, [C.c_void_p] * 5 + [C.POINTER(VIOpts), C.POINTER(VIReport),
                                                      C.c_void_p]),
    "pf_relax_u": (C.c_int, [C.c_void_p] * 3 + [C.c_double, C.c_void_p, C.c_void_p]),
    "pf_relax_alpha": (C.c_int, [C.c_void_p] * 4 + [C.c_double, C.c_void_p, C.c_void_p,
                                                     C.c_void_p]),
    "pf_relax_alpha_physics": (C.c_int, [C.c_void_p] * 5 + [C.c_double] + [C.c_void_p] * 4),
    "pf_snap_bc": (C.c_int, [C.c_void_p] * 3),
    "pf_newton": (C.c_int, [C.c_void_p] * 6 + [C.POINTER(VIOpts), C.POINTER(VIReport),
                                                C.c_void_p]),
    "pf_launch_count": (C.c_int64, [C.c_void_p]),
    "pf_check_guards": (C.c_int, [C.c_void_p, C.POINTER(C.c_int64), C.c_void_p]),
    "pf_profile": (C.c_int, [C.c_void_p, C.c_int32]),
    "pf_profile_read": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32]),
    # element-list meshes (umesh.py)
    "pf_umesh_create": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p)]),
    "pf_umesh_destroy": (None, [C.c_void_p]),
    "pf_umesh_last_error": (C.c_char_p, [C.c_void_p]),
    "pf_umesh_workspace_bytes": (C.c_int64, [C.c_void_p]),
    "pf_umesh_bind_workspace": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]),
    "pf_umesh_set_dirichlet": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]),
    "pf_umesh_set_eps0": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "pf_umesh_apply_Kuu": (C.c_int, [C.c_void_p] * 4 + [C.c_int32, C.c_void_p]),
    "pf_umesh_apply_Kaa": (C.c_int, [C.c_void_p] * 5 + [C.c_void_p]),
    "pf_umesh_elastic_solve": (C.c_int, [C.c_void_p] * 4 + [C.POINTER(LinOpts), C.POINTER(LinReport),
                                                             C.c_void_p]),
    "pf_umesh_physics": (C.c_int, [C.c_void_p] * 6 + [C.c_void_p]),
    "pf_umesh_damage_solve": (C.c_int, [C.c_void_p] * 5 + [C.POINTER(VIOpts), C.POINTER(VIReport),
                                                         C.c_void_p]),
    "pf_umesh_launch_count": (C.c_int64, [C.c_void_p]),
}
KERNEL_KINDS = ["Kuu", "Kuu_cg", "Kuu_diag", "kappa", "Kaa", "Kaa_cg", "Kaa_diag", "Kaa_trial",
                "physics", "rhs", "Kua", "Kau", "jacobian", "cg_vec", "vec", "gmg_cycle", "gmg_setup"]

_lib = None


def load():
    """Load (building first when the sources are newer) and type the library."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        try:
            from . import build as _b
            _b.build()
        except Exception as exc:  # noqa: BLE001
            raise ImportError(f"libphasefrac_b200.so is missing and could not be built: {exc}")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in EXPORTS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def raise_for(code: int, ctx) -> None:
    if code == PF_OK:
        return
    msg = load().pf_last_error(ctx).decode(errors="replace") or f"status {code}"
    if code == PF_EBREAKDOWN:
        raise BreakdownError(msg)
    if code == PF_ESTALL:
        raise LinearSolverError(msg)
    if code == PF_EINNER:
        raise InnerSolverError("?", RuntimeError(msg))
    if code in (PF_EINVAL, PF_ENOWS):
        raise ValueError(msg)
    raise RuntimeError(f"CUDA failure in libphasefrac_b200: {msg}")


def ptr(t) -> int:
    """Raw device pointer of a contiguous tensor (None -> NULL)."""
    if t is None:
        return None
    if not t.is_contiguous():
        raise ValueError("device buffers must be contiguous")
    return t.data_ptr()
