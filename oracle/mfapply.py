"""ctypes front end of oracle/mfapply.c -- ORACLE (test infrastructure only).

Matrix-free CPU restatement of the assembled oracle SpMV (oracle/p1.py ``Kuu`` / ``Kaa``;
reference fem.py:233-276) for the config-5 check at sizes the assembled matrix cannot reach.
``build()`` compiles oracle/_c/libpf_oracle_mf.so with gcc (-O2 -fopenmp); it is called by
``__graft_entry__.build()`` so the library travels to the GPU box with the snapshot.
Validated against the assembled oracle in tests/test_oracle_mf.py.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "mfapply.c")
LIB = os.path.join(HERE, "_c", "libpf_oracle_mf.so")
_PAT = {"union_jack": 0, "right": 1, "crossed": 2}
_REG = {"plane_stress": 0, "plane_strain": 1, "3d": 2}


class _Mat(C.Structure):
    _fields_ = [("E", C.c_double), ("nu", C.c_double), ("Gc", C.c_double), ("ell", C.c_double),
                ("k_ell", C.c_double), ("model", C.c_int), ("regime", C.c_int)]


def build(force: bool = False) -> str:
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= os.path.getmtime(SRC):
        return LIB
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    subprocess.run(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", SRC, "-o", LIB + ".tmp", "-lm"],
                   check=True)
    os.replace(LIB + ".tmp", LIB)
    return LIB


_lib = None


def _load():
    global _lib
    if _lib is None:
        lib = C.CDLL(build())
        dp = C.POINTER(C.c_double)
        lib.pf_oracle_mf_2d.argtypes = [C.c_int, C.c_int, C.c_long, C.c_long, C.c_double, C.c_double,
                                        C.POINTER(_Mat), dp, dp, dp, dp, C.c_int]
        lib.pf_oracle_mf_3d.argtypes = [C.c_int, C.c_long, C.c_long, C.c_long, C.c_double, C.c_double,
                                        C.c_double, C.POINTER(_Mat), dp, dp, dp, dp, C.c_int]
        _lib = lib
    return _lib


def _p(a):
    if a is None:
        return None
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _c(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.float64)


def apply(op: str, shape, extent, pattern: str, spec, alpha=None, u=None, x=None, threads: int = 0):
    """y = Kuu(alpha) x (op "Kuu") or Kaa(u) x (op "Kaa") without Dirichlet elimination.

    ``shape`` = (nx, ny) or (nx, ny, nz) cells, ``extent`` = (lx, ly[, lz]), ``spec`` an
    oracle.p1.MaterialSpec (scalar E and Gc)."""
    lib = _load()
    m = _Mat(spec.E, spec.nu, spec.Gc, spec.ell, spec.k_ell, 0 if spec.model == "AT1" else 1,
             _REG[spec.regime])
    threads = threads or os.cpu_count() or 1
    alpha, u, x = _c(alpha), _c(u), _c(x)
    kop = 0 if op == "Kuu" else 1
    if len(shape) == 2:
        nx, ny = shape
        nv = (nx + 1) * (ny + 1) + (nx * ny if pattern == "crossed" else 0)
        y = np.empty(nv * (2 if kop == 0 else 1))
        lib.pf_oracle_mf_2d(kop, _PAT[pattern], nx, ny, extent[0], extent[1], C.byref(m), _p(alpha),
                            _p(u), _p(x), _p(y), threads)
    else:
        nx, ny, nz = shape
        nv = (nx + 1) * (ny + 1) * (nz + 1)
        y = np.empty(nv * (3 if kop == 0 else 1))
        lib.pf_oracle_mf_3d(kop, nx, ny, nz, extent[0], extent[1], extent[2], C.byref(m), _p(alpha),
                            _p(u), _p(x), _p(y), threads)
    return y
