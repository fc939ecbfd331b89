"""CPU oracle for the phase-field fracture load step -- TEST INFRASTRUCTURE ONLY.

This package is a plain numpy/scipy restatement of the reference package
``phasefrac`` (Farrell & Maurini, arXiv:1511.08463; reference tree
``/root/reference/pkg/src/phasefrac``) extended with the physics the
BASELINE configs need and the reference lacks (AT2, plane strain, right /
crossed triangle patterns, 3D Kuhn tetrahedra, per-cell E / Gc fields,
isotropic y-profile inelastic strain, absolute Newton switch).

Rules ("Oracle"):

* Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU
  baseline / ``--impl reference`` arm may import this package, and only as
  the checker or the timed CPU baseline -- never as part of the product path.
  The product package ``paper_1511_08463_b200`` never imports it.
* Parity is pinned: ``tests/golden/make_golden.py`` runs the reference
  itself (importable in the build container) and commits its outputs under
  ``tests/golden/``; ``tests/test_oracle_golden.py`` checks this oracle
  against them.  Where the oracle extends the reference (AT2, plane strain,
  3D, other patterns) it is pinned by finite-difference consistency and
  closed-form energies (``tests/test_oracle_fd.py``).

Each function cites the reference file:line it restates (paths relative to
``/root/reference/pkg/src/phasefrac``).
"""

from .meshgen import (PATTERNS, SimplexMesh, grid_mesh, kuhn_mesh)  # noqa: F401
from .p1 import (P1Model, MaterialSpec, EnergyParts)  # noqa: F401
