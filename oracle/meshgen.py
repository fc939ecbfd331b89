"""Structured simplex meshes for the oracle (test infrastructure only).

Vertex numbering and element order follow the reference layout contract
(``mesh.py:3-10, 78-109``): grid vertex (i, j) is ``i*(ny+1) + j``; triangles
are stored type-major (all first triangles of the cells in I-major order,
then all second triangles, ...).  The union-jack pattern reproduces the
reference's ``_grid`` exactly (``mesh.py:95-99``).  Extensions:

* ``right``   -- every cell split along its v00-v11 diagonal;
* ``crossed`` -- every cell split into 4 triangles around a centre vertex;
  centre vertices are appended after the (nx+1)(ny+1) corner vertices with
  index ``Vc + I*ny + J``;
* ``kuhn6``   -- 3D: every hex cell split into 6 tetrahedra around its
  v000-v111 diagonal; vertex (i, j, k) is ``(i*(ny+1) + j)*(nz+1) + k``.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from itertools import permutations

from typing import Optional

import numpy as np

PATTERNS = ("union_jack", "right", "crossed", "kuhn6")


@dataclass
class SimplexMesh:
    vertices: np.ndarray          # (V, d)
    elements: np.ndarray          # (T, d+1), positively oriented
    pattern: str
    shape: tuple                  # (nx, ny) or (nx, ny, nz)
    extent: tuple                 # (lx, ly[, lz])
    origin: tuple
    boundary: dict = field(default_factory=dict)   # tag -> sorted vertex ids

    @property
    def dim(self) -> int:
        return self.vertices.shape[1]

    @property
    def n_vertices(self) -> int:
        return self.vertices.shape[0]

    @property
    def n_elements(self) -> int:
        return self.elements.shape[0]

    @property
    def n_cells(self) -> int:
        return int(np.prod(self.shape))

    def element_cell(self) -> np.ndarray:
        """Grid-cell index (I-major) of every element."""
        per = self.n_elements // self.n_cells
        return np.tile(np.arange(self.n_cells), per)


def grid_mesh(nx: int, ny: int, lx: float = 1.0, ly: float = 1.0,
              pattern: str = "union_jack", ox: float = 0.0, oy: float = 0.0,
              ys: Optional[np.ndarray] = None) -> SimplexMesh:
    """2D structured triangulation of [ox, ox+lx] x [oy, oy+ly]; ``ys`` (ny+1 increasing row
    coordinates) gives graded rows (banded_rect_mesh, mesh.py:163-190)."""
    if nx < 1 or ny < 1:
        raise ValueError("grid_mesh needs nx, ny >= 1")
    xs = np.linspace(ox, ox + lx, nx + 1)
    if ys is None:
        ys = np.linspace(oy, oy + ly, ny + 1)
    else:
        ys = np.asarray(ys, dtype=float)
        if ys.shape != (ny + 1,) or np.any(np.diff(ys) <= 0):
            raise ValueError("ys must hold ny+1 increasing row coordinates")
        oy, ly = float(ys[0]), float(ys[-1] - ys[0])
    X, Y = np.meshgrid(xs, ys, indexing="ij")
    corners = np.column_stack([X.ravel(), Y.ravel()])
    nv = ny + 1
    I, J = np.meshgrid(np.arange(nx), np.arange(ny), indexing="ij")
    I = I.ravel()
    J = J.ravel()
    a = I * nv + J          # v00
    b = (I + 1) * nv + J    # v10
    c = (I + 1) * nv + J + 1  # v11
    d = I * nv + J + 1      # v01
    if pattern == "union_jack":
        ev = ((I + J) % 2 == 0)[:, None]
        first = np.where(ev, np.column_stack([a, b, c]), np.column_stack([a, b, d]))
        second = np.where(ev, np.column_stack([a, c, d]), np.column_stack([b, c, d]))
        elements = np.vstack([first, second])
        vertices = corners
    elif pattern == "right":
        elements = np.vstack([np.column_stack([a, b, c]), np.column_stack([a, c, d])])
        vertices = corners
    elif pattern == "crossed":
        ctr = corners.shape[0] + I * ny + J
        centres = np.column_stack([0.5 * (xs[I] + xs[I + 1]), 0.5 * (ys[J] + ys[J + 1])])
        vertices = np.vstack([corners, centres])
        elements = np.vstack([np.column_stack([a, b, ctr]), np.column_stack([b, c, ctr]),
                              np.column_stack([c, d, ctr]), np.column_stack([d, a, ctr])])
    else:
        raise ValueError(f"unknown 2D pattern {pattern!r}")
    jj = np.arange(ny + 1)
    ii = np.arange(nx + 1)
    boundary = {"left": jj.copy(), "right": nx * nv + jj,
                "bottom": ii * nv, "top": ii * nv + ny}
    return SimplexMesh(vertices, elements.astype(np.intp), pattern, (nx, ny), (lx, ly),
                       (ox, oy), boundary)


def graded_heights(span: float, h_fine: float, h_coarse: float, ratio: float = 1.3) -> np.ndarray:
    """Row heights tiling ``span``: geometric growth from h_fine by ``ratio``, capped at h_coarse,
    then shrunk uniformly to tile the span exactly (mesh.py:145-160; same operation order)."""
    if span <= 1e-12:
        return np.zeros(0)
    rows = []
    h = h_fine
    while sum(rows) < span:  # Python's sequential sum, as the reference
        h = min(h * ratio, h_coarse)
        rows.append(h)
    rows = np.asarray(rows)
    return rows * (span / rows.sum())


def banded_rows(L: float, H: float, h_fine: float, h_coarse: float, band_halfwidth: float):
    """(nx, ys) of the band-refined grid on [0, L] x [-H/2, H/2] (banded_rect_mesh,
    mesh.py:163-190): rows of h_fine within the band (+ one guard row), graded outside."""
    nb = int(np.ceil(band_halfwidth / h_fine)) + 1
    nx = max(1, round(L / h_fine))
    if nb * h_fine >= H / 2:
        ny = max(1, round(H / h_fine))
        return nx, np.linspace(-H / 2, -H / 2 + H, ny + 1)
    y_band = nb * h_fine
    upper = graded_heights(H / 2 - y_band, h_fine, h_coarse)
    y_up = y_band + np.cumsum(upper)
    ys = np.concatenate([-y_up[::-1], np.arange(-nb, nb + 1) * h_fine, y_up])
    ys[0] = -H / 2
    ys[-1] = H / 2
    return nx, ys


def kuhn_mesh(nx: int, ny: int, nz: int, lx: float = 1.0, ly: float = 1.0,
              lz: float = 1.0) -> SimplexMesh:
    """3D structured mesh of hexes split into 6 Kuhn tetrahedra."""
    xs = np.linspace(0.0, lx, nx + 1)
    ys = np.linspace(0.0, ly, ny + 1)
    zs = np.linspace(0.0, lz, nz + 1)
    X, Y, Z = np.meshgrid(xs, ys, zs, indexing="ij")
    vertices = np.column_stack([X.ravel(), Y.ravel(), Z.ravel()])

    def vid(i, j, k):
        return (i * (ny + 1) + j) * (nz + 1) + k

    I, J, K = np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij")
    I, J, K = I.ravel(), J.ravel(), K.ravel()
    blocks = []
    for perm in kuhn_paths():
        path = [(0, 0, 0)]
        cur = [0, 0, 0]
        for ax in perm:
            cur[ax] = 1
            path.append(tuple(cur))
        tet = np.column_stack([vid(I + p[0], J + p[1], K + p[2]) for p in path])
        blocks.append(tet)
    elements = np.vstack(blocks).astype(np.intp)
    # orient positively
    p = vertices[elements]
    vol = np.einsum("ti,ti->t", np.cross(p[:, 1] - p[:, 0], p[:, 2] - p[:, 0]), p[:, 3] - p[:, 0])
    neg = vol < 0
    elements[neg] = elements[neg][:, [0, 2, 1, 3]]
    i = np.arange(nx + 1)
    j = np.arange(ny + 1)
    k = np.arange(nz + 1)
    A, B = np.meshgrid(j, k, indexing="ij")
    C, Dd = np.meshgrid(i, k, indexing="ij")
    E_, F_ = np.meshgrid(i, j, indexing="ij")
    boundary = {
        "x0": np.sort(vid(0, A, B).ravel()), "x1": np.sort(vid(nx, A, B).ravel()),
        "y0": np.sort(vid(C, 0, Dd).ravel()), "y1": np.sort(vid(C, ny, Dd).ravel()),
        "z0": np.sort(vid(E_, F_, 0).ravel()), "z1": np.sort(vid(E_, F_, nz).ravel()),
    }
    return SimplexMesh(vertices, elements, "kuhn6", (nx, ny, nz), (lx, ly, lz),
                       (0.0, 0.0, 0.0), boundary)


def kuhn_paths():
    """The 6 axis orders (x=0, y=1, z=2) defining the Kuhn tetrahedra, in storage order."""
    return list(permutations((0, 1, 2)))


def jitter_interior(mesh: SimplexMesh, jitter: float, seed: int = 0) -> SimplexMesh:
    """Move every interior vertex by a seeded uniform offset of up to ``jitter`` cell sizes per
    axis (the reference's rect_mesh jitter, mesh.py:127-141: ``default_rng(seed).uniform(-j, j,
    (n_interior, d)) * h`` on the strictly interior vertices in index order).  Connectivity is
    unchanged; a non-positive element raises as the reference's _validate_orientation
    (mesh.py:66-75).  Applies in 3D too (the reference's jitter is 2D only)."""
    if not 0.0 <= jitter <= 0.4:
        raise ValueError(f"jitter must lie in [0, 0.4]; got {jitter}")
    v = mesh.vertices.copy()
    lo = np.asarray(mesh.origin, float)
    hi = lo + np.asarray(mesh.extent, float)
    h = np.asarray(mesh.extent, float) / np.asarray(mesh.shape, float)
    interior = np.all((v > lo) & (v < hi), axis=1)
    if jitter > 0.0:
        rng = np.random.default_rng(seed)
        v[interior] += rng.uniform(-jitter, jitter, size=(int(interior.sum()), v.shape[1])) * h
    out = SimplexMesh(v, mesh.elements.copy(), mesh.pattern, mesh.shape, mesh.extent, mesh.origin,
                      dict(mesh.boundary))
    P = v[out.elements]
    if out.dim == 2:
        det = ((P[:, 1, 0] - P[:, 0, 0]) * (P[:, 2, 1] - P[:, 0, 1])
               - (P[:, 1, 1] - P[:, 0, 1]) * (P[:, 2, 0] - P[:, 0, 0]))
    else:
        det = np.einsum("ti,ti->t", np.cross(P[:, 1] - P[:, 0], P[:, 2] - P[:, 0]), P[:, 3] - P[:, 0])
    if np.any(det <= 0):
        raise ValueError(f"mesh has {int(np.sum(det <= 0))} non-CCW/degenerate elements")
    return out
