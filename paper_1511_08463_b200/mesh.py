"""Structured mesh descriptors (reference mesh.py).

The device never sees an element list: geometry is implicit in (pattern, nx, ny,
extents).  This module keeps the reference's layout contract (mesh.py:3-10):
vertex (i, j) = i*(ny+1) + j, displacement interleaved per vertex, triangles
type-major in I-major cell order; crossed centre vertices follow the corners.
Host-side coordinates and boundary sets are produced lazily for BC setup and
post-processing only.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

BOUNDARY_TAGS = ("left", "right", "bottom", "top")
PATTERNS_2D = ("union_jack", "right", "crossed")
_FIELDS = {"displacement_x1": (2, 0), "displacement_x2": (2, 1), "damage": (1, 0)}


@dataclass
class StructuredMesh:
    """Structured triangulation of [x0, x0+lx] x [y0, y0+ly] with nx x ny cells."""

    nx: int
    ny: int
    lx: float = 1.0
    ly: float = 1.0
    pattern: str = "union_jack"
    x0: float = 0.0
    y0: float = 0.0
    ys: np.ndarray | None = field(default=None, repr=False)  # graded rows: ny+1 coordinates
    _vertices: np.ndarray | None = field(default=None, repr=False)

    def __post_init__(self):
        if self.nx < 1 or self.ny < 1:
            raise ValueError("StructuredMesh needs nx, ny >= 1")
        if self.pattern not in PATTERNS_2D:
            raise ValueError(f"unknown pattern {self.pattern!r}; choose from {PATTERNS_2D}")
        if self.ys is not None:
            ys = np.asarray(self.ys, dtype=float)
            if ys.shape != (self.ny + 1,) or np.any(np.diff(ys) <= 0):
                raise ValueError("ys must hold ny+1 increasing row coordinates")
            self.ys = ys
            self.y0, self.ly = float(ys[0]), float(ys[-1] - ys[0])
        if self.lx <= 0 or self.ly <= 0:
            raise ValueError("extents must be positive")

    dim = 2

    @property
    def n_corner_vertices(self) -> int:
        return (self.nx + 1) * (self.ny + 1)

    @property
    def n_cells(self) -> int:
        return self.nx * self.ny

    @property
    def n_vertices(self) -> int:
        return self.n_corner_vertices + (self.n_cells if self.pattern == "crossed" else 0)

    @property
    def n_triangles(self) -> int:
        return self.n_cells * (4 if self.pattern == "crossed" else 2)

    @property
    def hx(self) -> float:
        return self.lx / self.nx

    @property
    def hy(self) -> float:
        return self.ly / self.ny

    @property
    def row_heights(self):
        """Cell-row heights of a graded mesh (None when rows are uniform)."""
        return None if self.ys is None else np.diff(self.ys)

    def _ys(self) -> np.ndarray:
        return self.ys if self.ys is not None else np.linspace(self.y0, self.y0 + self.ly, self.ny + 1)

    @property
    def vertices(self) -> np.ndarray:
        if self._vertices is None:
            xs = np.linspace(self.x0, self.x0 + self.lx, self.nx + 1)
            ys = self._ys()
            X, Y = np.meshgrid(xs, ys, indexing="ij")
            v = np.column_stack([X.ravel(), Y.ravel()])
            if self.pattern == "crossed":
                I, J = np.meshgrid(np.arange(self.nx), np.arange(self.ny), indexing="ij")
                cx = 0.5 * (xs[I.ravel()] + xs[I.ravel() + 1])
                cy = 0.5 * (ys[J.ravel()] + ys[J.ravel() + 1])
                v = np.vstack([v, np.column_stack([cx, cy])])
            self._vertices = v
        return self._vertices

    def vid(self, i, j):
        return np.asarray(i) * (self.ny + 1) + np.asarray(j)

    def boundary_vertices(self, tag: str) -> np.ndarray:
        jj = np.arange(self.ny + 1)
        ii = np.arange(self.nx + 1)
        if tag == "left":
            return self.vid(0, jj)
        if tag == "right":
            return self.vid(self.nx, jj)
        if tag == "bottom":
            return self.vid(ii, 0)
        if tag == "top":
            return self.vid(ii, self.ny)
        raise KeyError(f"unknown boundary tag {tag!r}; have {BOUNDARY_TAGS}")

    def all_boundary_vertices(self) -> np.ndarray:
        return np.unique(np.concatenate([self.boundary_vertices(t) for t in BOUNDARY_TAGS]))

    def cell_row_centroid_y(self) -> np.ndarray:
        """(n_types, ny) centroid heights of each element type per cell row (for eps0 tables)."""
        ys = self._ys()
        y0, y1 = ys[:-1], ys[1:]
        yc = 0.5 * (y0 + y1)
        if self.pattern == "union_jack":
            # even-parity types (0,1,3),(0,3,2); odd (0,1,2),(1,3,2); local y: 0,0,1,1
            t = [(y0 + y0 + y1), (y0 + y1 + y1), (y0 + y0 + y1), (y0 + y1 + y1)]
            return np.stack([v / 3.0 for v in t])
        if self.pattern == "right":
            t = [(y0 + y0 + y1), (y0 + y1 + y1)]
            return np.stack([v / 3.0 for v in t] + [v / 3.0 for v in t])
        t = [(y0 + y0 + yc), (y0 + y1 + yc), (y1 + y1 + yc), (y1 + y0 + yc)]
        return np.stack([v / 3.0 for v in t])


@dataclass
class StructuredMesh3D:
    """Structured hex grid of [0,lx]x[0,ly]x[0,lz], each hex split into 6 Kuhn tetrahedra.

    Vertex (i, j, k) = (i*(ny+1) + j)*(nz+1) + k; u interleaved (3 comps per vertex);
    tetrahedra type-major (the 6 axis permutations in itertools order) over I-major cells.
    """

    nx: int
    ny: int
    nz: int
    lx: float = 1.0
    ly: float = 1.0
    lz: float = 1.0
    pattern: str = "kuhn6"
    _vertices: np.ndarray | None = field(default=None, repr=False)

    dim = 3

    def __post_init__(self):
        if min(self.nx, self.ny, self.nz) < 1:
            raise ValueError("StructuredMesh3D needs nx, ny, nz >= 1")
        if self.pattern != "kuhn6":
            raise ValueError("3D pattern must be 'kuhn6'")

    @property
    def n_vertices(self) -> int:
        return (self.nx + 1) * (self.ny + 1) * (self.nz + 1)

    @property
    def n_cells(self) -> int:
        return self.nx * self.ny * self.nz

    @property
    def n_tets(self) -> int:
        return 6 * self.n_cells

    @property
    def vertices(self) -> np.ndarray:
        if self._vertices is None:
            xs = np.linspace(0.0, self.lx, self.nx + 1)
            ys = np.linspace(0.0, self.ly, self.ny + 1)
            zs = np.linspace(0.0, self.lz, self.nz + 1)
            X, Y, Z = np.meshgrid(xs, ys, zs, indexing="ij")
            self._vertices = np.column_stack([X.ravel(), Y.ravel(), Z.ravel()])
        return self._vertices

    def vid(self, i, j, k):
        return (np.asarray(i) * (self.ny + 1) + np.asarray(j)) * (self.nz + 1) + np.asarray(k)

    def face_vertices(self, tag: str) -> np.ndarray:
        """Sorted vertex ids of a face: x0, x1, y0, y1, z0, z1."""
        r = {"x": np.arange(self.nx + 1), "y": np.arange(self.ny + 1), "z": np.arange(self.nz + 1)}
        ax, side = tag[0], tag[1]
        n = {"x": self.nx, "y": self.ny, "z": self.nz}[ax]
        r[ax] = np.array([0 if side == "0" else n])
        I, J, K = np.meshgrid(r["x"], r["y"], r["z"], indexing="ij")
        return np.sort(self.vid(I, J, K).ravel())


def rect_mesh(L: float, H: float, h: float, origin_x2: float = 0.0,
              pattern: str = "union_jack") -> StructuredMesh:
    """Uniform mesh of [0, L] x [origin_x2, origin_x2 + H] with target size h (mesh.py:112-142;
    jitter is not supported on the structured device path)."""
    if L <= 0 or H <= 0 or h <= 0:
        raise ValueError(f"rect_mesh needs positive L, H, h; got L={L}, H={H}, h={h}")
    nx = max(1, round(L / h))
    ny = max(1, round(H / h))
    return StructuredMesh(nx, ny, L, H, pattern, 0.0, origin_x2)


def _graded_heights(span: float, h_fine: float, h_coarse: float, ratio: float = 1.3) -> np.ndarray:
    """Heights tiling ``span``, growing by ``ratio`` from h_fine and capped at h_coarse, then
    uniformly shrunk to tile it exactly (mesh.py:145-160)."""
    if span <= 1e-12:
        return np.zeros(0)
    hs = []
    h = h_fine
    while sum(hs) < span:
        h = min(h * ratio, h_coarse)
        hs.append(h)
    hs = np.asarray(hs)
    return hs * (span / hs.sum())


def banded_rect_mesh(L: float, H: float, h_fine: float, h_coarse: float,
                     band_halfwidth: float) -> StructuredMesh:
    """Union-jack mesh of [0, L] x [-H/2, H/2] refined in a band around y = 0 (mesh.py:163-190):
    uniform columns of ~h_fine, rows of h_fine within |y| <= band_halfwidth (+ one guard row),
    graded (ratio <= 1.3, capped at h_coarse) towards the edges.  Uniform when the band fills H."""
    if L <= 0 or H <= 0 or h_fine <= 0 or band_halfwidth < 0:
        raise ValueError("banded_rect_mesh needs positive L, H, h_fine and band_halfwidth >= 0")
    if h_coarse < h_fine:
        raise ValueError(f"h_coarse ({h_coarse}) must be >= h_fine ({h_fine})")
    nb = int(np.ceil(band_halfwidth / h_fine)) + 1
    if nb * h_fine >= H / 2:
        return rect_mesh(L, H, h_fine, origin_x2=-H / 2)
    y_band = nb * h_fine
    upper = _graded_heights(H / 2 - y_band, h_fine, h_coarse)
    y_up = y_band + np.cumsum(upper)
    ys = np.concatenate([-y_up[::-1], np.arange(-nb, nb + 1) * h_fine, y_up])
    ys[0] = -H / 2
    ys[-1] = H / 2
    nx = max(1, round(L / h_fine))
    return StructuredMesh(nx, len(ys) - 1, L, H, "union_jack", 0.0, -H / 2, ys=ys)


def boundary_dofs(mesh: StructuredMesh, tag: str, fieldname: str) -> np.ndarray:
    """Sorted global dof indices of ``fieldname`` on the tagged boundary (mesh.py:193-205)."""
    if fieldname not in _FIELDS:
        raise KeyError(f"unknown field {fieldname!r}; have {sorted(_FIELDS)}")
    stride, offset = _FIELDS[fieldname]
    return (stride * np.sort(mesh.boundary_vertices(tag)) + offset).astype(np.intp)
