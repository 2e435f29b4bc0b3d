"""Output mesh type and grid spec, mirroring the reference's data model.

``TriangleMesh`` follows /root/reference/pkg/src/occmesh/mesh.py:11-76 (the
extraction path's output type: vertices (V,3) f64, triangles (T,3) i64,
provenance kind/ref) and ``GridSpec`` follows grid.py:17-91 (index
conventions: vertex id x + y*S + z*S^2, h = (hi - lo) / R).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class GridSpec:
    """Axis-aligned box divided into resolution^3 cells (grid.py:17-31)."""

    lo: tuple
    hi: tuple
    resolution: int

    def __post_init__(self):
        object.__setattr__(self, "lo", tuple(float(v) for v in self.lo))
        object.__setattr__(self, "hi", tuple(float(v) for v in self.hi))
        if self.resolution < 2:
            raise ValueError("resolution must be at least 2")
        if any(h <= l for l, h in zip(self.lo, self.hi)):
            raise ValueError("grid box must have positive extent")

    @property
    def shape(self):
        return self.resolution + 1

    @property
    def cell_size(self):
        return (np.array(self.hi) - np.array(self.lo)) / self.resolution

    @property
    def n_vertices(self):
        return self.shape**3

    @property
    def n_cells(self):
        return self.resolution**3


@dataclass
class TriangleMesh:
    """Indexed triangle mesh with per-vertex provenance (mesh.py:11-36).

    Provenance kind: 0 = cell partition point, 1 = edge point, 2 = repair
    duplicate; ref carries (cell id, partition index) or (edge key, -1).
    """

    vertices: np.ndarray
    triangles: np.ndarray
    provenance_kind: np.ndarray | None = None
    provenance_ref: np.ndarray | None = None

    def __post_init__(self):
        self.vertices = np.asarray(self.vertices, dtype=np.float64).reshape(-1, 3)
        self.triangles = np.asarray(self.triangles, dtype=np.int64).reshape(-1, 3)
        if len(self.triangles):
            if self.triangles.min() < 0 or self.triangles.max() >= len(self.vertices):
                raise ValueError("triangle index out of range")
            t = self.triangles
            if ((t[:, 0] == t[:, 1]) | (t[:, 1] == t[:, 2]) | (t[:, 2] == t[:, 0])).any():
                raise ValueError("triangle with repeated vertex index")

    @classmethod
    def trusted(cls, vertices, triangles, provenance_kind=None, provenance_ref=None):
        """Wrap arrays produced by libodc (already f64/i64, in range, no repeated
        index) without re-running the O(T) validation of __post_init__."""
        m = object.__new__(cls)
        m.vertices, m.triangles = vertices, triangles
        m.provenance_kind, m.provenance_ref = provenance_kind, provenance_ref
        return m

    @property
    def n_vertices(self):
        return len(self.vertices)

    def corners(self):
        """(T, 3, 3) triangle corner positions (mesh.py:46-47)."""
        return self.vertices[self.triangles]

    def face_normals(self, normalized=True):
        """Per-triangle cross((c1 - c0), (c2 - c0)), unit length unless
        degenerate (zero) when ``normalized`` (mesh.py:49-55)."""
        c = self.corners()
        n = np.cross(c[:, 1] - c[:, 0], c[:, 2] - c[:, 0])
        if normalized:
            lens = np.linalg.norm(n, axis=1, keepdims=True)
            n = np.divide(n, lens, out=np.zeros_like(n), where=lens > 0)
        return n

    def areas(self):
        """Triangle areas (mesh.py:57-61)."""
        c = self.corners()
        return 0.5 * np.linalg.norm(np.cross(c[:, 1] - c[:, 0], c[:, 2] - c[:, 0]), axis=1)

    @property
    def n_triangles(self):
        return len(self.triangles)

    def undirected_edges(self):
        e = np.concatenate([self.triangles[:, [0, 1]], self.triangles[:, [1, 2]], self.triangles[:, [2, 0]]])
        return np.sort(e, axis=1)

    def euler_characteristic(self):
        if len(self.triangles) == 0:
            return 0
        n_edges = len(np.unique(self.undirected_edges(), axis=0))
        return self.n_vertices - n_edges + self.n_triangles


@dataclass
class ManifoldReport:
    """validate_manifold's result (mesh.py:79-88 of the reference)."""

    manifold: bool
    nonmanifold_edges: list
    pinched_vertices: list
    boundary_edges: int
    isolated_vertices: list

    def __bool__(self):
        return self.manifold


def validate_manifold(mesh, device=0):
    """Edge incidence (at most two triangles per edge) and fan connectivity,
    computed on the GPU (libodc ``odc_validate_manifold``); same report as
    occmesh.mesh.validate_manifold (mesh.py:91-150): non-manifold edges as
    (a, b) with a < b in key order, pinched and isolated vertex ids ascending,
    the boundary-edge count."""
    from . import _lib

    ctx = _lib.context(device)
    L = _lib.load()
    t = np.ascontiguousarray(mesh.triangles, dtype=np.int64).reshape(-1, 3)
    rep = _lib.ManifoldReport()
    rc = L.odc_validate_manifold(ctx.handle, t.ctypes.data if len(t) else None, len(t), int(len(mesh.vertices)),
                                 ctypes.byref(rep))
    if rc != _lib.ODC_OK:
        msg = L.odc_last_error(ctx.handle).decode()
        raise (ValueError(msg) if rc == _lib.ODC_E_VALUE else RuntimeError(msg))
    e = np.empty((rep.n_nonmanifold_edges, 2), dtype=np.int64)
    p = np.empty(rep.n_pinched_vertices, dtype=np.int64)
    iso = np.empty(rep.n_isolated_vertices, dtype=np.int64)
    ptr = lambda a: a.ctypes.data if a.size else None  # noqa: E731
    L.odc_validate_copy(ctx.handle, ptr(e), ptr(p), ptr(iso))
    return ManifoldReport(bool(rep.manifold), [(int(a), int(b)) for a, b in e.tolist()], p.tolist(),
                          int(rep.n_boundary_edges), iso.tolist())


def count_self_intersections(mesh, tolerance=1e-12, return_pairs=False, device=0):
    """Triangle pairs with positive-measure intersection, on the GPU (libodc
    ``odc_count_self_intersections``); same contract as
    occmesh.mesh.count_self_intersections (mesh.py:395-487): pairs sharing a
    vertex or involving a degenerate triangle are excluded; with
    ``return_pairs`` also the sorted list of (a, b) pairs."""
    from . import _lib

    ctx = _lib.context(device)
    L = _lib.load()
    v = np.ascontiguousarray(mesh.vertices, dtype=np.float64).reshape(-1, 3)
    t = np.ascontiguousarray(mesh.triangles, dtype=np.int64).reshape(-1, 3)
    n = ctypes.c_int64()
    rc = L.odc_count_self_intersections(ctx.handle, v.ctypes.data if len(v) else None, len(v),
                                        t.ctypes.data if len(t) else None, len(t), float(tolerance),
                                        ctypes.byref(n))
    if rc != _lib.ODC_OK:
        msg = L.odc_last_error(ctx.handle).decode()
        raise (ValueError(msg) if rc == _lib.ODC_E_VALUE else RuntimeError(msg))
    if not return_pairs:
        return int(n.value)
    pairs = np.empty((n.value, 2), dtype=np.int64)
    L.odc_self_intersection_pairs(ctx.handle, pairs.ctypes.data if n.value else None)
    return int(n.value), [(int(a), int(b)) for a, b in pairs.tolist()]
