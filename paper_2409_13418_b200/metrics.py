"""Mesh quality metrics on top of the GPU distance queries
(occmesh.metrics, /root/reference/pkg/src/occmesh/metrics.py:1-70, and
occmesh.mesh.MeshDistanceIndex / sample_surface, mesh.py:202-297).

Surface sampling stays in numpy so the samples are the reference's for the
same seed (same generator calls in the same order); the exact closest-point
queries -- the O(samples x triangles) part -- run in libodc
(``odc_mesh_distance``, csrc/odc_distance.cu).
"""

from __future__ import annotations


import numpy as np

from . import _lib


def triangle_areas(mesh, device=0):
    """TriangleMesh.areas() computed on the GPU (same values as numpy)."""
    v = np.ascontiguousarray(mesh.vertices, dtype=np.float64).reshape(-1, 3)
    t = np.ascontiguousarray(mesh.triangles, dtype=np.int64).reshape(-1, 3)
    out = np.empty(len(t))
    if len(t):
        ctx = _lib.context(device)
        L = _lib.load()
        rc = L.odc_triangle_areas(ctx.handle, v.ctypes.data, len(v), t.ctypes.data, len(t), out.ctypes.data)
        if rc != _lib.ODC_OK:
            raise ValueError(L.odc_last_error(ctx.handle).decode())
    return out


def sample_surface(mesh, n, seed=0, rng=None):
    """Area-weighted uniform surface samples with their face normals and
    triangle indices; the reference's generator sequence (mesh.py:273-297)."""
    if mesh.n_triangles == 0:
        raise ValueError("cannot sample an empty mesh")
    if n < 1:
        raise ValueError("sample count must be at least 1")
    rng = rng or np.random.default_rng(seed)
    areas = triangle_areas(mesh)
    total = areas.sum()
    if total <= 0:
        raise ValueError("mesh has zero total area")
    cdf = np.cumsum(areas) / total
    idx = np.minimum(np.searchsorted(cdf, rng.random(n), side="right"), mesh.n_triangles - 1)
    u = rng.random(n)
    v = rng.random(n)
    over = u + v > 1.0
    u[over] = 1.0 - u[over]
    v[over] = 1.0 - v[over]
    # only the sampled triangles' corners and normals (row-wise identical to
    # indexing the full arrays, without materialising them)
    c = mesh.vertices[mesh.triangles[idx]]
    pts = c[:, 0] + u[:, None] * (c[:, 1] - c[:, 0]) + v[:, None] * (c[:, 2] - c[:, 0])
    return pts, _normals(c), idx


def _normals(c):
    n = np.cross(c[:, 1] - c[:, 0], c[:, 2] - c[:, 0])
    lens = np.linalg.norm(n, axis=1, keepdims=True)
    return np.divide(n, lens, out=np.zeros_like(n), where=lens > 0)


class MeshDistanceIndex:
    """Exact point-to-mesh distances on the GPU (mesh.py:202-270 contract:
    ``query(points) -> (distance, closest triangle, closest point)``)."""

    def __init__(self, mesh, device=0):
        if mesh.n_triangles == 0:
            raise ValueError("distance index needs a non-empty mesh")
        self.mesh = mesh
        self.device = device
        self._v = np.ascontiguousarray(mesh.vertices, dtype=np.float64).reshape(-1, 3)
        self._t = np.ascontiguousarray(mesh.triangles, dtype=np.int64).reshape(-1, 3)

    def query(self, points, chunk=None):
        pts = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 3)
        n = len(pts)
        dist = np.empty(n)
        tri = np.empty(n, dtype=np.int64)
        cp = np.empty((n, 3))
        if n == 0:
            return dist, tri, cp
        ctx = _lib.context(self.device)
        L = _lib.load()
        rc = L.odc_mesh_distance(ctx.handle, self._v.ctypes.data, len(self._v), self._t.ctypes.data, len(self._t),
                                 pts.ctypes.data, n, dist.ctypes.data, tri.ctypes.data, cp.ctypes.data)
        if rc != _lib.ODC_OK:
            msg = L.odc_last_error(ctx.handle).decode()
            raise (ValueError(msg) if rc == _lib.ODC_E_VALUE else RuntimeError(msg))
        return dist, tri, cp


def metric_fit(mesh, field, n=100_000, seed=0, device=0):
    """Mean |raw - iso| over surface samples, the field evaluated on the GPU;
    None for binary-only fields (metrics.py:18-23)."""
    if not field.continuous:
        return None
    from .pipeline import eval_raw

    pts, _, _ = sample_surface(mesh, n, seed=seed)
    raw = np.asarray(eval_raw(field, pts, device=device), dtype=np.float64)
    return float(np.mean(np.abs(raw - field.iso_level)))


def metric_md2(mesh_a, mesh_b, n=100_000, seed=0, device=0):
    """Mean squared point-to-mesh distance, both directions (metrics.py:26-32)."""
    pa, _, _ = sample_surface(mesh_a, n, seed=seed)
    pb, _, _ = sample_surface(mesh_b, n, seed=seed + 1)
    d_ab, _, _ = MeshDistanceIndex(mesh_b, device).query(pa)
    d_ba, _, _ = MeshDistanceIndex(mesh_a, device).query(pb)
    return 0.5 * (float(np.mean(d_ab**2)) + float(np.mean(d_ba**2)))


def metric_nic(mesh_gt, mesh_out, n=100_000, seed=0, return_directions=False, device=0):
    """Mean angle between sample normals and the nearest triangle's normal on
    the other mesh, both directions (metrics.py:35-57)."""
    pg, ng, _ = sample_surface(mesh_gt, n, seed=seed)
    po, no, _ = sample_surface(mesh_out, n, seed=seed + 1)
    _, t_go, _ = MeshDistanceIndex(mesh_out, device).query(pg)
    _, t_og, _ = MeshDistanceIndex(mesh_gt, device).query(po)
    n_out = _normals(mesh_out.vertices[mesh_out.triangles[t_go]])
    n_gt = _normals(mesh_gt.vertices[mesh_gt.triangles[t_og]])
    fwd = float(np.mean(np.arccos(np.clip(np.einsum("ij,ij->i", ng, n_out), -1.0, 1.0))))
    bwd = float(np.mean(np.arccos(np.clip(np.einsum("ij,ij->i", no, n_gt), -1.0, 1.0))))
    mean = 0.5 * (fwd + bwd)
    if return_directions:
        return mean, {"gt_to_out": fwd, "out_to_gt": bwd}
    return mean


def metric_hdd(mesh_a, mesh_b, n=100_000, seed=0, device=0):
    """Sampled Hausdorff distance (metrics.py:60-66)."""
    pa, _, _ = sample_surface(mesh_a, n, seed=seed)
    pb, _, _ = sample_surface(mesh_b, n, seed=seed + 1)
    d_ab, _, _ = MeshDistanceIndex(mesh_b, device).query(pa)
    d_ba, _, _ = MeshDistanceIndex(mesh_a, device).query(pb)
    return max(float(d_ab.max()), float(d_ba.max()))
