"""Drop-in ``contour`` for occmesh.pipeline.contour on the B200.

Same signature, options, result type, stats keys, eval accounting and
exception types as /root/reference/pkg/src/occmesh/pipeline.py:154-240; the
whole extraction runs in libodc (hand-written sm_100a kernels) behind the
C-ABI in include/odc.h.  Fields are lowered to device programs
(fields.py); an unsupported field raises instead of falling back to a CPU.
"""

from __future__ import annotations

import ctypes
import os
import math
import time
from dataclasses import dataclass, field as dc_field

import numpy as np

from . import _lib
from .fields import (LoweringError, SurfaceCoincidenceError, field_continuous, is_mesh_winding, is_mlp, is_voxels,
                     lower_program)
from .mesh import GridSpec, TriangleMesh

ONE_D_MODES = ("midpoint", "linear-interp", "binary-search")
NORMAL_MODES = ("fd-gradient", "two-d-points")
SPLIT_MODES = ("mdc", "ic")

STATUS_EXACT, STATUS_MIDPOINT_FALLBACK, STATUS_CLAMPED, STATUS_RANGE_EXHAUSTED = 0, 1, 2, 3
STATUS_NAMES = {0: "exact", 1: "midpoint-fallback", 2: "clamped", 3: "range-exhausted"}


class ConfigurationError(ValueError):
    """Bad pipeline mode (pipeline.py:26-27)."""


class InternalContractError(RuntimeError):
    """An internal pipeline invariant was violated (dualize.py:23-24)."""


@dataclass(frozen=True)
class LineBudget:
    """search.py:29-36"""

    n_linear: int
    n_binary: int
    max_range_factor: float


@dataclass(frozen=True)
class SearchBudget:
    """search.py:39-58: 15 evaluations per edge, (4+11) + 2*(3+12) per 2D point."""

    iters_1d: int = 15
    step1: LineBudget = dc_field(default_factory=lambda: LineBudget(4, 11, 0.8))
    step2: LineBudget = dc_field(default_factory=lambda: LineBudget(3, 12, math.sqrt(2.0) / 2.0))

    @property
    def evals_per_2d_point(self):
        return self.step1.n_linear + self.step1.n_binary + 2 * (self.step2.n_linear + self.step2.n_binary)


@dataclass
class ContourOptions:
    """pipeline.py:60-78; the defaults are the full method."""

    one_d: str = "binary-search"
    normals: str = "two-d-points"
    split: str = "ic"
    budget: SearchBudget = dc_field(default_factory=SearchBudget)
    qef_truncation: float = 0.1
    fd_step_factor: float = 0.01
    repair: bool = True

    def validate(self):
        if self.one_d not in ONE_D_MODES:
            raise ConfigurationError(f"unknown 1D mode {self.one_d!r}")
        if self.normals not in NORMAL_MODES:
            raise ConfigurationError(f"unknown normal mode {self.normals!r}")
        if self.split not in SPLIT_MODES:
            raise ConfigurationError(f"unknown split mode {self.split!r}")


class EvalCounter:
    """Logical batched-evaluation accounting per category (pipeline.py:30-57).

    The device fuses analytic searches per element; the counts recorded here
    are the reference's lock-step batch counts, reported by libodc."""

    def __init__(self, field):
        self.field = field
        self.stats = {}

    def record(self, category, batches, evals):
        entry = self.stats.setdefault(category, {"batches": 0, "evals": 0})
        entry["batches"] += batches
        entry["evals"] += evals

    @property
    def total_evals(self):
        return sum(e["evals"] for e in self.stats.values())

    def snapshot(self):
        out = {k: dict(v) for k, v in self.stats.items()}
        out["total_evals"] = self.total_evals
        return out


@dataclass
class ContourResult:
    mesh: TriangleMesh
    raw_mesh: TriangleMesh
    counter: EvalCounter
    stats: dict


_ERRORS = {
    _lib.ODC_E_ASSERT: AssertionError,
    _lib.ODC_E_CONTRACT: InternalContractError,
    _lib.ODC_E_CONFIG: ConfigurationError,
    _lib.ODC_E_VALUE: ValueError,
    _lib.ODC_E_ARG: ValueError,
}


def _raise(rc, ctx, dfield=None):
    if dfield is not None and dfield.error is not None:  # the field's own exception (callback fields)
        err, dfield.error = dfield.error, None
        raise err
    msg = _lib.load().odc_last_error(ctx.handle).decode()
    if rc == _lib.ODC_E_VALUE and "off the surface" in msg:
        raise SurfaceCoincidenceError(msg)
    raise _ERRORS.get(rc, RuntimeError)(msg)


_DEVICE_KINDS = {"SphereField", "BoxField", "TorusField", "PlaneField", "CsgField", "SmoothedOccupancy",
                 "MlpField", "VoxelField", "MeshWindingField"}


class _CudaView:
    """Zero-copy view of a device buffer (__cuda_array_interface__)."""

    def __init__(self, ptr, shape, typestr):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (int(ptr), False),
                                         "version": 3, "strides": None}


def _make_callback(dfield, field):
    """The evaluation callback of a field the device cannot run itself (the
    reference's duck type: an object with ``eval_raw``, fields.py:51-61).
    The pipeline still runs on the device; for every batch of query points
    it would pass to eval_raw it calls the field: ``eval_raw_torch(points)``
    (a CUDA tensor in, a tensor out: the points never leave the device) when
    the field has one, else ``eval_raw`` on a host copy of the points, as
    the reference does.  label = raw > iso_level (fields.py:35-48).  An
    exception inside the field is kept and re-raised by the caller."""
    import torch

    iso = float(getattr(field, "iso_level", 0.5))
    torch_fn = getattr(field, "eval_raw_torch", None)
    dev = torch.device("cuda", dfield.ctx.device)

    def cb(user, pts_ptr, n, lab_ptr, raw_ptr, stream):
        try:
            with torch.cuda.device(dev):
                pts = torch.as_tensor(_CudaView(pts_ptr, (n, 3), "<f8"), device=dev)
                if torch_fn is not None:
                    raw = torch.as_tensor(torch_fn(pts), device=dev).to(torch.float64).reshape(-1)
                else:
                    host = np.asarray(field.eval_raw(pts.cpu().numpy()), dtype=np.float64).reshape(-1)
                    raw = torch.from_numpy(host).to(dev)
                if raw.shape[0] != n:
                    raise ValueError(f"eval_raw returned {raw.shape[0]} values for {n} points")
                torch.as_tensor(_CudaView(lab_ptr, (n,), "|u1"), device=dev).copy_((raw > iso).to(torch.uint8))
                if raw_ptr:
                    torch.as_tensor(_CudaView(raw_ptr, (n,), "<f8"), device=dev).copy_(raw)
                torch.cuda.synchronize(dev)
            return 0
        except BaseException as e:  # noqa: BLE001 -- re-raised by _raise via dfield.error
            dfield.error = e
            return 1

    return cb


class DeviceField:
    """A field uploaded to one libodc context (program, MLP weights, mesh,
    voxels) or, for any other occupancy function, a callback field."""

    def __init__(self, ctx, field):
        L = _lib.load()
        self.ctx = ctx
        self.handle = ctypes.c_void_p()
        self.error = None
        self.continuous = field_continuous(field)
        self.analytic = False  # a lowered field program (interval-boundable)
        if is_mlp(field):
            keep = [
                np.ascontiguousarray(field.weights[0], dtype=np.float32),
                np.ascontiguousarray(np.stack(field.weights[1:]), dtype=np.float32),
                np.ascontiguousarray(np.stack(field.biases), dtype=np.float32),
                np.ascontiguousarray(field.w_head, dtype=np.float32),
            ]
            d = _lib.MlpDesc()
            d.d_in, d.width, d.depth, d.n_freq = field.d_in, field.width, field.depth, field.n_freq
            d.w0, d.w_hidden, d.biases, d.w_head = [a.ctypes.data for a in keep]
            d.b_head, d.amplitude = float(field.b_head), float(field.amplitude)
            d.prior_scale, d.prior_radius = float(field.prior_scale), float(field.prior_radius)
            for i in range(3):
                d.prior_center[i] = float(field.prior_center[i])
            rc = L.odc_field_mlp(ctx.handle, ctypes.byref(d), ctypes.byref(self.handle))
        elif is_voxels(field):
            vals = np.ascontiguousarray(field.values, dtype=np.float64)
            o = (ctypes.c_double * 3)(*[float(x) for x in field.origin])
            sp = (ctypes.c_double * 3)(*[float(x) for x in field.spacing])
            nx, ny, nz = vals.shape
            rc = L.odc_field_voxels(ctx.handle, o, sp, vals.ctypes.data, nx, ny, nz, ctypes.byref(self.handle))
        elif is_mesh_winding(field):
            v = np.ascontiguousarray(field.vertices, dtype=np.float64).reshape(-1, 3)
            t = np.ascontiguousarray(field.triangles, dtype=np.int64).reshape(-1, 3)
            rc = L.odc_field_mesh(ctx.handle, v.ctypes.data if len(v) else None, len(v),
                                  t.ctypes.data if len(t) else None, len(t), ctypes.byref(self.handle))
        else:
            try:
                prog = lower_program(field)
            except LoweringError:
                # the reference's own field types always lower (a failure there is
                # a bug to surface, never a silent switch to host evaluation)
                if type(field).__name__ in _DEVICE_KINDS or not (hasattr(field, "eval_raw")
                                                                 or hasattr(field, "eval_raw_torch")):
                    raise
                prog = None
            if prog is None:  # any other occupancy function: a callback field
                self._fn = _lib.EVAL_FN(_make_callback(self, field))
                rc = L.odc_field_callback(ctx.handle, self._fn, None, int(self.continuous),
                                          float(getattr(field, "iso_level", 0.5)), ctypes.byref(self.handle))
            else:
                self.analytic = True
                nodes = np.ascontiguousarray(prog)
                rc = L.odc_field_analytic(ctx.handle, nodes.ctypes.data_as(ctypes.POINTER(_lib.Node)), len(nodes),
                                          int(self.continuous), float(getattr(field, "iso_level", 0.5)),
                                          ctypes.byref(self.handle))
        if rc != _lib.ODC_OK:
            _raise(rc, ctx)

    def free(self):
        if self.handle:
            _lib.load().odc_field_free(self.ctx.handle, self.handle)
            self.handle = ctypes.c_void_p()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.free()


def make_options(options, keep_intermediates=False):
    o = _lib.Options()
    _lib.load().odc_default_options(ctypes.byref(o))
    o.one_d = {"midpoint": 0, "linear-interp": 1, "binary-search": 2}[options.one_d]
    o.normals = {"fd-gradient": 0, "two-d-points": 1}[options.normals]
    o.split = {"mdc": 0, "ic": 1}[options.split]
    o.repair = int(bool(options.repair))
    b = options.budget
    o.iters_1d = b.iters_1d
    o.s1_lin, o.s1_bin, o.s1_range = b.step1.n_linear, b.step1.n_binary, b.step1.max_range_factor
    o.s2_lin, o.s2_bin, o.s2_range = b.step2.n_linear, b.step2.n_binary, b.step2.max_range_factor
    o.qef_truncation = options.qef_truncation
    o.fd_step_factor = options.fd_step_factor
    o.keep_intermediates = int(bool(keep_intermediates))
    return o


_PINNED_OUTPUT = os.environ.get("ODC_PINNED_OUTPUT", "1") != "0"


def _host_arrays(specs):
    """Output arrays of a mesh copy-back, carved from one page-locked block of
    torch's caching host allocator: libodc DMAs straight into them (no
    staging copy), and a block freed with the caller's last array is reused
    by the next call, so no page of it faults again -- first writes into
    fresh numpy buffers run at ~9 GB/s per thread on the B200 hosts, against
    56 GB/s of pinned D2H.  Falls back to plain numpy arrays.  The arrays
    are views of the block, which lives as long as any of them."""
    sizes = [int(np.prod(sh)) * np.dtype(dt).itemsize for sh, dt in specs]
    offs = np.cumsum([0] + [(n + 63) // 64 * 64 for n in sizes])
    buf = None
    if _PINNED_OUTPUT and offs[-1] >= (1 << 20):
        try:
            import torch

            if torch.cuda.is_available():
                buf = torch.empty(int(offs[-1]), dtype=torch.uint8, pin_memory=True).numpy()
        except Exception:  # no torch / no pinned memory: pageable arrays
            buf = None
    if buf is None:
        return [np.empty(sh, dtype=dt) for sh, dt in specs]
    return [np.frombuffer(buf, dtype=dt, count=int(np.prod(sh)), offset=int(o)).reshape(sh)
            for (sh, dt), o in zip(specs, offs[:-1])]


def _copy_mesh(ctx, which, st, provenance=True):
    L = _lib.load()
    raw = which == 1
    V = st.raw_n_vertices if raw else st.n_vertices
    T = st.raw_n_triangles if raw else st.n_triangles
    if provenance:
        v, t, kind, ref = _host_arrays([((V, 3), np.float64), ((T, 3), np.int64), ((V,), np.int64),
                                        ((V, 2), np.int64)])
    else:
        v, t = _host_arrays([((V, 3), np.float64), ((T, 3), np.int64)])
        kind = ref = None
    ptr = lambda a: a.ctypes.data if a is not None and a.size else None  # noqa: E731
    rc = L.odc_copy_mesh(ctx.handle, which, ptr(v), ptr(t), ptr(kind), ptr(ref))
    if rc != _lib.ODC_OK:
        _raise(rc, ctx)
    return TriangleMesh.trusted(v, t, kind, ref)


def _copy_meshes(ctx, st, provenance=True):
    """(mesh, raw_mesh) in one pipelined device-to-host transfer.  Repair
    only appends duplicates of existing vertices and renames triangle corners
    to them (polygonize.py:348-373), so the raw mesh's vertices and
    provenance are views of the repaired mesh's first rows and only its
    triangles are copied."""
    if st.repair_added_vertices == 0:
        mesh = _copy_mesh(ctx, 0, st, provenance)
        return mesh, mesh
    V, T, V0, T0 = int(st.n_vertices), int(st.n_triangles), int(st.raw_n_vertices), int(st.raw_n_triangles)
    if provenance:
        v, t, rt, kind, ref = _host_arrays([((V, 3), np.float64), ((T, 3), np.int64), ((T0, 3), np.int64),
                                            ((V,), np.int64), ((V, 2), np.int64)])
    else:
        v, t, rt = _host_arrays([((V, 3), np.float64), ((T, 3), np.int64), ((T0, 3), np.int64)])
        kind = ref = None
    ptr = lambda a: a.ctypes.data if a is not None and a.size else None  # noqa: E731
    rc = _lib.load().odc_copy_mesh_pair(ctx.handle, ptr(v), ptr(t), ptr(kind), ptr(ref), ptr(rt))
    if rc != _lib.ODC_OK:
        _raise(rc, ctx)
    mesh = TriangleMesh.trusted(v, t, kind, ref)
    raw = TriangleMesh.trusted(v[:V0], rt, kind[:V0] if kind is not None else None,
                               ref[:V0] if ref is not None else None)
    return mesh, raw


def _raw_from_repaired(ctx, mesh, st):
    """The pre-repair mesh: repair only appends duplicates of existing
    vertices and renames triangle corners to them (polygonize.py:348-373), so
    its vertices and provenance are the first V0 rows of the repaired mesh
    (views, no copy) and its triangles are the device's pre-repair buffer."""
    V0, T = int(st.raw_n_vertices), int(st.raw_n_triangles)
    t = np.empty((T, 3), dtype=np.int64)
    rc = _lib.load().odc_copy_mesh(ctx.handle, 1, None, t.ctypes.data if T else None, None, None)
    if rc != _lib.ODC_OK:
        _raise(rc, ctx)
    kind = mesh.provenance_kind[:V0] if mesh.provenance_kind is not None else None
    ref = mesh.provenance_ref[:V0] if mesh.provenance_ref is not None else None
    return TriangleMesh.trusted(mesh.vertices[:V0], t, kind, ref)


def stats_dict(st, options, mesh_counts=True):
    """ContourResult.stats with the reference's keys (pipeline.py:160-239)."""
    stats = {"options": options, "warnings": []}
    bi = int(st.boundary_inside_vertices)
    stats["boundary_inside_vertices"] = bi
    if bi:
        stats["warnings"].append(
            f"{bi} boundary grid vertices are inside; the output will have an open boundary")
    stats["n_crossing_edges"] = int(st.n_crossing_edges)
    stats["n_crossing_cells"] = int(st.n_crossing_cells)
    if st.n_crossing_edges == 0:
        stats["n_2d_points"] = 0
        stats["open_boundary"] = False
        return stats
    stats["n_partitions"] = int(st.n_partitions)
    stats["n_2d_points"] = int(st.n_2d_points)
    if options.normals == "two-d-points":
        stats["point2d_status_counts"] = {
            STATUS_NAMES[c]: int(st.point2d_status_counts[c]) for c in range(4) if st.point2d_status_counts[c]}
    stats["normal_fallbacks"] = int(st.normal_fallbacks)
    stats["qef_rank_counts"] = {r: int(st.qef_rank_counts[r]) for r in range(4) if st.qef_rank_counts[r]}
    stats["qef_max_residual"] = float(st.qef_max_residual)
    stats["split_case_counts"] = {c: int(st.split_case_counts[c]) for c in range(1, 4) if st.split_case_counts[c]}
    stats["open_boundary"] = st.skipped_boundary_edges > 0
    stats["skipped_boundary_edges"] = int(st.skipped_boundary_edges)
    stats["repair_added_vertices"] = int(st.repair_added_vertices)
    return stats


def record_counts(counter, st):
    for c in list(st.cat_order):
        if c < 0:
            break
        counter.record(_lib.CATEGORIES[c], int(st.eval_batches[c]), int(st.eval_evals[c]))


def _grid_args(grid):
    lo = (ctypes.c_double * 3)(*[float(v) for v in grid.lo])
    hi = (ctypes.c_double * 3)(*[float(v) for v in grid.hi])
    return lo, hi, int(grid.resolution)


def contour(field, grid, options=None, counter=None, *, device=0, provenance=True, keep_intermediates=False,
            return_context=False, _ctx=None):
    """Run the dual contouring pipeline on the GPU and return the repaired mesh.

    Signature and result follow occmesh.pipeline.contour (pipeline.py:154);
    ``grid`` may be this package's or the reference's GridSpec."""
    options = options or ContourOptions()
    options.validate()
    counter = counter or EvalCounter(field)
    t0 = time.perf_counter()
    ctx = _ctx if _ctx is not None else _lib.context(device)  # _ctx: contour_batch's own contexts
    L = _lib.load()
    st = _lib.Stats()
    lo, hi, R = _grid_args(grid)
    if R < 2:
        raise ValueError("resolution must be at least 2")
    o = make_options(options, keep_intermediates)
    with DeviceField(ctx, field) as dfield:
        rc = L.odc_extract(ctx.handle, dfield.handle, lo, hi, R, ctypes.byref(o), ctypes.byref(st))
        if rc != _lib.ODC_OK:
            _raise(rc, ctx, dfield)
    stats = stats_dict(st, options)
    if st.n_crossing_edges == 0:
        empty = TriangleMesh(np.zeros((0, 3)), np.zeros((0, 3), dtype=np.int64))
        mesh = raw_mesh = empty
    else:
        mesh, raw_mesh = _copy_meshes(ctx, st, provenance)
    record_counts(counter, st)
    stats["wall_time_s"] = time.perf_counter() - t0
    stats["eval_counts"] = counter.snapshot()
    stats["device_ms"] = float(st.device_ms)
    result = ContourResult(mesh, raw_mesh, counter, stats)
    if return_context:
        return result, ctx, st
    return result


def stage_arrays(ctx, names):
    """Intermediate arrays of the last extraction (needs keep_intermediates)."""
    L = _lib.load()
    out = {}
    for name in names:
        which, dt = _lib.ARR[name]
        n = ctypes.c_int64()
        rc = L.odc_copy_array(ctx.handle, which, None, 0, ctypes.byref(n))
        if rc != _lib.ODC_OK:
            _raise(rc, ctx)
        a = np.empty(n.value, dtype=dt)
        if n.value:
            rc = L.odc_copy_array(ctx.handle, which, a.ctypes.data, a.nbytes, ctypes.byref(n))
            if rc != _lib.ODC_OK:
                _raise(rc, ctx)
        out[name] = a
    return out


def eval_raw(field, points, device=0):
    """Field raw values evaluated on the device (EvalCounter.raw semantics)."""
    pts = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 3)
    ctx = _lib.context(device)
    out = np.empty(len(pts))
    with DeviceField(ctx, field) as f:
        rc = _lib.load().odc_eval_raw(ctx.handle, f.handle, pts.ctypes.data, len(pts), out.ctypes.data)
        if rc != _lib.ODC_OK:
            _raise(rc, ctx, f)
    return out


def eval_labels(field, points, device=0):
    """Binary labels evaluated on the device (fields.py:35-48 semantics)."""
    pts = np.asarray(points, dtype=np.float64)
    squeeze = pts.ndim == 1
    pts = np.ascontiguousarray(pts.reshape(-1, 3))
    ctx = _lib.context(device)
    out = np.empty(len(pts), dtype=np.uint8)
    with DeviceField(ctx, field) as f:
        rc = _lib.load().odc_eval_labels(ctx.handle, f.handle, pts.ctypes.data, len(pts), out.ctypes.data)
        if rc != _lib.ODC_OK:
            _raise(rc, ctx, f)
    return out[0] if squeeze else out


class SharedField:
    """A field whose evaluation runs on the device, bound to one context and
    upload -- the shared-field hook for parity oracles."""

    def __init__(self, field, device=0):
        self.field = field
        self.ctx = _lib.Context(device)  # own workspace: never clobbers a contour() result
        self.dev = DeviceField(self.ctx, field)
        self.continuous = field_continuous(field)
        self.iso_level = 0.5

    def eval_raw(self, points):
        pts = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 3)
        out = np.empty(len(pts))
        rc = _lib.load().odc_eval_raw(self.ctx.handle, self.dev.handle, pts.ctypes.data, len(pts), out.ctypes.data)
        if rc != _lib.ODC_OK:
            _raise(rc, self.ctx, self.dev)
        return out

    def close(self):
        self.dev.free()
