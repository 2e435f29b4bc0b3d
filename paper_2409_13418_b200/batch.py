"""Throughput mode: many extractions on one GPU (BASELINE config 5).

``contour_batch(jobs)`` takes (field, grid) pairs.  Analytic fields on grids
of one resolution run as ONE batched extraction (``odc_extract_batch``): the
shapes' grids are stacked along z, so every stage is a single launch over
all of them and the host round trips of an extraction are paid once per
batch.  Each result equals ``contour(field, grid)`` of that job alone (the
reference extracts the shapes one by one, ``occmesh.pipeline.contour``,
pipeline.py:154-240; a shape's elements never meet another's, search.py:1-6).

Anything else (MLP / winding / voxel fields, mixed resolutions, fd normals,
the marching-cubes baseline) runs as concurrent ``contour`` calls, one libodc
context and stream per worker thread (ctypes releases the GIL in the C
calls).  Both paths are the GPU; there is no CPU fallback.
"""

from __future__ import annotations

import ctypes
import threading
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from . import _lib
from .fields import LoweringError, field_continuous, is_mesh_winding, is_mlp, is_voxels, lower_program
from .mesh import TriangleMesh
from .pipeline import (ContourOptions, ContourResult, DeviceField, EvalCounter, _grid_args, _host_arrays, _raise,
                       contour, make_options, record_counts, stats_dict)

# Worker w of a threaded batch always runs jobs w, w + W, w + 2W, ... on its
# own persistent libodc context, so each context's workspace settles at the
# size of the same shapes on every call (no re-allocation, deterministic).
_state: dict = {}
_state_lock = threading.Lock()


def _workers(device, workers):
    with _state_lock:
        key = (device, workers)
        if key not in _state:
            _state[key] = (ThreadPoolExecutor(max_workers=workers, thread_name_prefix=f"odc{device}"),
                           [_lib.Context(device) for _ in range(workers)], threading.Lock())
        return _state[key]


def _batch_context(device):
    with _state_lock:
        key = (device, "batch")
        if key not in _state:
            _state[key] = (_lib.Context(device), threading.Lock())
        return _state[key]


def batchable(jobs, options):
    """The single-launch batch path applies: analytic fields, one resolution,
    dual contouring with two-d-point normals."""
    if len(jobs) < 2 or options.normals != "two-d-points":
        return False
    R = int(jobs[0][1].resolution)
    cont = None
    for f, g in jobs:
        if int(g.resolution) != R or is_mlp(f) or is_mesh_winding(f) or is_voxels(f):
            return False
        try:
            lower_program(f)  # a device program (callback fields run through the threaded path)
        except LoweringError:
            return False
        c = bool(field_continuous(f))
        if cont is not None and c != cont:
            return False
        cont = c
    return (R + 1) ** 3 * len(jobs) < 2 ** 32


def contour_batch(jobs, options=None, *, workers=8, device=0, provenance=True, batched=None):
    """``jobs``: iterable of (field, grid).  Returns the ContourResults in
    order.  ``batched``: force (True) or forbid (False) the single-launch
    path; by default it is used whenever it applies (``batchable``)."""
    jobs = list(jobs)
    if not jobs:
        return []
    options = options or ContourOptions()
    options.validate()
    use = batchable(jobs, options) if batched is None else batched
    if use:
        return _contour_stacked(jobs, options, device=device, provenance=provenance)
    return _contour_threads(jobs, options, workers=workers, device=device, provenance=provenance)


def _contour_threads(jobs, options, *, workers, device, provenance):
    W = max(1, min(workers, len(jobs)))
    pool, ctxs, busy = _workers(device, W)

    def run(w):
        return [contour(f, g, options, device=device, provenance=provenance, _ctx=ctxs[w]) for f, g in jobs[w::W]]

    # the contexts (workspace, stream, pair counters) serve one call at a
    # time: concurrent contour_batch calls on the same pool queue here
    with busy:
        parts = list(pool.map(run, range(W)))
    out = [None] * len(jobs)
    for w, res in enumerate(parts):
        out[w::W] = res
    return out


def _contour_stacked(jobs, options, *, device, provenance):
    """All jobs in one odc_extract_batch call (see the module docstring)."""
    L = _lib.load()
    ctx, busy = _batch_context(device)
    nb = len(jobs)
    t0 = time.perf_counter()
    R = int(jobs[0][1].resolution)
    lo = np.empty((nb, 3))
    hi = np.empty((nb, 3))
    for b, (_, g) in enumerate(jobs):
        lo_b, hi_b, _ = _grid_args(g)
        lo[b] = list(lo_b)
        hi[b] = list(hi_b)
    o = make_options(options, False)
    stats = (_lib.Stats * nb)()
    with busy:
        dfields = [DeviceField(ctx, f) for f, _ in jobs]
        try:
            handles = (ctypes.c_void_p * nb)(*[d.handle.value for d in dfields])
            rc = L.odc_extract_batch(ctx.handle, handles, nb, lo.ctypes.data, hi.ctypes.data, R, ctypes.byref(o),
                                     ctypes.cast(stats, ctypes.c_void_p))
            if rc != _lib.ODC_OK:
                _raise(rc, ctx)
        finally:
            for d in dfields:
                d.free()
        vstart = np.zeros(nb + 1, dtype=np.int64)
        raw_v = np.zeros(nb, dtype=np.int64)
        tstart = np.zeros(nb + 1, dtype=np.int64)
        rc = L.odc_batch_layout(ctx.handle, vstart.ctypes.data, raw_v.ctypes.data, tstart.ctypes.data)
        if rc != _lib.ODC_OK:
            _raise(rc, ctx)
        V, T = int(vstart[-1]), int(tstart[-1])
        if provenance:  # one page-locked block: libodc DMAs straight into it (pipeline._host_arrays)
            v, t, rt, kind, ref = _host_arrays([((V, 3), np.float64), ((T, 3), np.int64), ((T, 3), np.int64),
                                                ((V,), np.int64), ((V, 2), np.int64)])
        else:
            v, t, rt = _host_arrays([((V, 3), np.float64), ((T, 3), np.int64), ((T, 3), np.int64)])
            kind = ref = None
        if V:
            ptr = lambda a: a.ctypes.data if a is not None and a.size else None  # noqa: E731
            rc = L.odc_copy_batch_meshes(ctx.handle, ptr(v), ptr(t), ptr(rt), ptr(kind), ptr(ref))
            if rc != _lib.ODC_OK:
                _raise(rc, ctx)
    wall = time.perf_counter() - t0
    out = []
    empty = TriangleMesh(np.zeros((0, 3)), np.zeros((0, 3), dtype=np.int64))
    for b, (field, _) in enumerate(jobs):
        st = stats[b]
        counter = EvalCounter(field)
        record_counts(counter, st)
        sd = stats_dict(st, options)
        if st.n_crossing_edges == 0:
            mesh = raw = empty
        else:
            v0, v1, t0_, t1 = vstart[b], vstart[b + 1], tstart[b], tstart[b + 1]
            vb = v[v0:v1]
            kb = kind[v0:v1] if kind is not None else None
            rb = ref[v0:v1] if ref is not None else None
            mesh = TriangleMesh.trusted(vb, t[t0_:t1], kb, rb)
            if st.repair_added_vertices == 0:
                raw = mesh
            else:
                n0 = int(raw_v[b])
                raw = TriangleMesh.trusted(vb[:n0], rt[t0_:t1], kb[:n0] if kb is not None else None,
                                           rb[:n0] if rb is not None else None)
        sd["wall_time_s"] = wall
        sd["eval_counts"] = counter.snapshot()
        sd["device_ms"] = float(st.device_ms)
        sd["batch_size"] = nb
        out.append(ContourResult(mesh, raw, counter, sd))
    return out
