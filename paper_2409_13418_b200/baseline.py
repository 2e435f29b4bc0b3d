"""Marching-cubes baseline and the staged ablation ladder (the reference's
occmesh.baseline, /root/reference/pkg/src/occmesh/baseline.py:1-127), on
the GPU.

``marching_cubes`` shares the dual pipeline's device stages (labels, active
sets, face-centre probes, the per-cell cycle table) and replaces the 1D/2D
searches and the QEF with one vertex per crossing edge and a fan per cycle
(libodc, ``odc_options.method``).  ``run_stage`` is ``contour`` with the
component substitutions of the ablation ladder.
"""

from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass

import numpy as np

from . import _lib
from .mesh import TriangleMesh
from .pipeline import (ConfigurationError, ContourOptions, ContourResult, DeviceField, EvalCounter, SearchBudget,
                       _copy_mesh, _grid_args, _raise, contour, make_options, record_counts)


@dataclass(frozen=True)
class StageConfig:
    """Component selection for the ablation ladder (baseline.py:23-33)."""

    one_d: str = "binary-search"
    normals: str = "two-d-points"
    split: str = "ic"


def run_stage(field, grid, stage, budget=None, counter=None, qef_truncation=0.1):
    """contour with the selected component substitutions (baseline.py:36-45)."""
    options = ContourOptions(one_d=stage.one_d, normals=stage.normals, split=stage.split,
                             budget=budget or SearchBudget(), qef_truncation=qef_truncation)
    return contour(field, grid, options, counter=counter)


def marching_cubes(field, grid, mode="binary", counter=None, *, device=0):
    """Marching-cubes surface, one vertex per crossing edge (baseline.py:48-127):
    ``mode`` "binary" = edge midpoints, "continuous" = inverse lerp of the raw
    grid values (continuous fields only); face ambiguities resolved by the
    face-centre label like the dual pipeline; fans oriented outward."""
    if mode not in ("binary", "continuous"):
        raise ConfigurationError(f"unknown marching-cubes mode {mode!r}")
    counter = counter or EvalCounter(field)
    t0 = time.perf_counter()
    stats = {"warnings": [], "method": f"mc:{mode}"}
    ctx = _lib.context(device)
    L = _lib.load()
    st = _lib.Stats()
    lo, hi, R = _grid_args(grid)
    o = make_options(ContourOptions())
    o.method = 1 if mode == "binary" else 2
    with DeviceField(ctx, field) as dfield:
        rc = L.odc_extract(ctx.handle, dfield.handle, lo, hi, R, ctypes.byref(o), ctypes.byref(st))
        if rc != _lib.ODC_OK:
            _raise(rc, ctx, dfield)
    bi = int(st.boundary_inside_vertices)
    stats["boundary_inside_vertices"] = bi
    if bi:
        stats["warnings"].append(f"{bi} boundary grid vertices are inside; the output will have an open boundary")
    stats["n_crossing_edges"] = int(st.n_crossing_edges)
    stats["n_crossing_cells"] = int(st.n_crossing_cells)
    record_counts(counter, st)
    if st.n_crossing_edges == 0:
        mesh = TriangleMesh(np.zeros((0, 3)), np.zeros((0, 3), dtype=np.int64))
        stats["open_boundary"] = False
    else:
        mesh = _copy_mesh(ctx, 0, st, provenance=False)
        stats["open_boundary"] = bool(st.raw_n_vertices < st.n_crossing_edges) and bi > 0
    stats["wall_time_s"] = time.perf_counter() - t0
    stats["eval_counts"] = counter.snapshot()
    stats["device_ms"] = float(st.device_ms)
    return ContourResult(mesh, mesh, counter, stats)
