"""Throughput mode: many extractions in flight on one GPU (BASELINE config 5).

Each worker thread drives its own libodc context (own stream and workspace);
ctypes releases the GIL inside the C calls, so while one extraction waits on
a count read-back the others' kernels keep the GPU busy.  Results are
identical to sequential ``contour`` calls (every extraction is independent
and deterministic).
"""

from __future__ import annotations

from concurrent.futures import ThreadPoolExecutor

from .pipeline import contour


def contour_batch(jobs, options=None, *, workers=8, device=0, provenance=True):
    """``jobs``: iterable of (field, grid).  Returns the ContourResults in order."""
    jobs = list(jobs)
    if not jobs:
        return []

    def run(job):
        field, grid = job
        return contour(field, grid, options, device=device, provenance=provenance)

    with ThreadPoolExecutor(max_workers=max(1, min(workers, len(jobs)))) as pool:
        return list(pool.map(run, jobs))
