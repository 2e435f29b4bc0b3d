"""Property-style parity: random CSG scenes (spheres, boxes with arbitrary
rotations, tori, planes; union / intersection / difference / complement /
transform; optionally smoothed) at odd small resolutions and off-unit
domains, GPU vs the CPU oracle (pinned bit for bit to the reference) --
labels, crossing sets and the mesh, zero tolerance (the reference's own
field and pipeline tests at pkg/tests/test_fields.py and test_pipeline.py
cover the same field algebra on fixed cases)."""

import numpy as np
import pytest

import oracle
from paper_2409_13418_b200 import (BoxField, CsgField, GridSpec, PlaneField, SphereField, TorusField, contour,
                                   rotation_from_euler)
from paper_2409_13418_b200.pipeline import stage_arrays

pytestmark = pytest.mark.gpu


def _prim(rng):
    k = rng.integers(4)
    c = rng.uniform(0.25, 0.75, 3)
    if k == 0:
        return SphereField(c, float(rng.uniform(0.08, 0.3)))
    if k == 1:
        rot = rotation_from_euler(*rng.uniform(0, 90, 3)) if rng.random() < 0.7 else None
        return BoxField(c, rng.uniform(0.05, 0.25, 3), rotation=rot)
    if k == 2:
        return TorusField(c, float(rng.uniform(0.12, 0.22)), float(rng.uniform(0.03, 0.08)))
    n = rng.normal(size=3)
    return PlaneField(c, n)


def _field(rng, depth=0):
    if depth >= 2 or rng.random() < 0.35:
        return _prim(rng)
    op = ["union", "intersection", "difference", "complement", "transform"][rng.integers(5)]
    if op == "complement":
        return CsgField(op, [_field(rng, depth + 1)])
    if op == "transform":
        rot = rotation_from_euler(*rng.uniform(0, 60, 3))
        return CsgField(op, [_field(rng, depth + 1)], rotation=rot, translation=rng.uniform(-0.1, 0.1, 3))
    if op == "difference":
        return CsgField(op, [_field(rng, depth + 1), _field(rng, depth + 1)])
    return CsgField(op, [_field(rng, depth + 1) for _ in range(int(rng.integers(2, 4)))])


@pytest.mark.parametrize("seed", range(16))
def test_random_scene_matches_oracle(seed):
    rng = np.random.default_rng(1000 + seed)
    field = _field(rng)
    R = int(rng.choice([17, 23, 31, 40, 47]))
    lo = tuple(rng.uniform(-0.2, 0.1, 3))
    hi = tuple(np.asarray(lo) + rng.uniform(1.0, 1.4, 3))
    res, ctx, st = contour(field, GridSpec(lo, hi, R), keep_intermediates=True, return_context=True)
    arrs = stage_arrays(ctx, ["labels", "edge_key", "cells"])
    o = oracle.contour_oracle(field, lo, hi, R)
    assert np.array_equal(arrs["labels"], o["labels"])
    assert np.array_equal(arrs["edge_key"], o["edge_key"])
    assert np.array_equal(arrs["cells"], o["cells"])
    assert np.array_equal(res.mesh.triangles, o["triangles"])
    assert np.array_equal(res.mesh.vertices, o["vertices"])
    assert res.stats["eval_counts"] == o["eval_counts"]
