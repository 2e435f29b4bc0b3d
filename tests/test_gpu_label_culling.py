"""The grid-label pass decides a whole label word (32 vertices) from one
interval bound of the field over the word's vertices (k_labels_analytic,
field_label_ball): these cases try to break that bound -- features smaller
than a word, surfaces through grid vertices, non-orthonormal "rotations"
(the Lipschitz factor is the matrix norm), negative sharpness, iso levels
off 1/2, far-away domains (rounding margins scale with magnitudes), and a
deep CSG program (the interval interpreter rather than the fast paths).
Labels and the extracted mesh must equal the oracle's bit for bit
(grid.py:109-126, pipeline.py:154-240)."""

import numpy as np
import pytest

import oracle
from paper_2409_13418_b200 import (BoxField, CsgField, GridSpec, PlaneField, SmoothedOccupancy, SphereField,
                                   TorusField, contour, rotation_from_euler)
from paper_2409_13418_b200.pipeline import stage_arrays

pytestmark = pytest.mark.gpu


def _scaled_rotation(s, rx, ry, rz):
    return s * np.asarray(rotation_from_euler(rx, ry, rz))


def _cases():
    R = 64
    h = 1.0 / R
    yield "tiny_sphere", SphereField((0.5 + 0.3 * h, 0.5 + 0.1 * h, 0.5), 0.35 * h), (0, 0, 0), (1, 1, 1), R
    yield "sphere_through_vertices", SphereField((0.5, 0.5, 0.5), 16 * h), (0, 0, 0), (1, 1, 1), R
    yield "scaled_rotation_box", BoxField((0.5, 0.5, 0.5), (0.2, 0.05, 0.12),
                                          rotation=_scaled_rotation(1.7, 20, 35, 10)), (0, 0, 0), (1, 1, 1), R
    yield "shrinking_transform", CsgField("transform", [TorusField((0, 0, 0), 0.5, 0.1)],
                                          rotation=_scaled_rotation(2.5, 10, 0, 30),
                                          translation=(0.5, 0.5, 0.5)), (0, 0, 0), (1, 1, 1), R
    yield "plane_tilted", PlaneField((0.5, 0.5, 0.5), (1e-3, 1.0, 2.0)), (0, 0, 0), (1, 1, 1), R
    neg = SmoothedOccupancy(SphereField((0.5, 0.5, 0.5), 0.3), -40.0)
    yield "smoothed_negative_k", neg, (0, 0, 0), (1, 1, 1), R
    iso = SmoothedOccupancy(BoxField((0.5, 0.5, 0.5), (0.3, 0.2, 0.25)), 60.0)
    iso.iso_level = 0.9
    yield "smoothed_iso_0.9", iso, (0, 0, 0), (1, 1, 1), R
    far = SphereField((1000.5, -2000.5, 3000.5), 0.3)
    yield "far_domain", far, (1000.0, -2001.0, 3000.0), (1001.0, -2000.0, 3001.0), R
    shell = CsgField("difference", [SphereField((0.5, 0.5, 0.5), 0.35), SphereField((0.5, 0.5, 0.5), 0.35 - 0.4 * h)])
    yield "shell_thinner_than_a_cell", shell, (0, 0, 0), (1, 1, 1), R
    rng = np.random.default_rng(7)
    balls = [SphereField(tuple(rng.uniform(0.2, 0.8, 3)), float(rng.uniform(0.02, 0.12))) for _ in range(9)]
    deep = CsgField("difference", [CsgField("union", balls), BoxField((0.5, 0.5, 0.3), (0.4, 0.4, 0.05))])
    yield "deep_program", deep, (0, 0, 0), (1, 1, 1), R


@pytest.mark.parametrize("name,field,lo,hi,R", list(_cases()), ids=[c[0] for c in _cases()])
def test_culled_labels_and_mesh_match_oracle(name, field, lo, hi, R):
    res, ctx, st = contour(field, GridSpec(lo, hi, R), keep_intermediates=True, return_context=True)
    arrs = stage_arrays(ctx, ["labels", "edge_key", "cells"])
    o = oracle.contour_oracle(field, lo, hi, R)
    assert np.array_equal(arrs["labels"], o["labels"]), name
    assert np.array_equal(arrs["edge_key"], o["edge_key"])
    assert np.array_equal(arrs["cells"], o["cells"])
    assert np.array_equal(res.mesh.triangles, o["triangles"])
    # smoothed fields: the device exp may differ from glibc in the last ulp
    assert np.abs(res.mesh.vertices - o["vertices"]).max(initial=0.0) <= 1e-9 * max(1.0, float(np.abs(lo).max()))
