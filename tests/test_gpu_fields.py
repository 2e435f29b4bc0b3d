"""Field-level properties on the device evaluator, the reference's own test
strategy for the field boundary (/root/reference/pkg/tests/test_fields.py:
27-110, 181-194): label basics, the CSG algebra, rigid transforms, smoothed
occupancy, the iso tie, non-finite input.  The device labels come through
the C-ABI (odc_eval_labels / odc_eval_raw); the comparison values are
computed here in numpy."""

import numpy as np
import pytest

from paper_2409_13418_b200 import (
    BoxField,
    CsgField,
    PlaneField,
    SmoothedOccupancy,
    SphereField,
    TorusField,
    VoxelField,
    eval_labels,
    eval_raw,
    rotation_from_euler,
)

pytestmark = pytest.mark.gpu


def sphere_sd(p, c, r):
    return np.linalg.norm(p - np.asarray(c), axis=1) - r


def box_sd(p, c, half):
    q = np.abs(p - np.asarray(c)) - np.asarray(half)
    return np.linalg.norm(np.maximum(q, 0.0), axis=1) + np.minimum(q.max(axis=1), 0.0)


def test_sphere_labels_basic():
    f = SphereField((0.5, 0.5, 0.5), 0.3)
    assert eval_labels(f, (0.5, 0.5, 0.5)) == 1
    assert eval_labels(f, (0.99, 0.5, 0.5)) == 0


def test_sphere_labels_at_the_surface_match_the_oracle():
    """Points within a few ulps of a sphere: the device decides most labels
    from the exact sign of r^2 - s and takes the sqrt only in a thin band;
    every label must equal the oracle's sqrt(s) - r < 0 (fields.py:80-82)."""
    import oracle

    rng = np.random.default_rng(5)
    for c, r in (((0.5, 0.5, 0.5), 0.3), ((0.1, -0.2, 0.3), 1.0 / 3.0), ((0.0, 0.0, 0.0), 0.7071067811865476)):
        u = rng.normal(size=(200_000, 3))
        u /= np.linalg.norm(u, axis=1, keepdims=True)
        rad = r + rng.integers(-6, 7, size=len(u)) * np.spacing(r) * rng.uniform(0, 1, size=len(u))
        pts = np.asarray(c) + u * rad[:, None]
        f = SphereField(c, r)
        expect = (oracle.eval_raw_program(f, pts) > 0.5).astype(np.uint8)
        got = eval_labels(f, pts)
        assert 0 < expect.sum() < len(pts)
        assert np.array_equal(got, expect)


def test_union_is_max_of_children():
    a = SphereField((0.3, 0.5, 0.5), 0.1)
    b = SphereField((0.7, 0.5, 0.5), 0.1)
    p = (0.7, 0.5, 0.5)  # inside b only
    assert (eval_labels(a, p), eval_labels(b, p), eval_labels(CsgField("union", [a, b]), p)) == (0, 1, 1)


def test_nonfinite_point_rejected_with_index():
    f = SphereField((0.5, 0.5, 0.5), 0.3)
    pts = np.array([[0.5, 0.5, 0.5], [0.5, np.inf, 0.5], [np.nan, 0.5, 0.5]])
    with pytest.raises(ValueError, match="index 1"):
        eval_labels(f, pts)


def test_iso_tie_is_outside():
    """raw == iso level exactly (the zero set of a smoothed field) -> label 0."""
    f = SmoothedOccupancy(SphereField((0.0, 0.0, 0.0), 0.5), 4.0)
    assert eval_raw(f, np.array([[0.5, 0.0, 0.0]]))[0] == 0.5
    assert eval_labels(f, (0.5, 0.0, 0.0)) == 0


def test_csg_label_algebra_is_set_algebra():
    rng = np.random.default_rng(0)
    pts = rng.uniform(0, 1, size=(100_000, 3))
    a = SphereField((0.45, 0.5, 0.5), 0.25)
    b = BoxField((0.6, 0.5, 0.5), (0.2, 0.15, 0.3))
    in_a = sphere_sd(pts, (0.45, 0.5, 0.5), 0.25) < 0
    in_b = box_sd(pts, (0.6, 0.5, 0.5), (0.2, 0.15, 0.3)) < 0
    assert np.array_equal(eval_labels(CsgField("union", [a, b]), pts) == 1, in_a | in_b)
    assert np.array_equal(eval_labels(CsgField("intersection", [a, b]), pts) == 1, in_a & in_b)
    assert np.array_equal(eval_labels(CsgField("difference", [a, b]), pts) == 1, in_a & ~in_b)
    assert np.array_equal(eval_labels(CsgField("complement", [a]), pts) == 1, ~in_a)


def test_csg_transform_is_rigid():
    rot = rotation_from_euler(0, 0, 90)
    base = BoxField((0.0, 0.0, 0.0), (0.2, 0.1, 0.1))
    moved = CsgField("transform", [base], rotation=rot, translation=(1.0, 0.0, 0.0))
    # the long axis now points along +y around (1, 0, 0)
    assert eval_labels(moved, (1.0, 0.15, 0.0)) == 1
    assert eval_labels(moved, (1.15, 0.0, 0.0)) == 0
    assert eval_labels(base, (0.15, 0.0, 0.0)) == 1


ROT_30_30 = rotation_from_euler(30, 30, 0)
BOX_C, BOX_H = (0.5033, 0.4987, 0.4942), (0.2452, 0.1976, 0.1469)


def torus_sd(p, c, big, small):
    q = p - np.asarray(c)
    return np.hypot(np.hypot(q[:, 0], q[:, 1]) - big, q[:, 2]) - small


@pytest.mark.parametrize("make,sd", [
    (lambda: SphereField((0.5, 0.5, 0.5), 0.3), lambda p: sphere_sd(p, (0.5, 0.5, 0.5), 0.3)),
    (lambda: TorusField((0.5, 0.5, 0.5), 0.27, 0.12), lambda p: torus_sd(p, (0.5, 0.5, 0.5), 0.27, 0.12)),
    (lambda: BoxField(BOX_C, BOX_H, rotation=ROT_30_30),
     lambda p: box_sd((p - np.asarray(BOX_C)) @ np.asarray(ROT_30_30), (0, 0, 0), BOX_H)),
])
def test_smoothed_labels_match_base(make, sd):
    base = make()
    sm = SmoothedOccupancy(base, 64.0)
    rng = np.random.default_rng(1)
    pts = rng.uniform(0, 1, size=(100_000, 3))
    off = np.abs(sd(pts)) > 1e-12  # on the zero set the smoothed raw is a 0.5 tie
    assert np.array_equal(eval_labels(sm, pts[off]), eval_labels(base, pts[off]))


def test_smoothed_raw_is_logistic_of_distance():
    k = 10.0
    sm = SmoothedOccupancy(PlaneField((0.0, 0.0, 0.0), (0.0, 0.0, 1.0)), k)
    z = np.array([-0.2, -0.05, 0.0, 0.05, 0.2])
    pts = np.stack([np.zeros(5), np.zeros(5), z], axis=1)
    assert np.allclose(eval_raw(sm, pts), 1.0 / (1.0 + np.exp(k * z)), atol=1e-12)


def test_voxel_field_trilinear():
    vals = np.zeros((2, 2, 2))
    vals[1, :, :] = 1.0  # raw = x inside the unit cell
    f = VoxelField((0.0, 0.0, 0.0), (1.0, 1.0, 1.0), vals)
    pts = np.array([[0.25, 0.5, 0.5], [0.75, 0.1, 0.9], [0.5, 0.5, 0.5]])
    assert np.allclose(eval_raw(f, pts), [0.25, 0.75, 0.5], atol=1e-15)
    assert list(eval_labels(f, pts)) == [0, 1, 0]  # 0.5 is a tie -> outside


@pytest.mark.parametrize("rx,ry,rz", [(0, 0, 0), (30, 30, 0), (10, -70, 200), (90, 90, 90)])
def test_euler_rotation_is_orthonormal(rx, ry, rz):
    r = np.asarray(rotation_from_euler(rx, ry, rz))
    assert np.allclose(r @ r.T, np.eye(3), atol=1e-12)
    assert np.isclose(np.linalg.det(r), 1.0)
