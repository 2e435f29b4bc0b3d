"""Distance queries and mesh metrics (occmesh.mesh.MeshDistanceIndex,
mesh.py:202-270; occmesh.metrics, metrics.py:18-66).  The CPU oracle is
pinned to the reference's own query outputs (tests/golden/distance_golden.npz,
metrics.json, made by make_metrics_golden.py); the GPU queries must match
them exactly: distances, closest triangles (including the reference's tie
rule) and closest points."""

import json
from pathlib import Path

import numpy as np
import pytest

from oracle import mesh_checks
from paper_2409_13418_b200 import TriangleMesh

GOLDEN = Path(__file__).resolve().parent / "golden"
DIST = np.load(GOLDEN / "distance_golden.npz")
METRICS = json.loads((GOLDEN / "metrics.json").read_text())
NAMES = ("sphere_32", "torus_32", "mlp_amp4_32")


def golden_mesh(name):
    d = np.load(GOLDEN / f"{name}.npz")
    return TriangleMesh.trusted(np.ascontiguousarray(d["vertices"]), np.ascontiguousarray(d["triangles"]))


@pytest.mark.parametrize("name", NAMES)
def test_oracle_distance_matches_reference(name):
    m = golden_mesh(name)
    d, t, c = mesh_checks.mesh_distance(m.vertices, m.triangles, DIST["points"])
    assert np.array_equal(d, DIST[f"{name}_dist"])
    assert np.array_equal(t, DIST[f"{name}_tri"])
    assert np.array_equal(c, DIST[f"{name}_cp"])


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_gpu_distance_matches_reference(name):
    from paper_2409_13418_b200.metrics import MeshDistanceIndex

    d, t, c = MeshDistanceIndex(golden_mesh(name)).query(DIST["points"])
    assert np.array_equal(d, DIST[f"{name}_dist"])
    assert np.array_equal(t, DIST[f"{name}_tri"])
    assert np.array_equal(c, DIST[f"{name}_cp"])


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(3))
def test_gpu_distance_random_meshes(seed):
    from paper_2409_13418_b200.metrics import MeshDistanceIndex

    rng = np.random.default_rng(seed)
    n = 150 + 400 * seed
    v = rng.random((n, 3)) * np.array([1.0, 0.3, 2.0])
    t = rng.integers(0, n, size=(2 * n, 3))
    t = t[(t[:, 0] != t[:, 1]) & (t[:, 1] != t[:, 2]) & (t[:, 0] != t[:, 2])]
    pts = np.concatenate([rng.random((300, 3)) * 3 - 1, v[:50]])  # far points and exact vertices
    d, tri, c = MeshDistanceIndex(TriangleMesh.trusted(v, t)).query(pts)
    d0, t0, c0 = mesh_checks.mesh_distance(v, t, pts)
    assert np.array_equal(d, d0) and np.array_equal(tri, t0) and np.array_equal(c, c0)


@pytest.mark.gpu
@pytest.mark.parametrize("pair", sorted(METRICS))
def test_gpu_metrics_match_reference(pair):
    from paper_2409_13418_b200.metrics import metric_hdd, metric_md2, metric_nic

    a, b = (golden_mesh(x) for x in pair.split("|"))
    g = METRICS[pair]
    assert metric_md2(a, b, n=3000, seed=3) == g["md2"]
    assert metric_hdd(a, b, n=3000, seed=3) == g["hdd"]
    nic, dirs = metric_nic(a, b, n=3000, seed=3, return_directions=True)
    assert nic == g["nic"] and dirs == g["nic_directions"]


@pytest.mark.gpu
def test_gpu_metric_fit_and_errors():
    from paper_2409_13418_b200 import GridSpec, SphereField, contour
    from paper_2409_13418_b200.fields import SmoothedOccupancy
    from paper_2409_13418_b200.metrics import MeshDistanceIndex, metric_fit

    f = SphereField((0.5, 0.5, 0.5), 0.3)
    m = contour(f, GridSpec((0, 0, 0), (1, 1, 1), 64)).mesh
    assert metric_fit(m, f) is None  # binary field
    sm = SmoothedOccupancy(f, 40.0)
    fit = metric_fit(m, sm, n=5000)
    assert 0.0 <= fit < 0.2
    with pytest.raises(ValueError):
        MeshDistanceIndex(TriangleMesh(np.zeros((0, 3)), np.zeros((0, 3), dtype=np.int64)))


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_gpu_triangle_areas_equal_numpy(name):
    from paper_2409_13418_b200.metrics import triangle_areas

    m = golden_mesh(name)
    assert np.array_equal(triangle_areas(m), m.areas())


@pytest.mark.gpu
@pytest.mark.parametrize("tag", ["sphere_64", "torus_64", "rotated_box_64", "csg_union_64", "csg_difference_64",
                                 "smooth_sphere_64", "thin_shell_64"])
def test_gpu_chamfer_to_reference_mesh(tag):
    """north_star's tolerance check: the GPU mesh against the reference's own
    mesh (golden) -- symmetric mean squared surface distance (metric_md2,
    metrics.py:26-32) and the sampled Hausdorff distance, both far below
    (1e-4 h)."""
    from golden_util import field_of, load
    from paper_2409_13418_b200 import GridSpec, contour
    from paper_2409_13418_b200.metrics import metric_hdd, metric_md2

    f, lo, hi, R = field_of(tag)
    ref = load(tag)
    ours = contour(f, GridSpec(lo, hi, R)).mesh
    theirs = TriangleMesh.trusted(ref["vertices"], ref["triangles"])
    h = 1.0 / R
    assert metric_md2(ours, theirs, n=20000) <= (1e-4 * h) ** 2
    assert metric_hdd(ours, theirs, n=20000) <= 1e-4 * h
