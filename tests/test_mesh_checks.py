"""Mesh validation (occmesh.mesh.validate_manifold, mesh.py:91-150): the CPU
oracle is pinned to the reference's outputs (tests/golden/checks.json); the
GPU implementation must match both exactly."""

import json
from pathlib import Path

import numpy as np
import pytest

from oracle import mesh_checks
from paper_2409_13418_b200 import TriangleMesh

GOLDEN = Path(__file__).resolve().parent / "golden"
CHECKS = json.loads((GOLDEN / "checks.json").read_text())


def golden_mesh(name):
    syn = np.load(GOLDEN / "checks_meshes.npz")
    if f"{name}_v" in syn:
        return syn[f"{name}_v"], syn[f"{name}_t"]
    raw = name.endswith("_raw")
    d = np.load(GOLDEN / f"{name[:-4] if raw else name}.npz")
    return (d["raw_vertices"], d["raw_triangles"]) if raw else (d["vertices"], d["triangles"])


def as_tuple(r):
    return (bool(r.manifold), [list(e) for e in r.nonmanifold_edges], list(r.pinched_vertices),
            int(r.boundary_edges), list(r.isolated_vertices))


def golden_tuple(g):
    return (g["manifold"], g["nonmanifold_edges"], g["pinched_vertices"], g["boundary_edges"],
            g["isolated_vertices"])


@pytest.mark.parametrize("name", sorted(CHECKS))
def test_oracle_validate_manifold_matches_reference(name):
    v, t = golden_mesh(name)
    assert mesh_checks.validate_manifold(v, t) == golden_tuple(CHECKS[name])


def random_soup(seed, nv=300, nt=900):
    """Triangles over few vertices: many shared edges (multiplicity > 2),
    pinched fans, boundary edges and isolated vertices."""
    rng = np.random.default_rng(seed)
    t = rng.integers(0, nv - 20, size=(nt, 3))
    t = t[(t[:, 0] != t[:, 1]) & (t[:, 1] != t[:, 2]) & (t[:, 0] != t[:, 2])]
    return rng.random((nv, 3)), t


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(CHECKS))
def test_gpu_validate_manifold_matches_reference(name):
    from paper_2409_13418_b200.mesh import validate_manifold

    v, t = golden_mesh(name)
    assert as_tuple(validate_manifold(TriangleMesh.trusted(v, t))) == golden_tuple(CHECKS[name])


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(6))
def test_gpu_validate_manifold_random_soups(seed):
    from paper_2409_13418_b200.mesh import validate_manifold

    v, t = random_soup(seed, nv=60 + 200 * seed, nt=200 + 3000 * seed)
    assert as_tuple(validate_manifold(TriangleMesh.trusted(v, t))) == mesh_checks.validate_manifold(v, t)


@pytest.mark.gpu
def test_gpu_validate_manifold_edge_cases():
    from paper_2409_13418_b200.mesh import validate_manifold

    empty = TriangleMesh(np.zeros((5, 3)), np.zeros((0, 3), dtype=np.int64))
    assert as_tuple(validate_manifold(empty)) == (True, [], [], 0, [])
    bad = TriangleMesh.trusted(np.zeros((3, 3)), np.array([[0, 1, 3]]))
    with pytest.raises(ValueError):
        validate_manifold(bad)
    # one vertex with a 400-triangle fan (a fan-triangulated disk)
    n = 400
    ang = np.linspace(0, 2 * np.pi, n, endpoint=False)
    v = np.concatenate([[[0, 0, 0]], np.stack([np.cos(ang), np.sin(ang), 0 * ang], 1)])
    t = np.stack([np.zeros(n, int), 1 + np.arange(n), 1 + (np.arange(n) + 1) % n], 1)
    assert as_tuple(validate_manifold(TriangleMesh.trusted(v, t))) == mesh_checks.validate_manifold(v, t)


@pytest.mark.gpu
def test_gpu_validate_extraction_mesh_keeps_context_result():
    """Validation runs in its own workspace: the last extraction stays readable."""
    from paper_2409_13418_b200 import GridSpec, SphereField, contour
    from paper_2409_13418_b200.mesh import validate_manifold

    res = contour(SphereField((0.5, 0.5, 0.5), 0.3), GridSpec((0, 0, 0), (1, 1, 1), 96))
    rep = validate_manifold(res.mesh)
    assert rep.manifold and rep.boundary_edges == 0 and not rep.isolated_vertices
    assert as_tuple(rep) == mesh_checks.validate_manifold(res.mesh.vertices, res.mesh.triangles)


# ---- count_self_intersections (mesh.py:395-487) ----------------------------
@pytest.mark.parametrize("name", sorted(CHECKS))
def test_oracle_self_intersections_match_reference(name):
    v, t = golden_mesh(name)
    assert [list(p) for p in mesh_checks.count_self_intersections(v, t)] == CHECKS[name]["si_pairs"]


def crossing_soup(seed, n=400):
    """Small random triangles in the unit box: many crossing pairs, a few
    coplanar overlaps (copies shifted in-plane), shared-vertex pairs."""
    rng = np.random.default_rng(seed)
    c = rng.random((n, 3))
    v = (c[:, None, :] + rng.normal(scale=0.04, size=(n, 3, 3))).reshape(-1, 3)
    t = np.arange(3 * n).reshape(-1, 3)
    k = n // 10  # coplanar partners: same plane, shifted inside it
    base = v[: 3 * k].reshape(k, 3, 3)
    shift = 0.3 * (base[:, 1] - base[:, 0]) + 0.2 * (base[:, 2] - base[:, 0])
    cop = (base + shift[:, None, :]).reshape(-1, 3)
    v = np.concatenate([v, cop])
    t = np.concatenate([t, 3 * n + np.arange(3 * k).reshape(-1, 3)])
    t[5] = [t[4][0], t[4][1], t[5][2]]  # two triangles sharing an edge
    return v, t


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(CHECKS))
def test_gpu_self_intersections_match_reference(name):
    from paper_2409_13418_b200.mesh import count_self_intersections

    v, t = golden_mesh(name)
    n, pairs = count_self_intersections(TriangleMesh.trusted(v, t), return_pairs=True)
    assert n == CHECKS[name]["si_count"] and [list(p) for p in pairs] == CHECKS[name]["si_pairs"]


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(4))
def test_gpu_self_intersections_random(seed):
    from paper_2409_13418_b200.mesh import count_self_intersections

    v, t = crossing_soup(seed, n=200 + 300 * seed)
    n, pairs = count_self_intersections(TriangleMesh.trusted(v, t), return_pairs=True)
    want = mesh_checks.count_self_intersections(v, t)
    assert n > 0 and pairs == want
    assert count_self_intersections(TriangleMesh.trusted(v, t), tolerance=1e-3) == len(
        mesh_checks.count_self_intersections(v, t, tolerance=1e-3))


@pytest.mark.gpu
def test_gpu_self_intersections_mlp_extraction():
    from paper_2409_13418_b200 import GridSpec, MlpField, contour
    from paper_2409_13418_b200.mesh import count_self_intersections

    res = contour(MlpField(seed=0, amplitude=4.0), GridSpec((0, 0, 0), (1, 1, 1), 48))
    m = res.mesh
    n, pairs = count_self_intersections(m, return_pairs=True)
    assert pairs == mesh_checks.count_self_intersections(m.vertices, m.triangles)
    assert count_self_intersections(TriangleMesh(np.zeros((3, 3)), np.array([[0, 1, 2]]))) == 0
