"""Pin the C oracle against golden vectors from the unmodified reference.

The oracle calls the same LAPACK dsyevd numpy.linalg.eigh uses
(dualize.py:358) and must reproduce the reference bit-for-bit, every stage
and the mesh included.
"""

import numpy as np
import pytest

import oracle
from golden_util import cases, field_of, index, load

ALL = cases()


def _run(tag):
    field, lo, hi, R = field_of(tag)
    return oracle.contour_oracle(field, lo, hi, R)


EXACT_UPTO_QEF = ["labels", "edge_key", "v_in", "face_key", "face_n_crossing", "cells", "instance_edges",
                  "t1d", "pos1d", "pos2", "status", "part_cell", "part_index", "cyc_off", "cyc_edges",
                  "cyc_insts", "normals"]


@pytest.mark.parametrize("tag", ALL)
def test_oracle_lapack_bit_exact(tag):
    if oracle.numpy_dsyevd() is None:
        pytest.skip("numpy's LAPACK not loadable")
    g = load(tag)
    o = _run(tag)
    for k in EXACT_UPTO_QEF + ["qef_pos", "qef_rank", "split_cases", "raw_vertices", "raw_triangles",
                               "raw_kind", "raw_ref", "vertices", "triangles", "kind", "ref"]:
        assert np.array_equal(np.asarray(g[k]), np.asarray(o[k])), k
    assert o["eval_counts"] == g["eval_counts"]
    assert o["n_probes"] == g["n_probes"]


def test_known_answers():
    kat = index()["kat"]
    from paper_2409_13418_b200.fields import PlaneField, SphereField

    o = oracle.contour_oracle(SphereField((0.5, 0.5, 0.5), 0.3), (0, 0, 0), (1, 1, 1), 2)
    assert o["labels"].tolist() == kat["sphere_R2_labels"]
    assert int(o["labels"].sum()) == 1 and o["labels"][13] == 1
    o = oracle.contour_oracle(SphereField((0.5, 0.5, 0.5), 0.1), (0, 0, 0), (1, 1, 1), 4)
    assert [len(o["edge_key"]), len(o["face_key"]), len(o["cells"])] == kat["single_vertex_R4"] == [6, 12, 8]
    o = oracle.contour_oracle(PlaneField((0, 0, 0.3), (0, 0, 1)), (0, 0, 0), (1, 1, 1), 4)
    assert len(o["edge_key"]) == kat["halfspace_R4_edges"] == 25


def test_eval_accounting():
    """S^3 + 15K + F4 + 46Q."""
    g = load("rotated_box_64")
    ec = g["eval_counts"]
    S3 = 65**3
    K = len(g["edge_key"])
    Q = len(g["instance_edges"])
    F4 = int(g["n_probes"])
    assert ec["labels"] == {"batches": 1, "evals": S3}
    assert ec["search_1d"] == {"batches": 15, "evals": 15 * K}
    assert ec["probe_face_midpoint"] == {"batches": 1, "evals": Q}
    assert ec["search_2d"] == {"batches": 30, "evals": 45 * Q}
    assert ec["total_evals"] == S3 + 15 * K + F4 + 46 * Q


def test_golden_cases_cover_every_2d_status():
    """Every find_2d_points status (search.py:308-313) occurs in some golden
    case, so the device's status logic is pinned branch by branch."""
    seen = set()
    for tag in ALL:
        g = load(tag)
        if "status" in g:
            seen |= set(np.unique(g["status"]).tolist())
    assert seen == {0, 1, 2, 3}
