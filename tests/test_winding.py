"""MeshWindingField (occmesh.fields._winding_batch / MeshWindingField,
fields.py:281-386) on the GPU.  The CPU restatement (oracle/winding.py) is
pinned bit-for-bit to the reference's values; the device differs only by the
device atan2 (<= 2 ulp per triangle term), so raw values are compared with a
tolerance written here and labels / meshes exactly."""

from pathlib import Path

import numpy as np
import pytest

from oracle.winding import winding

GOLDEN = Path(__file__).resolve().parent / "golden"
G = np.load(GOLDEN / "winding_golden.npz")
RAW_TOL = 1e-11  # |device - numpy| winding number: atan2 ulps summed over 1280 terms


def test_oracle_winding_matches_reference():
    assert np.array_equal(winding(G["ico_v"], G["ico_t"], G["points"]), G["w_ico"])
    assert np.array_equal(winding(G["ico_v"], G["open_t"], G["points"][:600]), G["w_open"])


@pytest.mark.gpu
@pytest.mark.parametrize("which", ["ico", "open"])
def test_gpu_winding_values(which):
    from paper_2409_13418_b200 import MeshWindingField, eval_labels, eval_raw

    t = G["ico_t"] if which == "ico" else G["open_t"]
    pts = G["points"] if which == "ico" else G["points"][:600]
    want = G["w_ico"] if which == "ico" else G["w_open"]
    f = MeshWindingField(G["ico_v"], t)
    raw = eval_raw(f, pts)
    assert np.abs(raw - want).max() <= RAW_TOL
    assert np.array_equal(eval_labels(f, pts).astype(bool), want > 0.5)


@pytest.mark.gpu
def test_gpu_contour_mesh_field_matches_reference():
    from paper_2409_13418_b200 import GridSpec, MeshWindingField, contour

    R = int(G["R"])
    res = contour(MeshWindingField(G["ico_v"], G["ico_t"]), GridSpec((0, 0, 0), (1, 1, 1), R))
    assert np.array_equal(res.mesh.triangles, G["mesh_t"])
    assert np.abs(res.mesh.vertices - G["mesh_v"]).max() <= 1e-9 / R


@pytest.mark.gpu
def test_gpu_mesh_field_shared_oracle_stages():
    import oracle
    from paper_2409_13418_b200 import MeshWindingField, SharedField
    from test_gpu_parity import compare, gpu_run

    f = MeshWindingField(G["ico_v"], G["ico_t"])
    res, arrs = gpu_run(f, (0, 0, 0), (1, 1, 1), 32)
    shared = SharedField(f)
    try:
        o = oracle.contour_oracle(f, (0, 0, 0), (1, 1, 1), 32, continuous=True,
                                  raw_fn=lambda p, c: shared.eval_raw(p))
    finally:
        shared.close()
    compare(res, arrs, o)


@pytest.mark.gpu
def test_gpu_mesh_field_errors():
    from paper_2409_13418_b200 import MeshWindingField
    from paper_2409_13418_b200.pipeline import eval_raw

    with pytest.raises(ValueError):
        MeshWindingField(np.zeros((3, 3)), np.zeros((0, 3), dtype=np.int64))
    with pytest.raises(ValueError):
        eval_raw(MeshWindingField(np.zeros((3, 3)), np.array([[0, 1, 5]])), np.zeros((1, 3)))
