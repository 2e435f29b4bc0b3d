"""VoxelField (occmesh.fields.VoxelField, fields.py:245-278) on the GPU:
values, labels and the extracted mesh against the reference's own outputs
(tests/golden/voxel_golden.npz), and stage-wise against the oracle with the
device field shared."""

from pathlib import Path

import numpy as np
import pytest

import oracle
from oracle.voxel import voxel_raw

G = np.load(Path(__file__).resolve().parent / "golden" / "voxel_golden.npz")


def test_oracle_voxel_values_match_reference():
    assert np.array_equal(voxel_raw(G["origin"], G["spacing"], G["values"], G["points"]), G["raw"])


def test_oracle_voxel_mesh_matches_reference():
    from paper_2409_13418_b200 import VoxelField

    f = VoxelField(G["origin"], G["spacing"], G["values"])
    o = oracle.contour_oracle(f, tuple(G["lo"]), tuple(G["hi"]), int(G["R"]), continuous=True,
                              raw_fn=lambda p, c: voxel_raw(G["origin"], G["spacing"], G["values"], p))
    assert np.array_equal(o["triangles"], G["mesh_t"]) and np.array_equal(o["vertices"], G["mesh_v"])


@pytest.mark.gpu
def test_gpu_voxel_values():
    from paper_2409_13418_b200 import VoxelField, eval_labels, eval_raw

    f = VoxelField(G["origin"], G["spacing"], G["values"])
    raw = eval_raw(f, G["points"])
    assert np.array_equal(raw, G["raw"])
    assert np.array_equal(eval_labels(f, G["points"]).astype(bool), G["raw"] > 0.5)


@pytest.mark.gpu
def test_gpu_voxel_contour_matches_reference():
    from paper_2409_13418_b200 import GridSpec, VoxelField, contour

    R = int(G["R"])
    res = contour(VoxelField(G["origin"], G["spacing"], G["values"]), GridSpec(tuple(G["lo"]), tuple(G["hi"]), R))
    assert np.array_equal(res.mesh.triangles, G["mesh_t"])
    assert np.abs(res.mesh.vertices - G["mesh_v"]).max() <= 1e-9 / R


@pytest.mark.gpu
def test_gpu_voxel_stages_shared_oracle():
    from paper_2409_13418_b200 import ContourOptions, SharedField, VoxelField
    from test_gpu_parity import compare, gpu_run

    f = VoxelField(G["origin"], G["spacing"], G["values"])
    for opts in (None, ContourOptions(one_d="linear-interp"), ContourOptions(normals="fd-gradient")):
        res, arrs = gpu_run(f, tuple(G["lo"]), tuple(G["hi"]), 32, opts)
        shared = SharedField(f)
        try:
            o = oracle.contour_oracle(f, tuple(G["lo"]), tuple(G["hi"]), 32, options=opts, continuous=True,
                                      raw_fn=lambda p, c: shared.eval_raw(p))
        finally:
            shared.close()
        compare(res, arrs, o)


@pytest.mark.gpu
def test_gpu_voxel_errors():
    from paper_2409_13418_b200 import VoxelField
    from paper_2409_13418_b200.pipeline import eval_raw

    with pytest.raises(ValueError):
        VoxelField((0, 0, 0), (1, 1, 1), np.zeros((2, 2)))
    with pytest.raises(ValueError):
        eval_raw(VoxelField((0, 0, 0), (1, 1, 1), np.zeros((1, 4, 4))), np.zeros((1, 3)))
