"""Marching-cubes baseline (occmesh.baseline.marching_cubes, baseline.py:48-127).
The CPU oracle restatement is pinned to the reference's outputs
(tests/golden/mc_golden.*); the GPU path must match them."""

import json
from pathlib import Path

import numpy as np
import pytest

from oracle.mc import marching_cubes_oracle
from paper_2409_13418_b200 import GridSpec, MlpField, scenes

GOLDEN = Path(__file__).resolve().parent / "golden"
CASES = json.loads((GOLDEN / "mc_golden.json").read_text())
ARR = np.load(GOLDEN / "mc_golden.npz")


def scene_field(c):
    if c["scene"].startswith("mlp"):
        return MlpField(seed=0, amplitude=4.0), (0.0, 0.0, 0.0), (1.0, 1.0, 1.0)
    doc = scenes.thin_shell(c["R"]) if c["scene"] == "thin_shell" else scenes.SCENES[c["scene"]]
    return scenes.resolve(doc, c["R"])


@pytest.mark.parametrize("key", sorted(CASES))
def test_oracle_mc_matches_reference(key):
    c = CASES[key]
    f, lo, hi = scene_field(c)
    v, t, info = marching_cubes_oracle(f, lo, hi, c["R"], c["mode"])
    assert np.array_equal(t, ARR[f"{key}_t"])
    if key.startswith("mlp") and c["mode"] == "continuous":
        # raw values come from the numpy fp32 MLP: host BLAS kernels round differently
        assert np.abs(v - ARR[f"{key}_v"]).max() < 1e-6
    else:
        assert np.array_equal(v, ARR[f"{key}_v"])
    assert info["open_boundary"] == c["stats"]["open_boundary"]
    assert info["n_crossing_edges"] == c["stats"]["n_crossing_edges"]


@pytest.mark.gpu
@pytest.mark.parametrize("key", sorted(k for k in CASES if not k.startswith("mlp")))
def test_gpu_mc_matches_reference(key):
    from paper_2409_13418_b200.baseline import marching_cubes

    c = CASES[key]
    f, lo, hi = scene_field(c)
    res = marching_cubes(f, GridSpec(lo, hi, c["R"]), mode=c["mode"])
    assert np.array_equal(res.mesh.triangles, ARR[f"{key}_t"])
    v0 = ARR[f"{key}_v"]
    if c["mode"] == "continuous":  # device exp of the smoothed field: <= 1 ulp in raw
        assert np.abs(res.mesh.vertices - v0).max() <= 1e-12
    else:
        assert np.array_equal(res.mesh.vertices, v0)
    st = res.stats
    for k in ("method", "boundary_inside_vertices", "n_crossing_edges", "n_crossing_cells", "open_boundary"):
        assert st[k] == c["stats"][k], k
    ref_counts = {k: v for k, v in c["stats"]["eval_counts"].items()}
    assert st["eval_counts"] == ref_counts


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["binary", "continuous"])
def test_gpu_mc_mlp_shared_field(mode):
    from paper_2409_13418_b200 import SharedField
    from paper_2409_13418_b200.baseline import marching_cubes

    field = MlpField(seed=0, amplitude=4.0)
    shared = SharedField(field)
    res = marching_cubes(field, GridSpec((0, 0, 0), (1, 1, 1), 40), mode=mode)
    v, t, info = marching_cubes_oracle(field, (0, 0, 0), (1, 1, 1), 40, mode, raw_fn=lambda p, c: shared.eval_raw(p))
    assert np.array_equal(res.mesh.triangles, t) and np.array_equal(res.mesh.vertices, v)


@pytest.mark.gpu
def test_gpu_mc_errors():
    from paper_2409_13418_b200 import ConfigurationError, SphereField
    from paper_2409_13418_b200.baseline import marching_cubes

    g = GridSpec((0, 0, 0), (1, 1, 1), 16)
    with pytest.raises(ConfigurationError):
        marching_cubes(SphereField((0.5, 0.5, 0.5), 0.3), g, mode="continuous")
    with pytest.raises(ConfigurationError):
        marching_cubes(SphereField((0.5, 0.5, 0.5), 0.3), g, mode="cubic")
    empty = marching_cubes(SphereField((5.0, 5.0, 5.0), 0.1), g)
    assert empty.mesh.n_triangles == 0 and empty.stats["open_boundary"] is False
