"""Golden outputs of the reference's marching-cubes baseline
(occmesh.baseline.marching_cubes, baseline.py:48-127) on small scenes,
binary and continuous, run here from /root/reference.

    python tests/golden/make_mc_golden.py
"""
import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parent.parent
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(REPO))
sys.path.insert(0, str(HERE))

from occmesh import GridSpec  # noqa: E402
from occmesh.baseline import marching_cubes  # noqa: E402
from occmesh.fields import Scene, field_from_dict  # noqa: E402

from make_golden import ref_mlp_field  # noqa: E402
from paper_2409_13418_b200 import scenes as SC  # noqa: E402
from paper_2409_13418_b200.fields import MlpField  # noqa: E402

CASES = [("sphere", 32, "binary"), ("torus", 32, "binary"), ("rotated_box", 32, "binary"),
         ("csg_union", 32, "binary"), ("csg_difference", 32, "binary"), ("smooth_sphere", 32, "binary"),
         ("smooth_sphere", 32, "continuous"), ("thin_shell", 64, "binary"), ("mlp_amp4", 32, "binary"),
         ("mlp_amp4", 32, "continuous")]


def resolve(scene, R):
    doc = SC.SCENES[scene] if scene != "thin_shell" else SC.thin_shell(R)
    f = field_from_dict(doc["field"])
    sc = Scene(f, smooth_k=doc.get("smooth_k"))
    h = (sc.domain_hi - sc.domain_lo) / R
    return sc.resolve_field(h), GridSpec(sc.domain_lo, sc.domain_hi, R)


def main():
    out, arrays = {}, {}
    for scene, R, mode in CASES:
        if scene.startswith("mlp"):
            field = ref_mlp_field(MlpField(seed=0, amplitude=4.0))
            grid = GridSpec((0, 0, 0), (1, 1, 1), R)
        else:
            field, grid = resolve(scene, R)
        res = marching_cubes(field, grid, mode=mode)
        key = f"{scene}_{R}_{mode}"
        arrays[f"{key}_v"] = res.mesh.vertices
        arrays[f"{key}_t"] = res.mesh.triangles
        st = res.stats
        out[key] = {"scene": scene, "R": R, "mode": mode, "V": res.mesh.n_vertices, "T": res.mesh.n_triangles,
                    "stats": {k: st[k] for k in ("method", "boundary_inside_vertices", "n_crossing_edges",
                                                 "n_crossing_cells", "open_boundary", "eval_counts")}}
        print(key, out[key]["V"], out[key]["T"])
    np.savez_compressed(HERE / "mc_golden.npz", **arrays)
    (HERE / "mc_golden.json").write_text(json.dumps(out, indent=1) + "\n")


if __name__ == "__main__":
    main()
