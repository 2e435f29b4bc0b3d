"""Golden VoxelField values and a voxel-field extraction from the reference
(occmesh.fields.VoxelField.eval_raw, fields.py:245-278; pipeline.contour).

    python tests/golden/make_voxel_golden.py
"""
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")
from occmesh import GridSpec  # noqa: E402
from occmesh.fields import VoxelField  # noqa: E402
from occmesh.pipeline import contour  # noqa: E402


def main():
    n = 17
    ax = np.linspace(0.0, 1.0, n)
    X, Y, Z = np.meshgrid(ax, ax, ax, indexing="ij")
    # a soft blob and a bar: raw crosses 0.5 on a smooth surface
    vals = 1.0 / (1.0 + np.exp(12.0 * (np.sqrt((X - 0.45) ** 2 + (Y - 0.5) ** 2 + (Z - 0.55) ** 2) - 0.28)))
    vals = np.maximum(vals, np.where((np.abs(X - 0.6) < 0.12) & (np.abs(Y - 0.5) < 0.3) & (np.abs(Z - 0.4) < 0.1), 0.9, 0))
    origin, spacing = (0.0, 0.0, 0.0), (1.0 / (n - 1),) * 3
    f = VoxelField(origin, spacing, vals)
    rng = np.random.default_rng(9)
    pts = np.concatenate([rng.random((2000, 3)) * 1.2 - 0.1, np.stack([ax, ax, ax], 1)])
    raw = f.eval_raw(pts)
    R = 40
    res = contour(f, GridSpec((0.02, 0.03, 0.01), (0.97, 0.98, 0.99), R))
    np.savez_compressed(HERE / "voxel_golden.npz", values=vals, origin=np.array(origin), spacing=np.array(spacing),
                        points=pts, raw=raw, R=R, lo=np.array([0.02, 0.03, 0.01]), hi=np.array([0.97, 0.98, 0.99]),
                        mesh_v=res.mesh.vertices, mesh_t=res.mesh.triangles)
    print(res.mesh.n_vertices, res.mesh.n_triangles)


if __name__ == "__main__":
    main()
