"""CPU restatement of VoxelField.eval_raw -- TEST INFRASTRUCTURE ONLY (the
product evaluates it in csrc/odc_voxel.cu).  Trilinear interpolation of a
dense (nx, ny, nz) grid at origin + index * spacing, zero outside the grid
box, in the order of /root/reference/pkg/src/occmesh/fields.py:257-278 (x,
then y, then z lerps).  Pinned to the reference's values
(tests/golden/voxel_golden.npz, made by make_voxel_golden.py)."""

from __future__ import annotations

import numpy as np


def voxel_raw(origin, spacing, values, points):
    v = np.asarray(values, dtype=np.float64)
    p = np.asarray(points, dtype=np.float64).reshape(-1, 3)
    dims = np.array(v.shape)
    g = (p - np.asarray(origin, dtype=np.float64)) / np.asarray(spacing, dtype=np.float64)
    ok = np.all(g >= 0.0, axis=1) & np.all(g <= dims - 1, axis=1)
    out = np.zeros(len(p))
    if not ok.any():
        return out
    g = g[ok]
    i = np.clip(np.floor(g).astype(np.int64), 0, dims - 2)
    f = g - i
    x, y, z = i.T
    fx, fy, fz = f.T

    def lerp_x(dy, dz):
        return v[x, y + dy, z + dz] * (1 - fx) + v[x + 1, y + dy, z + dz] * fx

    c0 = lerp_x(0, 0) * (1 - fy) + lerp_x(1, 0) * fy
    c1 = lerp_x(0, 1) * (1 - fy) + lerp_x(1, 1) * fy
    out[ok] = c0 * (1 - fz) + c1 * fz
    return out
