"""Golden outputs of the reference's distance machinery and metrics:
occmesh.mesh.MeshDistanceIndex.query and occmesh.metrics.metric_md2 /
metric_hdd / metric_nic (metrics.py:26-66), on golden meshes, run here.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_metrics_golden.py
"""
import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")
from occmesh.mesh import MeshDistanceIndex, TriangleMesh  # noqa: E402
from occmesh.metrics import metric_hdd, metric_md2, metric_nic  # noqa: E402


def mesh(name):
    d = np.load(HERE / f"{name}.npz")
    return TriangleMesh(d["vertices"], d["triangles"])


def main():
    rng = np.random.default_rng(11)
    pts = np.concatenate([rng.random((400, 3)), 0.5 + 0.31 * rng.normal(size=(400, 3)) / 1.7,
                          rng.random((50, 3)) * 3 - 1])
    arrays = {"points": pts}
    for name in ("sphere_32", "torus_32", "mlp_amp4_32"):
        d, t, c = MeshDistanceIndex(mesh(name)).query(pts)
        arrays[f"{name}_dist"], arrays[f"{name}_tri"], arrays[f"{name}_cp"] = d, t, c
    np.savez_compressed(HERE / "distance_golden.npz", **arrays)
    out = {}
    for a, b in (("sphere_32", "sphere_64"), ("torus_32", "torus_64"), ("mlp_amp1_32", "mlp_amp4_32")):
        ma, mb = mesh(a), mesh(b)
        nic, dirs = metric_nic(ma, mb, n=3000, seed=3, return_directions=True)
        out[f"{a}|{b}"] = {"md2": metric_md2(ma, mb, n=3000, seed=3), "hdd": metric_hdd(ma, mb, n=3000, seed=3),
                           "nic": nic, "nic_directions": dirs}
    (HERE / "metrics.json").write_text(json.dumps(out, indent=1) + "\n")
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
