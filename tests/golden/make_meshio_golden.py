"""Golden hashes for the mesh writers: run the reference's own
occmesh.meshio.export_obj / export_ply (/root/reference, importable in the
build container only) on the golden meshes of tests/golden/*.npz and on a
synthetic mesh with awkward floats, and record sha256 + size of the bytes.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_meshio_golden.py
"""
import hashlib
import json
import sys
import tempfile
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")
from occmesh.mesh import TriangleMesh  # noqa: E402
from occmesh.meshio import export_obj, export_ply  # noqa: E402


def awkward_mesh():
    rng = np.random.default_rng(5)
    v = np.concatenate([
        rng.normal(size=(40, 3)) * 10.0 ** rng.integers(-12, 12, size=(40, 1)),
        np.array([[0.0, -0.0, 1e-5], [1e300, -1e-300, 5e-324], [0.1, 0.2, 0.3], [1 / 3, 2 / 3, 1.0]]),
    ])
    t = rng.integers(0, len(v), size=(60, 3))
    t = t[(t[:, 0] != t[:, 1]) & (t[:, 1] != t[:, 2]) & (t[:, 0] != t[:, 2])]
    return v, t


def main():
    out = {}
    cases = {}
    for name in ("sphere_32", "torus_32", "mlp_amp4_32", "csg_difference_64"):
        f = HERE / f"{name}.npz"
        if f.exists():
            d = np.load(f)
            cases[name] = (d["vertices"], d["triangles"])
    cases["awkward"] = awkward_mesh()
    cases["empty"] = (np.zeros((0, 3)), np.zeros((0, 3), dtype=np.int64))
    np.savez_compressed(HERE / "meshio_awkward.npz", vertices=cases["awkward"][0], triangles=cases["awkward"][1])
    with tempfile.TemporaryDirectory() as td:
        for name, (v, t) in cases.items():
            m = TriangleMesh(v, t)
            rec = {}
            for ext, fn in (("obj", export_obj), ("ply", export_ply)):
                p = Path(td) / f"{name}.{ext}"
                fn(m, p)
                b = p.read_bytes()
                rec[ext] = {"sha256": hashlib.sha256(b).hexdigest(), "bytes": len(b)}
            out[name] = rec
    (HERE / "meshio.json").write_text(json.dumps(out, indent=1) + "\n")
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
