"""Evaluator kernel time (device-resident points, CUDA events) on points
near the MLP surface (mesh vertices, where the fp32 label test is
undecided) vs random points: value-dependent cost of the label epilogue."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2409_13418_b200 import GridSpec, MlpField, _lib, contour  # noqa: E402
from paper_2409_13418_b200.pipeline import DeviceField  # noqa: E402

f = MlpField(seed=0)
mesh = contour(f, GridSpec((0, 0, 0), (1, 1, 1), 256)).mesh
n = 2_381_176
rng = np.random.default_rng(0)
sets = {"near": np.ascontiguousarray(mesh.vertices[rng.integers(0, mesh.n_vertices, n)]),
        "random": np.ascontiguousarray(rng.uniform(0, 1, size=(n, 3)))}
ctx = _lib.Context(0)
L = _lib.load()
tr = np.zeros(2048, dtype=np.int64)
L.odc_set_param(ctx.handle, b"mlp_debug", 192)
with DeviceField(ctx, f) as df:
    for _ in range(100):
        L.odc_profile_mlp(ctx.handle, df.handle, 8_000_000, tr.ctypes.data, len(tr))
    for name, dbg in (("near", 192), ("random", 192), ("near", 208), ("near", 192), ("random", 192)):
        L.odc_set_param(ctx.handle, b"mlp_debug", dbg)
        L.odc_set_param(ctx.handle, b"profile_points", sets[name].ctypes.data)
        ms = []
        for _ in range(15):
            assert L.odc_profile_mlp(ctx.handle, df.handle, n, tr.ctypes.data, len(tr)) == 0
            ms.append(tr[-1] / 1e6)
        print(f"{name:7s} debug {dbg} median {np.median(ms):.3f} ms")
    L.odc_set_param(ctx.handle, b"profile_points", 0)
