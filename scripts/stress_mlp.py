"""Stress: repeated 512^3 MLP extractions on one context (dynamic pair
schedule, compacted batches) must give the identical mesh every time."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2409_13418_b200 import GridSpec, MlpField, contour  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 20
R = int(sys.argv[2]) if len(sys.argv) > 2 else 512
f = MlpField(seed=0)
g = GridSpec((0, 0, 0), (1, 1, 1), R)
ref = contour(f, g)
t0 = time.perf_counter()
for i in range(n):
    r = contour(f, g)
    assert np.array_equal(r.mesh.triangles, ref.mesh.triangles), i
    assert np.array_equal(r.mesh.vertices, ref.mesh.vertices), i
print(f"{n} x {R}^3 identical, {(time.perf_counter() - t0) / n * 1e3:.1f} ms per call")
