"""Run a workload's extraction a few times (for ncu / compute-sanitizer runs)."""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from bench import workload  # noqa: E402
from paper_2409_13418_b200 import GridSpec, contour  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="mlp_128")
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
field, lo, hi, R, desc = workload(a.workload)
for _ in range(a.reps):
    res = contour(field, GridSpec(lo, hi, R))
print(desc, res.mesh.n_vertices, res.mesh.n_triangles, "%.3f ms" % res.stats["device_ms"])
