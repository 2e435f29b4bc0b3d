"""Run the config-5 batch (64 shapes at 256^3 by default) through
contour_batch a few times (for ncu launch lists)."""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2409_13418_b200 import GridSpec, scenes  # noqa: E402
from paper_2409_13418_b200.batch import contour_batch  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=64)
ap.add_argument("--R", type=int, default=256)
ap.add_argument("--reps", type=int, default=1)
a = ap.parse_args()
jobs = []
for s in scenes.batch_shapes(a.n):
    f, lo, hi = scenes.resolve(s, a.R)
    jobs.append((f, GridSpec(lo, hi, a.R)))
for _ in range(a.reps):
    res = contour_batch(jobs)
print(len(res), sum(r.mesh.n_vertices for r in res), "%.3f ms" % res[0].stats["device_ms"],
      "repaired shapes", sum(1 for r in res if r.stats.get("repair_added_vertices")))
