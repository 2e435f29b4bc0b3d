"""Where the end-to-end time of contour_batch (config 5) goes: cProfile of
a warm call (host-side phases; the device work shows up as the ctypes call
that waits for it)."""
import cProfile
import pstats
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2409_13418_b200 import GridSpec, scenes  # noqa: E402
from paper_2409_13418_b200.batch import contour_batch  # noqa: E402

jobs = []
for s in scenes.batch_shapes(64):
    f, lo, hi = scenes.resolve(s, 256)
    jobs.append((f, GridSpec(lo, hi, 256)))
for _ in range(3):
    contour_batch(jobs)
t0 = time.perf_counter()
contour_batch(jobs)
print("warm call %.1f ms" % ((time.perf_counter() - t0) * 1e3))
pr = cProfile.Profile()
pr.enable()
contour_batch(jobs)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
