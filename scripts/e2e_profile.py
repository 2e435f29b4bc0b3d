"""Break down the end-to-end contour() call (host side) for a workload."""
import cProfile
import pstats
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from bench import workload  # noqa: E402
from paper_2409_13418_b200 import GridSpec, contour  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "mlp_512"
field, lo, hi, R, desc = workload(name)
g = GridSpec(lo, hi, R)
contour(field, g)
t0 = time.perf_counter()
res = contour(field, g)
t1 = time.perf_counter()
print("e2e %.1f ms, device %.1f ms" % ((t1 - t0) * 1e3, res.stats["device_ms"]))
pr = cProfile.Profile()
pr.enable()
contour(field, g)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
