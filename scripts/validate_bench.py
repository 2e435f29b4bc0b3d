"""Time the GPU mesh checks on an extracted mesh (default: MLP 512^3):
validate_manifold, count_self_intersections, MD2 with 100k samples, and the
OBJ/PLY writers.  Prints one JSON line."""
import json
import sys
import tempfile
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from bench import workload  # noqa: E402
from paper_2409_13418_b200 import GridSpec, contour  # noqa: E402
from paper_2409_13418_b200.mesh import count_self_intersections, validate_manifold  # noqa: E402
from paper_2409_13418_b200.meshio import export_obj, export_ply  # noqa: E402
from paper_2409_13418_b200.metrics import metric_md2  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "mlp_512"
field, lo, hi, R, desc = workload(name)
m = contour(field, GridSpec(lo, hi, R)).mesh
out = {"workload": name, "V": m.n_vertices, "T": m.n_triangles}


def timed(key, fn, reps=3):
    fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        r = fn()
        ts.append(time.perf_counter() - t0)
    out[key + "_s"] = min(ts)
    return r


rep = timed("validate_manifold", lambda: validate_manifold(m))
out["manifold"] = rep.manifold
out["nonmanifold_edges"] = len(rep.nonmanifold_edges)
out["self_intersections"] = timed("count_self_intersections", lambda: count_self_intersections(m))
out["md2_100k"] = timed("metric_md2_100k", lambda: metric_md2(m, m, n=100_000), reps=1)
with tempfile.TemporaryDirectory() as td:
    timed("export_obj", lambda: export_obj(m, Path(td) / "m.obj"), reps=1)
    timed("export_ply", lambda: export_ply(m, Path(td) / "m.ply"), reps=1)
print(json.dumps(out))
if len(sys.argv) > 2:
    import cProfile
    import pstats

    pr = cProfile.Profile()
    pr.enable()
    metric_md2(m, m, n=100_000)
    pr.disable()
    pstats.Stats(pr, stream=sys.stderr).sort_stats("cumulative").print_stats(15)
