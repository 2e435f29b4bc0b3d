"""Search a seeded stream of shapes leaving the unit box for extractions that
keep partition vertices no triangle references (open boundaries,
polygonize.py:204-214); tests/test_gpu_parity.py uses the cases found.

    python scripts/probe_unused_partitions.py
"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2409_13418_b200 import BoxField, GridSpec, PlaneField, SphereField, TorusField, contour  # noqa: E402


def main(n=400, want=7):
    rng = np.random.default_rng(0)
    found = 0
    for i in range(n):
        k = i % 4
        if k == 0:
            f = SphereField(tuple(rng.uniform(-0.2, 1.2, 3)), float(rng.uniform(0.2, 0.9)))
        elif k == 1:
            f = BoxField(tuple(rng.uniform(-0.2, 1.2, 3)), tuple(rng.uniform(0.1, 0.8, 3)))
        elif k == 2:
            f = PlaneField(tuple(rng.uniform(0, 1, 3)), tuple(rng.normal(size=3)))
        else:
            f = TorusField(tuple(rng.uniform(0, 1, 3)), float(rng.uniform(0.2, 0.5)), float(rng.uniform(0.05, 0.2)))
        R = int(rng.choice([9, 12, 16, 20]))
        res = contour(f, GridSpec((0, 0, 0), (1, 1, 1), R))
        if res.mesh.provenance_kind is None or res.stats.get("n_partitions", 0) == 0:
            continue
        used = int((res.raw_mesh.provenance_kind == 0).sum())
        if used < res.stats["n_partitions"]:
            found += 1
            print(f"case {i}: {type(f).__name__} at {R}^3, {used} of {res.stats['n_partitions']} partitions used, "
                  f"{res.stats.get('skipped_boundary_edges')} skipped boundary edges")
            if found >= want:
                break
    print("found", found)


if __name__ == "__main__":
    main()
