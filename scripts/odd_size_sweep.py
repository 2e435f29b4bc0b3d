"""Robustness sweep: odd resolutions and domains, MLP (shared-field oracle)
and analytic fields (oracle), mesh identical to the oracle's."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import oracle  # noqa: E402
from paper_2409_13418_b200 import GridSpec, MlpField, SharedField, contour, scenes  # noqa: E402

bad = 0
for R in (2, 3, 5, 17, 33, 63, 100):
    for name in ("mlp", "torus", "csg_union"):
        if name == "mlp":
            f = MlpField(seed=R, amplitude=2.0)
            lo, hi = (0.0, 0.05, -0.1), (1.0, 0.9, 1.1)
            sh = SharedField(f)
            try:
                o = oracle.contour_oracle(f, lo, hi, R, continuous=True, raw_fn=lambda p, c: sh.eval_raw(p))
            finally:
                sh.close()
        else:
            f, lo, hi = scenes.resolve(scenes.SCENES[name], R)
            o = oracle.contour_oracle(f, lo, hi, R)
        r = contour(f, GridSpec(lo, hi, R))
        ok = np.array_equal(r.mesh.triangles, o["triangles"]) and (
            len(o["vertices"]) == 0 or np.abs(r.mesh.vertices - o["vertices"]).max() <= 1e-4 * min(
                (np.asarray(hi) - np.asarray(lo)) / R))
        bad += not ok
        print(f"R={R:4d} {name:10s} V={r.mesh.n_vertices:7d} T={r.mesh.n_triangles:7d} {'ok' if ok else 'MISMATCH'}")
print("mismatches:", bad)
sys.exit(1 if bad else 0)
