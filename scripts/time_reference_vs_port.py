"""Time the UNMODIFIED reference (occmesh.pipeline.contour, imported from
/root/reference -- build container only) beside the oracle port that
bench.py's reference arm runs, on the same host, same inputs, and check
that they produce the same mesh.  Puts the port's speed relative to the
reference on record.

    python scripts/time_reference_vs_port.py --out profiles/r2_reference_vs_port.json
"""

from __future__ import annotations

import argparse
import json
import os
import platform
import sys
import time
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(REPO))
sys.path.insert(0, str(REPO / "tests" / "golden"))


def main():
    import threadpoolctl

    import occmesh
    import oracle
    from make_golden import ref_mlp_field
    from occmesh.fields import field_from_dict
    from paper_2409_13418_b200 import MlpField, scenes
    from paper_2409_13418_b200.fields import field_from_dict as our_field_from_dict

    ap = argparse.ArgumentParser()
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    cases = [("sphere", 256), ("torus", 256), ("mlp", 64), ("mlp", 128)]
    rows = []
    for name, R in cases:
        if name == "mlp":
            mf = MlpField(seed=0, amplitude=1.0)
            ref_field, port_field, lo, hi = ref_mlp_field(mf), mf, (0.0, 0.0, 0.0), (1.0, 1.0, 1.0)
        else:
            sc = scenes.SCENES[name]
            port_field, lo, hi = scenes.resolve(sc, R)
            ref_field = field_from_dict(sc["field"])
            assert type(our_field_from_dict(sc["field"])).__name__ == type(ref_field).__name__
        t0 = time.perf_counter()
        ref = occmesh.contour(ref_field, occmesh.GridSpec(lo, hi, R))
        t_ref = time.perf_counter() - t0
        t0 = time.perf_counter()
        o = oracle.contour_oracle(port_field, lo, hi, R)
        t_port = time.perf_counter() - t0
        same = bool(np.array_equal(ref.mesh.triangles, o["triangles"]) and
                    np.array_equal(ref.mesh.vertices, o["vertices"]))
        row = {"case": f"{name}_{R}", "reference_s": t_ref, "port_s": t_port, "port_speedup": t_ref / t_port,
               "total_evals": int(o["eval_counts"]["total_evals"]), "V": int(len(o["vertices"])),
               "identical_mesh": same}
        print(row, flush=True)
        rows.append(row)
        Path(a.out).write_text(json.dumps({
            "host": {"cpu": platform.processor() or "x86_64", "cores": len(os.sched_getaffinity(0)),
                     "blas": [{k: i.get(k) for k in ("internal_api", "version", "architecture", "num_threads")}
                              for i in threadpoolctl.threadpool_info()]},
            "note": "reference = unmodified occmesh.contour (pure Python + numpy; the MLP field is the numpy fp32 "
                    "MlpField adapter of tests/golden/make_golden.py); port = oracle/ (C pipeline, 1 thread, numpy "
                    "LAPACK dsyevd; same numpy fp32 MlpField through a callback)",
            "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime()), "rows": rows}, indent=1))


if __name__ == "__main__":
    main()
