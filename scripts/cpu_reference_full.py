"""One full-size run of the CPU reference arm, cached for bench.py.

The reference arm (bench.py --impl reference) is the oracle port -- the C
restatement of occmesh.pipeline.contour with numpy's own LAPACK for the QEF
-- plus the numpy fp32 MlpField, on the host cores.  At 512^3 that is
~2x10^8 MLP evaluations (~15-35 min), too long to repeat inside every
bench run, so it is measured once per host class here and cached by input
hash; each bench run re-times a bounded sample live and scales the cached
full-size time by the live/cached sample ratio (a different or busier host
shows up as a ratio != 1).

    python scripts/cpu_reference_full.py --workload mlp_512 --out profiles/r2_cpu_reference_mlp_512.json
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import platform
import statistics
import sys
import time
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor()


def input_hash(field, lo, hi, R):
    """Hash of everything that determines the workload: field parameters and
    weights (or the lowered program), the box and the resolution."""
    from paper_2409_13418_b200.fields import is_mlp, lower_program

    h = hashlib.sha256()
    h.update(repr((tuple(map(float, lo)), tuple(map(float, hi)), int(R))).encode())
    if is_mlp(field):
        for a in list(field.weights) + list(field.biases) + [field.w_head]:
            h.update(np.ascontiguousarray(a).tobytes())
        h.update(repr((field.b_head, field.amplitude, field.prior_center.tolist(), field.prior_radius,
                       field.prior_scale)).encode())
    else:
        h.update(np.ascontiguousarray(lower_program(field)).tobytes())
    return h.hexdigest()[:16]


def time_oracle(field, lo, hi, R):
    import oracle

    t0 = time.perf_counter()
    o = oracle.contour_oracle(field, lo, hi, R)
    return time.perf_counter() - t0, o


def main():
    import threadpoolctl

    import bench

    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="mlp_512")
    ap.add_argument("--sample-r", type=int, default=64)
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    field, lo, hi, R, desc = bench.workload(a.workload)
    cores = len(os.sched_getaffinity(0))
    samples = [time_oracle(field, lo, hi, a.sample_r)[0] for _ in range(3)]
    print(f"sample {a.sample_r}^3: {samples}", flush=True)
    t_full, o = time_oracle(field, lo, hi, R)
    print(f"full {R}^3: {t_full:.1f} s", flush=True)
    rec = {
        "workload": a.workload, "desc": desc, "R": R, "cells": R**3, "input_hash": input_hash(field, lo, hi, R),
        "full_wall_s": t_full, "cells_per_s": R**3 / t_full,
        "total_evals": int(o["eval_counts"]["total_evals"]), "V": int(len(o["vertices"])),
        "T": int(len(o["triangles"])),
        "sample_r": a.sample_r, "sample_wall_s": statistics.median(samples), "sample_wall_s_all": samples,
        "host": {"cpu": cpu_model(), "cores": cores, "node": platform.node(),
                 "blas": [{k: i.get(k) for k in ("internal_api", "version", "architecture", "num_threads")}
                          for i in threadpoolctl.threadpool_info()]},
        "impl": "oracle port: C lock-step pipeline (1 thread, numpy LAPACK dsyevd for the QEF) + numpy fp32 "
                "MlpField (OpenBLAS sgemm, all host threads)",
        "measured_at": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime()),
    }
    Path(a.out).parent.mkdir(parents=True, exist_ok=True)
    Path(a.out).write_text(json.dumps(rec, indent=1))
    print(json.dumps(rec))


if __name__ == "__main__":
    main()
