"""SURVEY 8(c) parity mode 2 for the MLP field: the device path (bf16
operands, fp32 accumulation, tcgen05) against the reference's own float32
numpy MlpField run through the CPU oracle pipeline (the reference algorithm,
pinned bit for bit elsewhere).  Reports grid-label agreement over all S^3
vertices and the distance between the two meshes (symmetric mean squared
surface distance metric_md2 and the sampled Hausdorff distance metric_hdd,
metrics.py:18-66) in units of the cell size h.

    python scripts/mlp_fp32_agreement.py --R 64 128 --out profiles/r2_mlp_fp32_agreement.json
"""
import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import oracle  # noqa: E402  (test infrastructure: the CPU reference side of the comparison)
from paper_2409_13418_b200 import GridSpec, MlpField, contour  # noqa: E402
from paper_2409_13418_b200.mesh import TriangleMesh  # noqa: E402
from paper_2409_13418_b200.metrics import metric_hdd, metric_md2  # noqa: E402
from paper_2409_13418_b200.pipeline import stage_arrays  # noqa: E402


def compare(R, amplitude=1.0, n=50000):
    field = MlpField(seed=0, amplitude=amplitude)
    lo, hi = (0.0, 0.0, 0.0), (1.0, 1.0, 1.0)
    h = 1.0 / R
    res, ctx, _ = contour(field, GridSpec(lo, hi, R), keep_intermediates=True, return_context=True)
    gl = stage_arrays(ctx, ["labels"])["labels"]
    t = time.perf_counter()
    o = oracle.contour_oracle(field, lo, hi, R)  # numpy float32 MlpField, C pipeline
    cpu_s = time.perf_counter() - t
    cpu = TriangleMesh.trusted(o["vertices"], o["triangles"])
    gpu = res.mesh
    agree = float(np.mean(gl == o["labels"]))
    return {
        "R": R, "amplitude": amplitude, "grid_vertices": int(gl.size),
        "label_agreement": agree, "label_mismatches": int(np.sum(gl != o["labels"])),
        "gpu_triangles": int(gpu.n_triangles), "cpu_fp32_triangles": int(cpu.n_triangles),
        "md2_over_h2": float(metric_md2(gpu, cpu, n=n) / h ** 2),
        "hdd_over_h": float(metric_hdd(gpu, cpu, n=n) / h),
        "cpu_fp32_pipeline_s": cpu_s,
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--R", type=int, nargs="+", default=[64, 128])
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    rows = []
    for R in a.R:
        r = compare(R)
        print(json.dumps(r), flush=True)
        rows.append(r)
    if a.out:
        Path(a.out).write_text(json.dumps({
            "what": "MLP 512^3 config's field (MlpField seed 0, amplitude 1): device bf16/tcgen05 path vs the "
                    "reference float32 numpy MlpField through the CPU oracle pipeline; label agreement over the "
                    "whole S^3 grid, mesh distances in cell units",
            "results": rows}, indent=1))


if __name__ == "__main__":
    main()
