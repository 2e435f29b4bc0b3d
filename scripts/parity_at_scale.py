"""GPU parity against the CPU oracle at BASELINE.json's configuration sizes.

The oracle (oracle/, a C restatement of occmesh.pipeline.contour that calls
numpy's own LAPACK dsyevd for the QEF, pinned bit-for-bit to the unmodified
reference on the golden cases by tests/test_oracle_golden.py) runs on the
GPU box's host cores beside libodc; every stage array and both meshes are
compared with zero tolerance.  Any differing entry is listed.

    python scripts/parity_at_scale.py --cases c2,c3 --out gpurun_out/r2_parity.json

Cases (BASELINE.json configs):
  c1   sphere 64^3
  c2   torus / csg_union / csg_difference / rotated_box at 256^3
  c3   MLP 512^3, shared field (the oracle's field callback evaluates the
       same device MLP, so labels are identical and topology must match)
  c3b  MLP 128^3, GPU bf16 vs the numpy fp32 MlpField: grid-label agreement
       and MD2/HDD between the two meshes (SURVEY 8(c) parity mode 2)
  c4   thin shell 1024^3: one extraction, then z-slab decompositions (2/4/8
       slabs run serially on one GPU: same kernels and id arithmetic as the
       multi-GPU path) against it
  c5   the 64 config-5 shapes at 256^3 through contour_batch, each against
       the oracle
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))

import oracle  # noqa: E402
from paper_2409_13418_b200 import ContourOptions, GridSpec, MlpField, SharedField, contour, scenes  # noqa: E402
from paper_2409_13418_b200.fields import is_mlp  # noqa: E402
from paper_2409_13418_b200.pipeline import stage_arrays  # noqa: E402

STAGES = ["labels", "edge_key", "v_in", "face_key", "face_n_crossing", "cells", "instance_edges", "t1d", "pos1d",
          "pos2", "status", "part_cell", "part_index", "cyc_len", "cyc_edges", "cyc_insts", "normals", "qef_pos",
          "qef_rank", "split_cases"]


def gpu_run(field, lo, hi, R):
    t0 = time.perf_counter()
    res, ctx, st = contour(field, GridSpec(lo, hi, R), keep_intermediates=True, return_context=True)
    wall = time.perf_counter() - t0
    arrs = stage_arrays(ctx, STAGES)
    arrs["cyc_off"] = np.concatenate([[0], np.cumsum(arrs.pop("cyc_len"))])
    return res, arrs, wall


def oracle_run(field, lo, hi, R):
    t0 = time.perf_counter()
    if is_mlp(field):
        shared = SharedField(field)
        try:
            o = oracle.contour_oracle(field, lo, hi, R, continuous=True, raw_fn=lambda p, c: shared.eval_raw(p))
        finally:
            shared.close()
    else:
        o = oracle.contour_oracle(field, lo, hi, R)
    return o, time.perf_counter() - t0


def diff(a, b, name, h=None):
    a = np.asarray(a)
    b = np.asarray(b)
    if a.size == b.size:
        a = a.reshape(b.shape)
    d = {"n": int(b.shape[0]) if b.ndim else 1}
    if a.shape != b.shape:
        d.update(equal=False, shape_gpu=list(a.shape), shape_ref=list(b.shape))
        return d
    neq = a != b
    if neq.ndim > 1:
        neq = neq.reshape(neq.shape[0], -1).any(1)
    bad = np.nonzero(neq)[0]
    d["equal"] = bad.size == 0
    if bad.size:
        d["mismatches"] = int(bad.size)
        d["first_rows"] = bad[:10].tolist()
        if h is not None and a.dtype.kind == "f":
            d["max_abs_diff_in_h"] = float(np.abs(a - b).max() / h)
    return d


def compare(res, arrs, o):
    h = float(np.min(o["h"]))
    out = {}
    for k in STAGES[:-1] + ["cyc_off"]:
        if k == "cyc_len":
            continue
        out[k] = diff(arrs[k], o[k], k, h)
    out["split_cases"] = diff(arrs["split_cases"], o["split_cases"], "split_cases")
    out["raw_vertices"] = diff(res.raw_mesh.vertices, o["raw_vertices"], "raw_vertices", h)
    out["raw_triangles"] = diff(res.raw_mesh.triangles, o["raw_triangles"], "raw_triangles")
    out["vertices"] = diff(res.mesh.vertices, o["vertices"], "vertices", h)
    out["triangles"] = diff(res.mesh.triangles, o["triangles"], "triangles")
    out["provenance_kind"] = diff(res.mesh.provenance_kind, o["kind"], "kind")
    out["provenance_ref"] = diff(res.mesh.provenance_ref, o["ref"], "ref")
    out["eval_counts_equal"] = res.stats["eval_counts"] == o["eval_counts"]
    return out


def summarize(cmp):
    return all(v["equal"] for k, v in cmp.items() if isinstance(v, dict)) and cmp["eval_counts_equal"]


def sizes(res, o):
    return {"K": int(len(o["edge_key"])), "F": int(len(o["face_key"])), "C": int(len(o["cells"])),
            "Q": int(len(o["instance_edges"])), "P": int(len(o["qef_pos"])), "V": int(res.mesh.n_vertices),
            "T": int(res.mesh.n_triangles), "repair_added": int(res.stats.get("repair_added_vertices", 0)),
            "split_case_counts": {str(k): int(v) for k, v in res.stats.get("split_case_counts", {}).items()},
            "qef_rank_counts": {str(k): int(v) for k, v in res.stats.get("qef_rank_counts", {}).items()}}


def one_case(name, field, lo, hi, R):
    print(f"[{name}] gpu ...", flush=True)
    res, arrs, gw = gpu_run(field, lo, hi, R)
    print(f"[{name}] oracle ...", flush=True)
    o, ow = oracle_run(field, lo, hi, R)
    cmp = compare(res, arrs, o)
    ok = summarize(cmp)
    print(f"[{name}] bit-exact={ok} gpu {gw:.2f}s oracle {ow:.1f}s", flush=True)
    return {"case": name, "R": R, "bit_exact": ok, "sizes": sizes(res, o), "gpu_wall_s": gw, "oracle_wall_s": ow,
            "compare": cmp}


def _prov(a):
    """An empty mesh carries no provenance (pipeline.py:88-90): None == empty."""
    return np.zeros(0) if a is None else np.asarray(a).reshape(-1)


def mesh_equal(a, b):
    return {"vertices": bool(np.array_equal(a.vertices, b.vertices)),
            "triangles": bool(np.array_equal(a.triangles, b.triangles)),
            "provenance_kind": bool(np.array_equal(a.provenance_kind, b.provenance_kind)),
            "provenance_ref": bool(np.array_equal(a.provenance_ref, b.provenance_ref))}


def case_c1():
    field, lo, hi = scenes.resolve(scenes.SCENES["sphere"], 64)
    return [one_case("c1_sphere_64", field, lo, hi, 64)]


def case_c2():
    out = []
    for name in ("torus", "csg_union", "csg_difference", "rotated_box"):
        field, lo, hi = scenes.resolve(scenes.SCENES[name], 256)
        out.append(one_case(f"c2_{name}_256", field, lo, hi, 256))
    return out


def case_c3():
    return [one_case("c3_mlp_512_shared_field", MlpField(seed=0, amplitude=1.0), (0, 0, 0), (1, 1, 1), 512)]


def case_c3b(R=128):
    """GPU bf16 MLP vs the numpy fp32 MlpField (its own fp32 forward pass)."""
    from paper_2409_13418_b200.mesh import TriangleMesh
    from paper_2409_13418_b200.metrics import metric_hdd, metric_md2
    from paper_2409_13418_b200.pipeline import eval_labels

    field = MlpField(seed=0, amplitude=1.0)
    g = GridSpec((0, 0, 0), (1, 1, 1), R)
    res = contour(field, g)
    t0 = time.perf_counter()
    o = oracle.contour_oracle(field, (0, 0, 0), (1, 1, 1), R)  # numpy fp32 MlpField through the callback
    ow = time.perf_counter() - t0
    S = R + 1
    idx = np.arange(S ** 3)
    pts = np.stack([idx % S, (idx // S) % S, idx // (S * S)], 1) * (1.0 / R)
    gl = eval_labels(field, pts)
    agree = float(np.mean(gl == o["labels"]))
    cpu_mesh = TriangleMesh(o["vertices"], o["triangles"])
    h = 1.0 / R
    md2 = metric_md2(res.mesh, cpu_mesh, n=200_000)
    hdd = metric_hdd(res.mesh, cpu_mesh, n=200_000)
    print(f"[c3b] label agreement {agree:.6f} md2 {md2} hdd {hdd}", flush=True)
    return [{"case": f"c3b_mlp_{R}_bf16_gpu_vs_fp32_cpu", "R": R, "grid_label_agreement": agree,
             "grid_label_mismatches": int(np.sum(gl != o["labels"])), "n_grid": int(S ** 3),
             "md2": md2, "md2_over_h2": md2 / h / h if isinstance(md2, float) else None, "hdd": hdd,
             "hdd_over_h": hdd / h if isinstance(hdd, float) else None,
             "V_gpu": int(res.mesh.n_vertices), "V_cpu": int(len(o["vertices"])),
             "T_gpu": int(res.mesh.n_triangles), "T_cpu": int(len(o["triangles"])), "oracle_wall_s": ow}]


def case_c4(R=1024, slabs=(2, 4, 8)):
    from paper_2409_13418_b200.slab import contour_slabs_serial

    field, lo, hi = scenes.resolve(scenes.thin_shell(R), R)
    out = [one_case(f"c4_thin_shell_{R}", field, lo, hi, R)]
    single = contour(field, GridSpec(lo, hi, R))
    for n in slabs:
        mesh, _, _ = contour_slabs_serial(field, GridSpec(lo, hi, R), n)
        eq = mesh_equal(mesh, single.mesh)
        print(f"[c4] {n} slabs == single extraction: {eq}", flush=True)
        out.append({"case": f"c4_thin_shell_{R}_{n}_slabs_vs_single", "R": R, "bit_exact": all(eq.values()),
                    "compare": eq, "V": int(mesh.n_vertices), "T": int(mesh.n_triangles)})
    return out


def case_c5(n=64, R=256):
    from paper_2409_13418_b200.batch import contour_batch

    jobs = []
    for s in range(n):
        field, lo, hi = scenes.resolve(scenes.batch_shape(s), R)
        jobs.append((field, GridSpec(lo, hi, R)))
    t0 = time.perf_counter()
    results = contour_batch(jobs)
    gw = time.perf_counter() - t0
    rows, ok_all = [], True
    for s, ((field, g), r) in enumerate(zip(jobs, results)):
        t1 = time.perf_counter()
        o = oracle.contour_oracle(field, g.lo, g.hi, R)
        eq = {"vertices": bool(np.array_equal(r.mesh.vertices, o["vertices"])),
              "triangles": bool(np.array_equal(r.mesh.triangles, o["triangles"])),
              "raw_triangles": bool(np.array_equal(r.raw_mesh.triangles, o["raw_triangles"])),
              "provenance_ref": bool(np.array_equal(_prov(r.mesh.provenance_ref), _prov(o["ref"]))),
              "eval_counts": r.stats["eval_counts"] == o["eval_counts"]}
        ok = all(eq.values())
        ok_all &= ok
        rows.append({"shape": s, "bit_exact": ok, "V": int(r.mesh.n_vertices), "T": int(r.mesh.n_triangles),
                     "oracle_wall_s": time.perf_counter() - t1, **({} if ok else {"compare": eq})})
        print(f"[c5] shape {s}: bit-exact={ok} V={r.mesh.n_vertices}", flush=True)
    return [{"case": f"c5_batch{n}_{R}", "R": R, "bit_exact": ok_all, "gpu_batch_wall_s": gw, "shapes": rows}]


CASES = {"c1": case_c1, "c2": case_c2, "c3": case_c3, "c3b": case_c3b, "c4": case_c4, "c5": case_c5}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", default="c1,c2,c3,c3b,c4,c5")
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    import platform

    import threadpoolctl

    report = {"host": platform.node(), "cpu": platform.processor(),
              "blas": [{k: i.get(k) for k in ("internal_api", "version", "architecture")}
                       for i in threadpoolctl.threadpool_info()],
              "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime()), "results": []}
    for c in a.cases.split(","):
        report["results"] += CASES[c]()
        Path(a.out).parent.mkdir(parents=True, exist_ok=True)
        Path(a.out).write_text(json.dumps(report, indent=1, default=str))
    bad = [r["case"] for r in report["results"] if r.get("bit_exact") is False]
    print("NOT bit-exact:", bad if bad else "none")


if __name__ == "__main__":
    main()
