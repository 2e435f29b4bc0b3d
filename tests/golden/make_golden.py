"""Generate golden vectors from the UNMODIFIED reference (occmesh).

Run in the build container only (needs /root/reference):

    python tests/golden/make_golden.py

Every fixture is the reference's own output on the named input: the
intermediate arrays of occmesh.pipeline.contour's stages (grid.py,
search.py, dualize.py, polygonize.py) plus the final mesh, stats and eval
counts.  The reference is driven stage by stage exactly as
pipeline.contour (pipeline.py:154-240) drives it, and the final mesh is
checked to be identical to a plain ``contour()`` call.

The fixtures pin the C oracle (tests/test_oracle_golden.py); the GPU tests
compare the device path with the oracle.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parent.parent
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(REPO))

import occmesh  # noqa: E402
from occmesh import GridSpec  # noqa: E402
from occmesh import dualize as D  # noqa: E402
from occmesh import grid as G  # noqa: E402
from occmesh import pipeline as PL  # noqa: E402
from occmesh import polygonize as PG  # noqa: E402
from occmesh import search as SR  # noqa: E402
from occmesh.fields import field_from_dict  # noqa: E402

from paper_2409_13418_b200 import scenes as SC  # noqa: E402
from paper_2409_13418_b200.fields import MlpField  # noqa: E402


def ref_mlp_field(mf):
    """The NEW MlpField as a reference-side OccupancyField (numpy fp32)."""
    import oracle

    class RefMlp(occmesh.OccupancyField):
        continuous = True

        def eval_raw(self, pts):
            return oracle.mlp_raw_numpy(mf, pts)

    return RefMlp()


def run_reference(field, grid):
    opts = PL.ContourOptions()
    cnt = PL.EvalCounter(field)
    vol = G.sample_labels(field, grid, cnt)
    act = G.extract_active(vol)
    out = dict(labels_packed=np.packbits(vol.labels), n_labels=len(vol.labels),
               edge_key=act.edge_key, v_in=act.v_in, face_key=act.face_key,
               face_n_crossing=act.face_n_crossing, cells=act.cells)
    if act.n_edges == 0:
        return out
    p1 = PL._edge_points(vol, act, opts, cnt)
    pair = D.face_pairings(act, lambda p, c: cnt.labels(p, c))
    parts = D.partition_cells(act, pair)
    batch = D.build_face_batch(act, pair, p1)
    p2 = SR.find_2d_points(batch, lambda p, c: cnt.labels(p, c), opts.budget)
    pr, er, pe, nrm, nfb = D.build_plane_samples(act, parts, p1, p2.position3)
    pos, rank, resid = D.place_3d_points(act, parts, pr, pe, nrm)
    poly = PG.build_mesh(act, parts, pos, p1)
    mesh = PG.repair_nonmanifold(poly.mesh)
    lens = np.array([len(c) for c in parts.cycles_edges], dtype=np.int64)
    out.update(
        instance_edges=pair.instance_edges, n_probes=pair.n_probes,
        t1d=p1.t, pos1d=p1.position, pos2=p2.position2, status=p2.status,
        part_cell=parts.cell_ids, part_index=parts.partition_index,
        cyc_off=np.concatenate([[0], np.cumsum(lens)]),
        cyc_edges=np.concatenate([np.asarray(c, dtype=np.int64) for c in parts.cycles_edges]),
        cyc_insts=np.concatenate([np.asarray(c, dtype=np.int64) for c in parts.cycles_instances]),
        normals=nrm, n_fallback=nfb, qef_pos=pos, qef_rank=rank, qef_resid=resid,
        split_cases=poly.split_cases, skipped=poly.skipped_boundary_edges,
        raw_vertices=poly.mesh.vertices, raw_triangles=poly.mesh.triangles,
        raw_kind=poly.mesh.provenance_kind, raw_ref=poly.mesh.provenance_ref,
        vertices=mesh.vertices, triangles=mesh.triangles,
        kind=mesh.provenance_kind, ref=mesh.provenance_ref,
        eval_counts=json.dumps(cnt.snapshot()),
    )
    # the staged run must equal a plain contour() call
    full = occmesh.contour(field, grid)
    assert np.array_equal(full.mesh.triangles, mesh.triangles)
    assert np.array_equal(full.mesh.vertices, mesh.vertices)
    stats = {k: v for k, v in full.stats.items() if k not in ("options", "wall_time_s")}
    out["stats"] = json.dumps(stats, default=str)
    return out


def cases():
    for name in ("sphere", "torus", "rotated_box", "csg_union", "csg_difference", "smooth_sphere"):
        for R in (32, 64):
            yield f"{name}_{R}", SC.SCENES[name], R
    yield "thin_shell_64", SC.SCENES["thin_shell"], 64
    yield "mlp_amp1_32", {"field": {"type": "mlp", "seed": 0, "amplitude": 1.0}}, 32
    yield "mlp_amp4_32", {"field": {"type": "mlp", "seed": 0, "amplitude": 4.0}}, 32
    yield "thin_wall_18", SC.SCENES["thin_wall"], 18
    yield "thin_wall_b_29", SC.SCENES["thin_wall_b"], 29


def main():
    """``python make_golden.py [tag ...]``: regenerate the named cases only
    (default: all), keeping the other fixtures and index entries."""
    HERE.mkdir(exist_ok=True)
    only = set(sys.argv[1:])
    index = json.loads((HERE / "index.json").read_text()) if only else {}
    for tag, scene, R in cases():
        if only and tag not in only:
            continue
        doc = scene
        lo = tuple(doc.get("domain", {}).get("lo", (0, 0, 0)))
        hi = tuple(doc.get("domain", {}).get("hi", (1, 1, 1)))
        grid = GridSpec(lo, hi, R)
        if doc["field"]["type"] == "mlp":
            mf = MlpField(**{k: v for k, v in doc["field"].items() if k != "type"})
            field = ref_mlp_field(mf)
        else:
            field = field_from_dict(doc["field"])
            if doc.get("smooth_k") is not None:
                k = doc["smooth_k"]
                k = 2.0 / float(np.min(grid.cell_size)) if k == "auto" else k
                field = occmesh.SmoothedOccupancy(field, k)
        out = run_reference(field, grid)
        np.savez_compressed(HERE / f"{tag}.npz", **out)
        index[tag] = {"scene": scene, "R": R}
        print(tag, "V", len(out.get("vertices", [])), "T", len(out.get("triangles", [])))
    # known-answer tests from SPEC.md:118, :125-126
    kat = {}
    g2 = GridSpec((0, 0, 0), (1, 1, 1), 2)
    vol = G.sample_labels(occmesh.SphereField((0.5, 0.5, 0.5), 0.3), g2)
    kat["sphere_R2_labels"] = vol.labels.tolist()
    g4 = GridSpec((0, 0, 0), (1, 1, 1), 4)
    act = G.extract_active(G.sample_labels(occmesh.SphereField((0.5, 0.5, 0.5), 0.1), g4))
    kat["single_vertex_R4"] = [int(act.n_edges), int(len(act.face_key)), int(len(act.cells))]
    act = G.extract_active(G.sample_labels(occmesh.PlaneField((0, 0, 0.3), (0, 0, 1)), g4))
    kat["halfspace_R4_edges"] = int(act.n_edges)
    index["kat"] = kat
    (HERE / "index.json").write_text(json.dumps(index, indent=1, default=str))


if __name__ == "__main__":
    main()
