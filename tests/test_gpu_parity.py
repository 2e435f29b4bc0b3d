"""GPU parity: libodc (through its C-ABI) against the CPU oracle and the
reference's golden vectors, stage by stage.

Bit-exact, zero tolerance: labels, crossing edge/face/cell sets, v_in,
instance pairs, 1D t and positions, 2D positions/status, partitions and
cycles, normals, QEF positions and ranks (the device runs numpy.linalg.eigh's
LAPACK dsyevd bit for bit, csrc/odc_eigh3.cuh; the oracle calls numpy's own
dsyevd), split cases, raw and repaired mesh vertices and triangles,
provenance, eval counts.  The only tolerances are for raw values that come
from the device exp() (smoothed fields in continuous mode), written in the
tests that need them.
"""

import numpy as np
import pytest

import oracle
from golden_util import cases, field_of, load
from paper_2409_13418_b200 import ContourOptions, GridSpec, MlpField, SharedField, contour
from paper_2409_13418_b200.fields import is_mlp
from paper_2409_13418_b200.pipeline import stage_arrays

pytestmark = pytest.mark.gpu

STAGES = ["labels", "edge_key", "v_in", "face_key", "face_n_crossing", "cells", "instance_edges", "t1d", "pos1d",
          "pos2", "status", "part_cell", "part_index", "cyc_len", "cyc_edges", "cyc_insts", "normals", "qef_pos",
          "qef_rank", "split_cases"]


def gpu_run(field, lo, hi, R, options=None):
    res, ctx, st = contour(field, GridSpec(lo, hi, R), options, keep_intermediates=True, return_context=True)
    arrs = stage_arrays(ctx, STAGES)
    return res, arrs


def oracle_run(field, lo, hi, R, options=None):
    if is_mlp(field):
        shared = SharedField(field)
        try:
            return oracle.contour_oracle(field, lo, hi, R, options=options, continuous=True,
                                         raw_fn=lambda p, c: shared.eval_raw(p))
        finally:
            shared.close()
    return oracle.contour_oracle(field, lo, hi, R, options=options)


def _close(a, b, atol):
    a, b = np.asarray(a), np.asarray(b).reshape(np.shape(a))
    return a.shape == b.shape and (a.size == 0 or np.abs(a - b).max() <= atol)


def compare(res, arrs, o, exact_positions=True, tol=None):
    """Discrete outputs bit-exact; with ``tol`` (in units of h) continuous
    outputs are compared with that tolerance instead of bit-for-bit (used
    where raw values come from the device exp(), which is not glibc's)."""
    h = float(np.min(o["h"]))
    eq = (lambda a, b: _close(a, b, tol * h)) if tol is not None else (lambda a, b: np.array_equal(a, np.reshape(b, np.shape(a))))
    assert np.array_equal(arrs["labels"], o["labels"])
    for k in ("edge_key", "v_in", "face_key", "face_n_crossing", "cells"):
        assert np.array_equal(arrs[k], o[k]), k
    if len(o["edge_key"]) == 0:
        assert res.mesh.n_triangles == 0
        return
    assert np.array_equal(arrs["instance_edges"].reshape(-1, 2), o["instance_edges"])
    assert eq(arrs["t1d"], o["t1d"]) if tol is None else _close(arrs["t1d"], o["t1d"], tol)
    assert eq(arrs["pos1d"].reshape(-1, 3), o["pos1d"])
    assert eq(arrs["pos2"].reshape(-1, 2), o["pos2"])
    assert np.array_equal(arrs["status"], o["status"])
    assert np.array_equal(arrs["part_cell"], o["part_cell"])
    assert np.array_equal(arrs["part_index"], o["part_index"])
    assert np.array_equal(np.concatenate([[0], np.cumsum(arrs["cyc_len"])]), o["cyc_off"])
    assert np.array_equal(arrs["cyc_edges"], o["cyc_edges"])
    assert np.array_equal(arrs["cyc_insts"], o["cyc_insts"])
    assert eq(arrs["normals"].reshape(-1, 3), o["normals"]) if tol is None else _close(
        arrs["normals"].reshape(-1, 3), o["normals"], tol)
    qp = arrs["qef_pos"].reshape(-1, 3)
    assert np.abs(qp - o["qef_pos"]).max() <= 1e-4 * h
    if exact_positions and tol is None:
        assert np.array_equal(qp, o["qef_pos"])
        assert np.array_equal(res.mesh.vertices, o["vertices"])
        assert np.array_equal(res.raw_mesh.vertices, o["raw_vertices"])
    assert np.array_equal(arrs["qef_rank"], o["qef_rank"])
    assert np.array_equal(arrs["split_cases"], o["split_cases"])
    assert np.array_equal(res.raw_mesh.triangles, o["raw_triangles"])
    assert np.array_equal(res.mesh.triangles, o["triangles"])
    assert np.abs(res.mesh.vertices - o["vertices"]).max() <= 1e-4 * h
    assert np.array_equal(res.mesh.provenance_kind, o["kind"])
    assert np.array_equal(res.mesh.provenance_ref, o["ref"])
    assert res.stats["eval_counts"] == o["eval_counts"]


@pytest.mark.parametrize("tag", cases())
def test_gpu_vs_oracle_golden_cases(tag):
    field, lo, hi, R = field_of(tag)
    res, arrs = gpu_run(field, lo, hi, R)
    o = oracle_run(field, lo, hi, R)
    compare(res, arrs, o)


@pytest.mark.parametrize("tag", [t for t in cases() if not t.startswith("mlp")])
def test_gpu_vs_reference_golden(tag):
    """Against the reference's own recorded outputs (no oracle in the loop)."""
    field, lo, hi, R = field_of(tag)
    g = load(tag)
    res, arrs = gpu_run(field, lo, hi, R)
    assert np.array_equal(arrs["labels"], g["labels"])
    for k in ("edge_key", "v_in", "face_key", "face_n_crossing", "cells", "t1d", "status", "part_cell",
              "part_index", "cyc_edges", "cyc_insts"):
        assert np.array_equal(arrs[k].reshape(np.shape(g[k])), g[k]), k
    for k in ("pos1d", "pos2", "normals", "qef_pos"):
        assert np.array_equal(arrs[k].reshape(np.shape(g[k])), g[k]), k
    assert np.array_equal(arrs["qef_rank"], g["qef_rank"])
    assert np.array_equal(arrs["split_cases"], g["split_cases"])
    for a, k in ((res.raw_mesh.vertices, "raw_vertices"), (res.raw_mesh.triangles, "raw_triangles"),
                 (res.mesh.vertices, "vertices"), (res.mesh.triangles, "triangles"),
                 (res.mesh.provenance_kind, "kind"), (res.mesh.provenance_ref, "ref")):
        assert np.array_equal(a, g[k]), k
    assert res.stats["eval_counts"] == g["eval_counts"]


@pytest.mark.parametrize("opts", [
    ContourOptions(one_d="midpoint"),
    ContourOptions(one_d="linear-interp"),
    ContourOptions(split="mdc"),
    ContourOptions(repair=False),
])
def test_gpu_ablation_modes(opts):
    for tag in ("rotated_box_32", "smooth_sphere_32"):
        field, lo, hi, R = field_of(tag)
        res, arrs = gpu_run(field, lo, hi, R, opts)
        o = oracle_run(field, lo, hi, R, opts)
        # linear-interp on a smoothed field interpolates exp()-based raw values
        smooth_raw = opts.one_d == "linear-interp" and tag.startswith("smooth")
        compare(res, arrs, o, tol=1e-9 if smooth_raw else None)


def test_gpu_fd_gradient_normals():
    field, lo, hi, R = field_of("smooth_sphere_32")
    opts = ContourOptions(normals="fd-gradient", one_d="linear-interp", split="mdc")
    res, arrs = gpu_run(field, lo, hi, R, opts)
    o = oracle_run(field, lo, hi, R, opts)
    # raw values come from device exp(): tolerance on normals, exact topology
    assert np.array_equal(arrs["edge_key"], o["edge_key"])
    assert np.allclose(arrs["normals"].reshape(-1, 3), o["normals"], atol=1e-9)
    assert res.mesh.n_triangles == len(o["triangles"])


@pytest.mark.parametrize("name,R", [("torus", 128), ("csg_difference", 128), ("rotated_box", 96)])
def test_gpu_vs_oracle_medium(name, R):
    from paper_2409_13418_b200 import scenes

    field, lo, hi = scenes.resolve(scenes.SCENES[name], R)
    res, arrs = gpu_run(field, lo, hi, R)
    o = oracle_run(field, lo, hi, R)
    compare(res, arrs, o)


def test_gpu_mlp_shared_field_64():
    field = MlpField(seed=0, amplitude=4.0)
    res, arrs = gpu_run(field, (0, 0, 0), (1, 1, 1), 48)
    o = oracle_run(field, (0, 0, 0), (1, 1, 1), 48)
    compare(res, arrs, o)
    assert res.stats["repair_added_vertices"] == len(o["vertices"]) - len(o["raw_vertices"])


@pytest.mark.parametrize("s1,s2", [((2, 5, 0.8), (1, 6, 0.7)), ((6, 3, 0.9), (5, 4, 0.6)), ((1, 8, 0.8), (2, 7, 0.7))])
def test_gpu_mlp_search_budgets(s1, s2):
    """Lock-step 2D search on the MLP evaluator with other line budgets: the
    compacted linear-scan steps (only rays still scanning are evaluated) must
    leave every stage identical to the oracle, which evaluates every ray."""
    from paper_2409_13418_b200.pipeline import LineBudget, SearchBudget

    opts = ContourOptions(budget=SearchBudget(iters_1d=12, step1=LineBudget(*s1), step2=LineBudget(*s2)))
    field = MlpField(seed=1, amplitude=3.0)
    res, arrs = gpu_run(field, (0, 0, 0), (1, 1, 1), 40, opts)
    o = oracle_run(field, (0, 0, 0), (1, 1, 1), 40, opts)
    compare(res, arrs, o)


@pytest.mark.parametrize("opts", [dict(one_d="midpoint"), dict(one_d="linear-interp"),
                                  dict(normals="fd-gradient"), dict(split="mdc", repair=False),
                                  dict(one_d="linear-interp", normals="fd-gradient", split="mdc")])
def test_gpu_mlp_option_variants(opts):
    """The MLP field (continuous) under the other pipeline modes: linear-interp
    1D points from the raw grid values (lock-step endpoint evaluations) and
    fd-gradient normals (6 raw evaluations per edge, pipeline.py:126-151) run
    through the CTA-pair evaluator with raw output; every stage equals the
    shared-field oracle or both raise the same error."""
    options = ContourOptions(**opts)
    field = MlpField(seed=2, amplitude=3.0)
    gpu_err = ref_err = None
    try:
        res, arrs = gpu_run(field, (0, 0, 0), (1, 1, 1), 36, options)
    except Exception as e:  # noqa: BLE001
        gpu_err = e
    try:
        o = oracle_run(field, (0, 0, 0), (1, 1, 1), 36, options)
    except Exception as e:  # noqa: BLE001
        ref_err = e
    if gpu_err or ref_err:
        assert type(gpu_err) is type(ref_err) and str(gpu_err) == str(ref_err), (gpu_err, ref_err)
        return
    compare(res, arrs, o)


@pytest.mark.parametrize("s1,s2", [((0, 8, 0.8), (3, 12, 0.7)), ((4, 11, 0.8), (0, 7, 0.7))])
def test_gpu_zero_linear_budget_raises(s1, s2):
    """n_linear == 0 makes the reference's bracket [-inf, nan] (a division by
    zero, search.py:124-125), so its next query is non-finite and eval_labels
    raises ValueError (fields.py:42-45); the device path raises the same."""
    from paper_2409_13418_b200 import SphereField
    from paper_2409_13418_b200.pipeline import LineBudget, SearchBudget

    opts = ContourOptions(budget=SearchBudget(step1=LineBudget(*s1), step2=LineBudget(*s2)))
    for field in (SphereField((0.5, 0.5, 0.5), 0.3), MlpField(seed=0)):
        with pytest.raises(ValueError, match="non-finite query point"):
            contour(field, GridSpec((0, 0, 0), (1, 1, 1), 16), opts)


def test_gpu_errors():
    from paper_2409_13418_b200 import ConfigurationError, SphereField

    f = SphereField((0.5, 0.5, 0.5), 0.3)
    with pytest.raises(ConfigurationError):
        contour(f, GridSpec((0, 0, 0), (1, 1, 1), 8), ContourOptions(one_d="bogus"))
    with pytest.raises(ConfigurationError):  # pipeline.py:128-131
        contour(f, GridSpec((0, 0, 0), (1, 1, 1), 8), ContourOptions(normals="fd-gradient"))
    with pytest.raises(ValueError):
        GridSpec((0, 0, 0), (1, 1, 1), 1)
    empty = contour(SphereField((5, 5, 5), 0.1), GridSpec((0, 0, 0), (1, 1, 1), 8))
    assert empty.mesh.n_triangles == 0 and empty.stats["n_2d_points"] == 0


def test_gpu_determinism():
    from paper_2409_13418_b200 import scenes

    field, lo, hi = scenes.resolve(scenes.SCENES["csg_union"], 128)
    a = contour(field, GridSpec(lo, hi, 128))
    b = contour(field, GridSpec(lo, hi, 128))
    assert np.array_equal(a.mesh.vertices, b.mesh.vertices)
    assert np.array_equal(a.mesh.triangles, b.mesh.triangles)


def test_gpu_mlp_determinism_repeated():
    """The CTA-pair evaluator hands out pairs dynamically (a device counter)
    and compacts the linear scans with atomics: results must not depend on
    which cluster took which pair or on slot order.  Repeated runs, and runs
    on a context whose counters have advanced, give identical meshes."""
    field = MlpField(seed=2, amplitude=3.0)
    g = GridSpec((0, 0, 0), (1, 1, 1), 96)
    ref = contour(field, g)
    for _ in range(4):
        r = contour(field, g)
        assert np.array_equal(r.mesh.vertices, ref.mesh.vertices)
        assert np.array_equal(r.mesh.triangles, ref.mesh.triangles)
        assert np.array_equal(r.raw_mesh.triangles, ref.raw_mesh.triangles)


def test_gpu_copy_mesh_pair_matches_single_copies():
    """odc_copy_mesh_pair (one pipelined transfer of the repaired mesh and the
    raw mesh's triangles) returns exactly what two odc_copy_mesh calls do."""
    from paper_2409_13418_b200 import _lib
    from paper_2409_13418_b200.pipeline import _copy_mesh

    field = MlpField(seed=0, amplitude=4.0)
    res, ctx, st = contour(field, GridSpec((0, 0, 0), (1, 1, 1), 48), return_context=True)
    assert st.repair_added_vertices > 0  # the raw mesh differs from the repaired one
    m = _copy_mesh(ctx, 0, st, True)
    raw = _copy_mesh(ctx, 1, st, True)
    for a, b in ((res.mesh.vertices, m.vertices), (res.mesh.triangles, m.triangles),
                 (res.mesh.provenance_kind, m.provenance_kind), (res.mesh.provenance_ref, m.provenance_ref),
                 (res.raw_mesh.triangles, raw.triangles), (res.raw_mesh.vertices, raw.vertices)):
        assert np.array_equal(a, b)
    _lib.check(0)


def _open_boundary_case(i):
    """Case i of a seeded stream of shapes that leave the unit box (the
    stream scripts/probe_unused_partitions.py searched): 4 (sphere, 20^3), 6 (plane,
    16^3) and 7 (torus, 16^3) keep partition vertices no triangle uses."""
    from paper_2409_13418_b200 import BoxField, PlaneField, SphereField, TorusField

    rng = np.random.default_rng(0)
    for j in range(i + 1):
        k = j % 4
        if k == 0:
            f = SphereField(tuple(rng.uniform(-0.2, 1.2, 3)), float(rng.uniform(0.2, 0.9)))
        elif k == 1:
            f = BoxField(tuple(rng.uniform(-0.2, 1.2, 3)), tuple(rng.uniform(0.1, 0.8, 3)))
        elif k == 2:
            f = PlaneField(tuple(rng.uniform(0, 1, 3)), tuple(rng.normal(size=3)))
        else:
            f = TorusField(tuple(rng.uniform(0, 1, 3)), float(rng.uniform(0.2, 0.5)), float(rng.uniform(0.05, 0.2)))
        R = int(rng.choice([9, 12, 16, 20]))
    return f, R


@pytest.mark.parametrize("i", [4, 6, 7])
def test_gpu_open_boundary_drops_unused_partitions(i):
    """Open boundaries: some partition vertices are referenced by no
    triangle, and polygonize.py:204-214 drops them before the repair; the
    device path learns that from the first repair pass's readback and
    restarts the repair on the compacted mesh.  Mesh, raw mesh and
    provenance equal the oracle's."""
    field, R = _open_boundary_case(i)
    res = contour(field, GridSpec((0, 0, 0), (1, 1, 1), R))
    o = oracle.contour_oracle(field, (0, 0, 0), (1, 1, 1), R)
    assert int((res.raw_mesh.provenance_kind == 0).sum()) < res.stats["n_partitions"]  # the path under test
    assert np.array_equal(res.mesh.triangles, o["triangles"])
    assert np.array_equal(res.mesh.vertices, o["vertices"])
    assert np.array_equal(res.raw_mesh.triangles, o["raw_triangles"])
    assert np.array_equal(res.raw_mesh.vertices, o["raw_vertices"])


@pytest.mark.parametrize("R", [2, 3, 5])
def test_gpu_tiny_grids_match_oracle(R):
    """The smallest grids (R = 2: one interior vertex, every cell on the
    boundary) against the oracle, mesh and statistics included."""
    from paper_2409_13418_b200 import SphereField

    field = SphereField((0.45, 0.52, 0.5), 0.3)
    res = contour(field, GridSpec((0, 0, 0), (1, 1, 1), R))
    o = oracle.contour_oracle(field, (0, 0, 0), (1, 1, 1), R)
    assert np.array_equal(res.mesh.triangles, o["triangles"])
    assert np.array_equal(res.mesh.vertices, o["vertices"])
    assert res.stats["boundary_inside_vertices"] == o["boundary_inside"]


def test_gpu_all_inside_and_resolution_limit():
    """A field inside everywhere: no crossing, an empty mesh and the
    boundary warning (pipeline.py:174-179); a resolution past the 32-bit
    vertex-index space is refused with ValueError, not truncated."""
    from paper_2409_13418_b200 import SphereField

    full = contour(SphereField((0.5, 0.5, 0.5), 5.0), GridSpec((0, 0, 0), (1, 1, 1), 16))
    assert full.mesh.n_triangles == 0 and full.stats["boundary_inside_vertices"] > 0
    assert any("open boundary" in w for w in full.stats["warnings"])
    with pytest.raises(ValueError, match="1290"):
        contour(SphereField((0.5, 0.5, 0.5), 0.3), GridSpec((0, 0, 0), (1, 1, 1), 1300))


def test_gpu_output_arrays_are_independent():
    """The mesh arrays come from recycled page-locked blocks: results of
    successive calls must not alias (a block is reused only after every
    array of the previous result is gone), stay valid after later
    extractions, and be ordinary writable numpy arrays of the reference's
    dtypes."""
    import gc

    from paper_2409_13418_b200 import SphereField, TorusField

    g = GridSpec((0, 0, 0), (1, 1, 1), 48)
    a = contour(SphereField((0.5, 0.5, 0.5), 0.3), g)
    va, ta = a.mesh.vertices.copy(), a.mesh.triangles.copy()
    b = contour(TorusField((0.5, 0.5, 0.5), 0.25, 0.08), g)
    assert not np.shares_memory(a.mesh.vertices, b.mesh.vertices)
    assert np.array_equal(a.mesh.vertices, va) and np.array_equal(a.mesh.triangles, ta)
    assert a.mesh.vertices.dtype == np.float64 and a.mesh.triangles.dtype == np.int64
    assert a.mesh.provenance_kind.dtype == np.int64 and a.mesh.provenance_ref.dtype == np.int64
    a.mesh.vertices[0, 0] += 1.0  # writable
    del b
    gc.collect()
    c = contour(SphereField((0.5, 0.5, 0.5), 0.3), g)  # may reuse b's block, never a's
    assert not np.shares_memory(a.mesh.vertices, c.mesh.vertices)
    assert np.array_equal(c.mesh.vertices, va) and np.array_equal(c.mesh.triangles, ta)
