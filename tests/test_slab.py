"""z-slab decomposition.

CPU: the host-side exchange (count all-gather, global id offsets, halo id
mapping, point-to-point gather, assembly in rank order) runs over real gloo
collectives with world_size 2; each rank's contribution is derived from the
oracle's global result exactly as a GPU rank produces it (owned partitions,
halo partitions in local ids, owned fans and triangles).  The assembled mesh
must equal the oracle's mesh.

GPU: every slab of an N-way split extracted by libodc, stitched and
finished, must equal the single-GPU extraction bit for bit.
"""

import os
import socket

import numpy as np
import pytest

import oracle
from paper_2409_13418_b200 import scenes
from paper_2409_13418_b200.slab import assemble, global_offsets, globalize_ids, slab_ranges, SlabPiece, stitch


def test_slab_ranges():
    assert slab_ranges(10, 3) == [(0, 3), (3, 6), (6, 10)]
    assert slab_ranges(512, 8)[-1] == (448, 512)
    with pytest.raises(ValueError):
        slab_ranges(2, 3)


def test_offsets_and_ids():
    counts = [[5, 1, 12], [7, 2, 16], [3, 0, 6]]
    assert global_offsets(counts, 0) == (0, 15, 0)
    assert global_offsets(counts, 1) == (5, 15, 1)
    assert global_offsets(counts, 2) == (12, 15, 3)
    # rank 1 with 2 halo partitions, window of 9 partitions (2 halo + 7 owned)
    ids = globalize_ids([0, 1, 2, 8, 9, 10], 2, 9, 5, 15, 1)
    assert ids.tolist() == [3, 4, 5, 11, 16, 17]


def oracle_pieces(o, R, world):
    """Per-rank contributions, derived from the oracle's global result."""
    import torch

    S = R + 1
    ek = o["edge_key"]
    vid, ax = ek // 3, ek % 3
    c = np.stack([vid % S, (vid // S) % S, vid // (S * S)], axis=1)
    b_ax, c_ax = (ax + 1) % 3, (ax + 2) % 3
    cb, cc = c[np.arange(len(ek)), b_ax], c[np.arange(len(ek)), c_ax]
    interior = (cb >= 1) & (cb <= R - 1) & (cc >= 1) & (cc <= R - 1)
    cases = np.zeros(len(ek), np.int64)
    cases[interior] = o["split_cases"]
    ntri = np.where(cases == 3, 4, np.where(cases > 0, 2, 0))
    tri_off = np.concatenate([[0], np.cumsum(ntri)])
    fan_rank = np.concatenate([[0], np.cumsum(cases == 3)])
    P = len(o["part_cell"])
    pz = o["part_cell"] // (R * R)
    pieces = []
    for k, (c0, c1) in enumerate(slab_ranges(R, world)):
        last = k == world - 1
        p_lo, p_hi = np.searchsorted(pz, c0), np.searchsorted(pz, c1)
        h_lo = np.searchsorted(pz, c0 - 1) if c0 > 0 else p_lo
        ez = c[:, 2]
        e_sel = np.nonzero((ez >= c0) & ((ez < c1) | (last & (ez <= R))))[0]
        e_lo, e_hi = (e_sel[0], e_sel[-1] + 1) if len(e_sel) else (0, 0)
        t_lo, t_hi = tri_off[e_lo], tri_off[e_hi]
        f_lo, f_hi = fan_rank[e_lo], fan_rank[e_hi]
        n_halo, n_window = p_lo - h_lo, p_hi - h_lo
        tris = o["raw_triangles"][t_lo:t_hi]
        loc = np.where(tris < P, tris - h_lo, n_window + (tris - P - f_lo))
        assert ((tris < P) & ((tris < h_lo) | (tris >= p_hi))).sum() == 0
        fan_edges = ek[e_lo:e_hi][cases[e_lo:e_hi] == 3]
        pieces.append(SlabPiece(
            n_halo=int(n_halo), n_window=int(n_window),
            part_vertices=torch.as_tensor(o["raw_vertices"][p_lo:p_hi]),
            fan_vertices=torch.as_tensor(o["raw_vertices"][P + f_lo:P + f_hi]),
            triangles=torch.as_tensor(loc.astype(np.int32)),
            part_cell=torch.as_tensor(o["part_cell"][p_lo:p_hi]),
            part_index=torch.as_tensor(o["part_index"][p_lo:p_hi]),
            fan_edge=torch.as_tensor(fan_edges),
            stats=np.zeros(34, np.int64),
            c0=c0, c1=c1,
        ))
    return pieces


def _worker(rank, world, port, R, result_path):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        field, lo, hi = scenes.resolve(scenes.SCENES["torus"], R)
        o = oracle.contour_oracle(field, lo, hi, R)
        piece = oracle_pieces(o, R, world)[rank]
        out = stitch(piece, rank, world, dist, torch.device("cpu"), R=R)
        if rank == 0:
            verts, tris, kind, ref, P_tot, rows = out
            ok = (np.array_equal(verts.numpy(), o["raw_vertices"]) and np.array_equal(tris.numpy(), o["raw_triangles"])
                  and np.array_equal(kind.numpy(), o["raw_kind"]) and np.array_equal(ref.numpy(), o["raw_ref"])
                  and P_tot == len(o["part_cell"]))
            np.save(result_path, np.array([int(ok)]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_slab_stitch_matches_oracle(tmp_path, world):
    import torch.multiprocessing as mp

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    out = tmp_path / "ok.npy"
    mp.spawn(_worker, args=(world, port, 24, str(out)), nprocs=world, join=True)
    assert np.load(out)[0] == 1


@pytest.mark.gpu
@pytest.mark.parametrize("name,R,n", [("sphere", 64, 2), ("torus", 96, 4), ("rotated_box", 64, 3),
                                      ("csg_union", 64, 8), ("thin_shell", 64, 4)])
def test_gpu_slabs_equal_single_extraction(name, R, n):
    from paper_2409_13418_b200 import GridSpec, contour
    from paper_2409_13418_b200.slab import contour_slabs_serial

    sc = scenes.thin_shell(R) if name == "thin_shell" else scenes.SCENES[name]
    field, lo, hi = scenes.resolve(sc, R)
    g = GridSpec(lo, hi, R)
    ref = contour(field, g)
    mesh, pieces, rows = contour_slabs_serial(field, g, n)
    assert np.array_equal(mesh.vertices, ref.mesh.vertices)
    assert np.array_equal(mesh.triangles, ref.mesh.triangles)
    assert np.array_equal(mesh.provenance_kind, ref.mesh.provenance_kind)
    assert np.array_equal(mesh.provenance_ref, ref.mesh.provenance_ref)
    # owned counts add up to the single-extraction stats
    assert rows[:, 2].sum() == ref.stats["n_crossing_edges"]
    assert rows[:, 3].sum() == ref.stats["n_crossing_cells"]
    assert rows[:, 6].sum() == ref.stats["n_partitions"]


@pytest.mark.gpu
def test_gpu_slabs_mlp_repair():
    from paper_2409_13418_b200 import GridSpec, MlpField, contour
    from paper_2409_13418_b200.slab import contour_slabs_serial

    field = MlpField(seed=0, amplitude=4.0)
    g = GridSpec((0, 0, 0), (1, 1, 1), 48)
    ref = contour(field, g)
    mesh, pieces, rows = contour_slabs_serial(field, g, 3)
    assert ref.stats["repair_added_vertices"] > 0
    assert np.array_equal(mesh.triangles, ref.mesh.triangles)
    assert np.array_equal(mesh.vertices, ref.mesh.vertices)


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 4, 7])
def test_gpu_balanced_slabs_equal_single_extraction(world):
    """Work-balanced slab bounds (a coarse device probe of the crossing
    density per z) are a valid partition, give thinner slabs where the
    surface is, and reproduce the single-extraction mesh exactly."""
    from paper_2409_13418_b200 import GridSpec, MlpField, contour
    from paper_2409_13418_b200.slab import balanced_slab_ranges, contour_slabs_serial

    field = MlpField(seed=0, amplitude=2.0)
    g = GridSpec((0, 0, 0), (1, 1, 1), 64)
    ranges = balanced_slab_ranges(field, g, world)
    assert ranges[0][0] == 0 and ranges[-1][1] == 64
    assert all(a < b for a, b in ranges) and all(ranges[k][1] == ranges[k + 1][0] for k in range(world - 1))
    assert ranges == balanced_slab_ranges(field, g, world)  # deterministic: every rank agrees
    if world == 4:  # the sphere-like surface sits in the middle: the middle slabs are thinner
        widths = [b - a for a, b in ranges]
        assert widths[0] > widths[1] and widths[3] > widths[2]
    ref = contour(field, g)
    mesh, pieces, rows = contour_slabs_serial(field, g, world, ranges=ranges)
    assert np.array_equal(mesh.triangles, ref.mesh.triangles)
    assert np.array_equal(mesh.vertices, ref.mesh.vertices)


def test_check_ranges_rejects_gaps_and_overlaps():
    from paper_2409_13418_b200.slab import check_ranges

    def rows(rs):
        return np.array([[0, 0, 0, a, b] for a, b in rs])

    check_ranges(rows([(0, 3), (3, 8)]), 8)
    for bad in ([(0, 3), (4, 8)], [(0, 4), (3, 8)], [(1, 4), (4, 8)], [(0, 4), (4, 7)], [(0, 0), (0, 8)]):
        with pytest.raises(RuntimeError, match="do not tile"):
            check_ranges(rows(bad), 8)


@pytest.mark.gpu
def test_gpu_slab_globalize_device_equals_host():
    """k_globalize_tris (odc_slab_globalize, the ids the N-GPU path writes on
    the device) equals the host restatement globalize_ids for every slab."""
    import torch

    from paper_2409_13418_b200 import GridSpec, MlpField
    from paper_2409_13418_b200.pipeline import ContourOptions
    from paper_2409_13418_b200.slab import extract_piece, globalize

    field = MlpField(seed=0, amplitude=3.0)
    g = GridSpec((0, 0, 0), (1, 1, 1), 48)
    for c0, c1 in slab_ranges(48, 4):
        piece, _ = extract_piece(field, g, ContourOptions(), c0, c1)
        for part_base, P_tot, fan_base in ((1000, 50000, 7), (piece.n_halo, piece.n_window + 3, 0)):
            dev = globalize(piece, part_base, P_tot, fan_base, torch.device("cuda", 0)).cpu().numpy()
            host = globalize_ids(piece.triangles.cpu().numpy(), piece.n_halo, piece.n_window, part_base, P_tot,
                                 fan_base)
            assert np.array_equal(dev, host.astype(np.int32))


def _slab_worker(rank, world, port, backend, result_path, scene="mlp", distributed=True):
    import torch.distributed as dist

    from paper_2409_13418_b200 import GridSpec, MlpField, contour, scenes
    from paper_2409_13418_b200.slab import contour_slab

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dev = rank if backend == "nccl" else 0
    dist.init_process_group(backend, rank=rank, world_size=world)
    try:
        if scene == "mlp":
            field = MlpField(seed=0, amplitude=3.0)
            g = GridSpec((0, 0, 0), (1, 1, 1), 56)
        else:
            R = 72
            field, lo, hi = scenes.resolve(scenes.thin_shell(R) if scene == "thin_shell" else scenes.SCENES[scene], R)
            g = GridSpec(lo, hi, R)
        res = contour_slab(field, g, rank=rank, world=world, dist=dist, device=dev, distributed=distributed)
        if rank == 0:
            ref = contour(field, g, device=dev)
            ok = all(np.array_equal(a, b) for a, b in (
                (res.mesh.vertices, ref.mesh.vertices), (res.mesh.triangles, ref.mesh.triangles),
                (res.mesh.provenance_kind, ref.mesh.provenance_kind),
                (res.mesh.provenance_ref, ref.mesh.provenance_ref),
                (res.raw_mesh.triangles, ref.raw_mesh.triangles)))
            ok = ok and res.stats["eval_counts"] == ref.stats["eval_counts"]
            ok = ok and res.stats["repair_added_vertices"] == ref.stats["repair_added_vertices"]
            for k in ("n_crossing_edges", "n_crossing_cells", "n_partitions", "point2d_status_counts",
                      "qef_rank_counts", "split_case_counts", "skipped_boundary_edges"):
                ok = ok and res.stats.get(k) == ref.stats.get(k)
            np.save(result_path, np.array([int(ok), int(bool(res.stats.get("distributed_finish")))]))
        else:
            assert res is None
    finally:
        dist.destroy_process_group()


def _spawn(world, backend, tmp_path, scene="mlp", distributed=True):
    import torch.multiprocessing as mp

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    out = tmp_path / "ok.npy"
    mp.spawn(_slab_worker, args=(world, port, backend, str(out), scene, distributed), nprocs=world, join=True)
    r = np.load(out)
    assert r[0] == 1
    return bool(r[1])


@pytest.mark.gpu
@pytest.mark.parametrize("world,backend", [(1, "nccl"), (2, "gloo"), (3, "gloo")])
def test_gpu_contour_slab_processes(world, backend, tmp_path):
    """The real multi-process path (contour_slab: balanced bounds on every
    rank, device extraction, count all-gather, device id globalization, one
    grouped P2P gather, odc_mesh_finish on rank 0) equals contour().  NCCL
    with one rank per GPU; with more ranks than GPUs the ranks share GPU 0
    and the exchange goes over gloo with host staging (each rank's kernels
    run independently; only the host-side collectives synchronise them)."""
    _spawn(world, backend, tmp_path)


@pytest.mark.gpu
@pytest.mark.parametrize("scene,world", [("thin_shell", 2), ("thin_shell", 4), ("torus", 3), ("csg_union", 2)])
def test_gpu_contour_slab_distributed_finish(scene, world, tmp_path):
    """Closed surfaces: every fan is a disc, so each rank finishes its own
    piece (seam triangles one rank down, local unused-vertex removal) and
    the gathered mesh equals contour() bit for bit."""
    assert _spawn(world, "gloo", tmp_path, scene=scene) is True


@pytest.mark.gpu
def test_gpu_contour_slab_central_finish_when_repair_needed(tmp_path):
    """The MLP surface has non-manifold fans: the ranks detect it and fall
    back to the central finish on rank 0, which repairs."""
    assert _spawn(2, "gloo", tmp_path, scene="mlp") is False
    assert _spawn(2, "gloo", tmp_path, scene="thin_shell", distributed=False) is False


@pytest.mark.gpu
def test_gpu_contour_slab_two_gpus_nccl(tmp_path):
    import torch

    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    _spawn(2, "nccl", tmp_path)


@pytest.mark.gpu
def test_gpu_surface_probe_counts_thin_walls():
    """odc_surface_probe: the undecided boxes of the interval bound find a
    wall 2.5 cells thick that a 17x17 label probe misses; the per-layer
    estimate is zero away from the shell and every box layer the shell
    spans has work; MLP fields (no interval bound) are rejected."""
    import ctypes

    from paper_2409_13418_b200 import GridSpec, MlpField, _lib
    from paper_2409_13418_b200.pipeline import DeviceField
    from paper_2409_13418_b200.slab import surface_layer_crossings

    R = 256
    field, lo, hi = scenes.resolve(scenes.thin_shell(R), R)
    g = GridSpec(lo, hi, R)
    ctx = _lib.context(0)
    with DeviceField(ctx, field) as df:
        assert df.analytic
        k = surface_layer_crossings(g, df)
    assert k.shape == (R,) and (k >= 0).all()
    z = np.nonzero(k)[0]
    # the rotated shell spans a z-range inside the domain, with empty layers on both sides
    assert 0 < z[0] and z[-1] < R - 1 and (k[z[0]:z[-1] + 1] > 0).all()
    # the estimate is within a small factor of the true crossing count
    from paper_2409_13418_b200 import contour
    n_true = contour(field, g).stats["n_crossing_edges"]
    assert 0.3 < k.sum() / n_true < 3.0, (k.sum(), n_true)
    with DeviceField(ctx, MlpField(seed=0)) as dm:
        counts = np.zeros(4, dtype=np.int64)
        l3 = (ctypes.c_double * 3)(0, 0, 0)
        h3 = (ctypes.c_double * 3)(1, 1, 1)
        assert _lib.load().odc_surface_probe(ctx.handle, dm.handle, l3, h3, 16, 4, counts.ctypes.data) == _lib.ODC_E_ARG


@pytest.mark.gpu
@pytest.mark.parametrize("world", [3, 8])
def test_gpu_balanced_analytic_slabs_equal_single_extraction(world):
    """Analytic balance (surface probe) on the thin shell: a valid partition,
    deterministic, and the serial slab mesh equals the single extraction."""
    from paper_2409_13418_b200 import GridSpec, contour
    from paper_2409_13418_b200.slab import balanced_slab_ranges, contour_slabs_serial

    R = 96
    field, lo, hi = scenes.resolve(scenes.thin_shell(R), R)
    g = GridSpec(lo, hi, R)
    ranges = balanced_slab_ranges(field, g, world)
    assert ranges[0][0] == 0 and ranges[-1][1] == R
    assert all(a < b for a, b in ranges) and all(ranges[k][1] == ranges[k + 1][0] for k in range(world - 1))
    assert ranges == balanced_slab_ranges(field, g, world)
    ref = contour(field, g)
    mesh, _, _ = contour_slabs_serial(field, g, world, ranges=ranges)
    assert np.array_equal(mesh.triangles, ref.mesh.triangles)
    assert np.array_equal(mesh.vertices, ref.mesh.vertices)


@pytest.mark.gpu
def test_gpu_slab_seam_counts():
    """The seam (triangles with a halo corner, counted during the slab
    extraction) equals the host count from the slab's own triangles, and a
    slab without surface on the same context reports none."""
    import ctypes

    from paper_2409_13418_b200 import ContourOptions, GridSpec, _lib
    from paper_2409_13418_b200.slab import extract_piece

    R = 64
    field, lo, hi = scenes.resolve(scenes.thin_shell(R), R)
    g = GridSpec(lo, hi, R)
    ctx = _lib.context(0)
    L = _lib.load()
    piece = extract_piece(field, g, ContourOptions(), 30, 40)[0]
    n = ctypes.c_int64()
    assert L.odc_slab_seam(ctx.handle, None, ctypes.byref(n)) == 0
    tris = piece.triangles.cpu().numpy()
    assert n.value == int((tris < piece.n_halo).any(axis=1).sum()) > 0
    piece = extract_piece(field, g, ContourOptions(), 1, 3)[0]  # below the shell: no surface
    assert piece.triangles.shape[0] == 0
    assert L.odc_slab_seam(ctx.handle, None, ctypes.byref(n)) == 0 and n.value == 0


def test_balanced_slab_split_logic(monkeypatch):
    """The split of the cumulative work estimate (host logic; the device probe
    is replaced by a known work profile): equal shares, every rank >= 1 layer."""
    import paper_2409_13418_b200.slab as slab

    class G:
        resolution = 8

    # heavy middle layers: the middle ranks get fewer layers
    monkeypatch.setattr(slab, "layer_work", lambda field, grid, device=0, dfield=None:
                        np.array([1, 1, 4, 4, 4, 4, 1, 1], dtype=np.float64))
    assert slab.balanced_slab_ranges(None, G, 1) == [(0, 8)]
    r2 = slab.balanced_slab_ranges(None, G, 2)
    assert r2 == [(0, 4), (4, 8)]
    r4 = slab.balanced_slab_ranges(None, G, 4)
    assert r4[0][0] == 0 and r4[-1][1] == 8 and all(b > a for a, b in r4)
    assert [b - a for a, b in r4] == [3, 1, 1, 3]
    # more ranks than heavy layers: still one layer each at least
    r8 = slab.balanced_slab_ranges(None, G, 8)
    assert r8 == [(k, k + 1) for k in range(8)]
    with pytest.raises(ValueError):
        slab.balanced_slab_ranges(None, G, 9)
