"""z-slab multi-GPU extraction.

The grid's cells are numbered z-major (grid.py:84-87), edges and faces by
their lower vertex (grid.py:1-8), so the reference's global output order --
partition vertices in (cell, cycle) order, fan vertices and triangles in
edge-key order (polygonize.py:162-214) -- is exactly the concatenation of
per-slab outputs in slab order.  Rank k owns cell layers [c_k, c_{k+1}) and
the edges/faces whose lower vertex lies in those layers (the last rank also
owns the top vertex layer).  It recomputes the halo cell layer c_k - 1
(labels, searches, partitions and QEF are deterministic, hence identical to
the owner's result) so it can polygonize its seam edges without exchanging
any geometry.  The only collectives are

  1. an all-gather of the per-rank counts (owned partitions, fan vertices,
     triangles) from which every rank derives its global id offsets; a halo
     partition j of rank k is global id  part_base_k - n_halo_k + j;
  2. point-to-point sends of each rank's owned vertices / triangles /
     provenance to rank 0 (NCCL over NVLink on the GPU path),

after which rank 0 drops unreferenced vertices and runs the non-manifold
repair on the assembled mesh (polygonize.py:199-209, :253-374; a seam
vertex's fan spans two slabs).
"""

from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass

import numpy as np

from . import _lib
from .mesh import TriangleMesh

STAT_KEYS = ("n_grid_vertices", "boundary_inside_vertices", "n_crossing_edges", "n_crossing_cells",
             "n_face_center_probes", "n_2d_points", "n_partitions", "normal_fallbacks", "skipped_boundary_edges")


def slab_ranges(R, world):
    """Owned cell layers [c0, c1) of every rank (balanced split of R layers)."""
    if world < 1 or world > R:
        raise ValueError(f"cannot split {R} cell layers over {world} ranks")
    b = [R * k // world for k in range(world + 1)]
    return [(b[k], b[k + 1]) for k in range(world)]


# Cost of one crossing edge (its searches, cells, polygonization, repair) in
# units of one grid-pass evaluation, measured on one B200: MLP 512^3 --
# grid pass 76 ms for 1.35e8 evaluations, the rest 38 ms for 5.95e5
# crossing edges (~115, rounded up for the lower efficiency of the smaller
# per-slab launches); analytic thin shell 1024^3 (interval-culled labels,
# round 2) -- the grid pass far from the surface costs ~0.6 ps per vertex
# (one bound per 32 labels + the active-set pass), and everything near it
# (undecided label words, searches, cells, polygonization, finish) ~2 ns
# per crossing edge.
WORK_PER_CROSSING_MLP = 130.0
WORK_PER_CROSSING_ANALYTIC = 3000.0


def surface_layer_crossings(grid, dfield, device=0):
    """Crossing edges per cell layer of an analytic field, estimated from the
    device's surface probe (odc_surface_probe): cubic boxes of B vertices
    whose interval bound cannot exclude the surface.  A surface patch of
    area A leaves ~A (1 + sqrt 3) / (B h)^2 boxes undecided (the bound's
    margin is the box's circumradius) and crosses ~1.5 A / h^2 grid edges,
    so crossings ~ 0.55 B^2 x undecided boxes, spread over the box layer.
    Unlike a coarse label probe this sees walls thinner than its spacing
    (the config-4 thin shell)."""
    R = int(grid.resolution)
    box = max(4, R // 64)
    nbz = -(-R // box)
    counts = np.zeros(nbz, dtype=np.int64)
    lo = (ctypes.c_double * 3)(*[float(x) for x in grid.lo])
    hi = (ctypes.c_double * 3)(*[float(x) for x in grid.hi])
    ctx = _lib.context(device)
    _lib.check(_lib.load().odc_surface_probe(ctx.handle, dfield.handle, lo, hi, R, box, counts.ctypes.data),
               ctx.handle)
    k = np.zeros(R, dtype=np.float64)
    for bz in range(nbz):
        z0, z1 = bz * box, min(R, (bz + 1) * box)
        k[z0:z1] = 0.55 * box * box * counts[bz] / (z1 - z0)
    return k


def layer_work(field, grid, device=0, nxy=17, nz_max=129, dfield=None):
    """Estimated work of every cell layer, in grid-pass evaluations: S^2
    vertices per layer plus WORK_PER_CROSSING_* per crossing edge.
    Analytic fields: crossings from the device surface probe
    (surface_layer_crossings).  Others: crossings per layer from a coarse
    label probe (nxy^2 points on up to nz_max z-planes, evaluated on the
    device), scaled to the fine grid by the ratio of cell areas.
    Deterministic: every rank computes the same estimate, so no
    communication is needed to agree on slab bounds."""
    from .fields import is_mlp
    from .pipeline import DeviceField, eval_labels

    per_crossing = WORK_PER_CROSSING_MLP if is_mlp(field) else WORK_PER_CROSSING_ANALYTIC

    R = int(grid.resolution)
    if not is_mlp(field):
        if dfield is not None and getattr(dfield, "analytic", False):
            return np.full(R, float(R + 1) ** 2) + per_crossing * surface_layer_crossings(grid, dfield, device)
        if dfield is None:
            with DeviceField(_lib.context(device), field) as df:
                if df.analytic:
                    return np.full(R, float(R + 1) ** 2) + per_crossing * surface_layer_crossings(grid, df, device)
    lo, hi = np.asarray(grid.lo, dtype=np.float64), np.asarray(grid.hi, dtype=np.float64)
    zs = max(1, -(-R // (nz_max - 1)))  # z stride in vertex layers
    zi = np.arange(0, R + 1, zs)
    if zi[-1] != R:
        zi = np.append(zi, R)
    h = (hi - lo) / R
    xs = np.linspace(lo[0], hi[0], nxy)
    ys = np.linspace(lo[1], hi[1], nxy)
    zz = lo[2] + zi * h[2]
    Z, Y, X = np.meshgrid(zz, ys, xs, indexing="ij")
    pts = np.ascontiguousarray(np.stack([X.ravel(), Y.ravel(), Z.ravel()], axis=1))
    if dfield is not None:  # the caller's upload (contour_slab): no second field upload
        lab = np.empty(len(pts), dtype=np.uint8)
        ctx = _lib.context(device)
        _lib.check(_lib.load().odc_eval_labels(ctx.handle, dfield.handle, pts.ctypes.data, len(pts),
                                               lab.ctypes.data), ctx.handle)
    else:
        lab = eval_labels(field, pts, device=device)
    lab = lab.reshape(len(zi), nxy, nxy)
    cx = (lab[:, :, 1:] != lab[:, :, :-1]).sum(axis=(1, 2)).astype(np.float64)
    cy = (lab[:, 1:, :] != lab[:, :-1, :]).sum(axis=(1, 2)).astype(np.float64)
    cz = (lab[1:] != lab[:-1]).sum(axis=(1, 2)).astype(np.float64)
    Hx, Hy = (hi[0] - lo[0]) / (nxy - 1), (hi[1] - lo[1]) / (nxy - 1)
    work = np.full(R, float(R + 1) ** 2)
    for b in range(len(zi) - 1):
        z0, z1 = int(zi[b]), int(zi[b + 1])
        Hz = (z1 - z0) * h[2]
        # fine crossing edges in the band: coarse crossings x (coarse cell
        # face area / fine cell face area) for each axis
        kx = 0.5 * (cx[b] + cx[b + 1]) * (Hy * Hz) / (h[1] * h[2])
        ky = 0.5 * (cy[b] + cy[b + 1]) * (Hx * Hz) / (h[0] * h[2])
        kz = cz[b] * (Hx * Hy) / (h[0] * h[1])
        work[z0:z1] += per_crossing * (kx + ky + kz) / (z1 - z0)
    return work


def balanced_slab_ranges(field, grid, world, device=0, dfield=None):
    """Owned cell layers [c0, c1) of every rank, split so that the estimated
    work (layer_work) is equal: a surface concentrated in the middle z-range
    otherwise leaves the outer slabs idle (a centred sphere-like surface:
    per-rank times 24/37/36/25 ms over 4 equal slabs at 512^3)."""
    R = int(grid.resolution)
    if world < 1 or world > R:
        raise ValueError(f"cannot split {R} cell layers over {world} ranks")
    if world == 1:
        return [(0, R)]
    w = layer_work(field, grid, device, dfield=dfield)
    cum = np.concatenate([[0.0], np.cumsum(w)])
    b = [0]
    for k in range(1, world):
        target = cum[-1] * k / world
        c = int(np.searchsorted(cum, target))  # first layer boundary at or past the target
        if c > 0 and target - cum[c - 1] < cum[min(c, R)] - target:
            c -= 1  # the nearer boundary
        b.append(min(max(c, b[-1] + 1), R - (world - k)))  # every rank keeps >= 1 layer
    b.append(R)
    return [(b[k], b[k + 1]) for k in range(world)]


def global_offsets(counts, rank):
    """counts: (world, 3) [n_partitions, n_fans, n_triangles] of every rank.
    Returns (part_base, n_partitions_total, fan_base) of ``rank``."""
    counts = np.asarray(counts, dtype=np.int64)
    return int(counts[:rank, 0].sum()), int(counts[:, 0].sum()), int(counts[:rank, 1].sum())


def globalize_ids(local, n_halo, n_window, part_base, n_total, fan_base):
    """Host-side restatement of k_globalize_tris (odc_kernels.cu) for the
    CPU (gloo) path and tests: local -> global vertex ids."""
    local = np.asarray(local, dtype=np.int64)
    out = np.where(local < n_halo, part_base - n_halo + local,
                   np.where(local < n_window, part_base + (local - n_halo), n_total + fan_base + (local - n_window)))
    return out


@dataclass
class SlabPiece:
    """What one rank contributes (arrays are torch tensors on the rank's device)."""

    n_halo: int
    n_window: int
    part_vertices: object   # (P, 3) f64
    fan_vertices: object    # (NF, 3) f64
    triangles: object       # (T, 3) int32 local ids
    part_cell: object       # (P,) i64
    part_index: object      # (P,) i64
    fan_edge: object        # (NF,) i64
    stats: np.ndarray       # STAT_KEYS + eval counts
    c0: int = -1            # owned cell layers [c0, c1)
    c1: int = -1


class _CudaArray:
    """Zero-copy view of a libodc device buffer (__cuda_array_interface__)."""

    def __init__(self, ptr, shape, typestr):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (int(ptr), False),
                                         "version": 3, "strides": None}


def _dev(torch, ptr, shape, typestr, device):
    n = int(np.prod(shape))
    dt = {"<f8": torch.float64, "<i4": torch.int32, "<i8": torch.int64}[typestr]
    if n == 0 or not ptr:
        return torch.zeros(shape, dtype=dt, device=device)
    return torch.as_tensor(_CudaArray(ptr, shape, typestr), device=device).clone()


def extract_piece(field, grid, options, c0, c1, device=0, dfield=None):
    """Run libodc's slab extraction for owned cell layers [c0, c1)
    (``dfield``: an already uploaded DeviceField on this thread's context)."""
    import contextlib

    import torch

    from .pipeline import DeviceField, _grid_args, _raise, make_options

    ctx = _lib.context(device)
    L = _lib.load()
    st = _lib.Stats()
    info = _lib.SlabInfo()
    lo, hi, R = _grid_args(grid)
    o = make_options(options)
    with (contextlib.nullcontext(dfield) if dfield is not None else DeviceField(ctx, field)) as df:
        rc = L.odc_extract_slab(ctx.handle, df.handle, lo, hi, R, ctypes.byref(o), int(c0), int(c1), ctypes.byref(st),
                                ctypes.byref(info))
        if rc != _lib.ODC_OK:
            _raise(rc, ctx, df)
    dev = torch.device("cuda", device)
    P, NF, T = info.n_partitions, info.n_fans, info.n_triangles
    piece = SlabPiece(
        n_halo=int(info.n_halo_partitions), n_window=int(info.n_window_partitions),
        part_vertices=_dev(torch, info.partition_vertices, (P, 3), "<f8", dev),
        fan_vertices=_dev(torch, info.fan_vertices, (NF, 3), "<f8", dev),
        triangles=_dev(torch, info.triangles, (T, 3), "<i4", dev),
        part_cell=_dev(torch, info.partition_cell, (P,), "<i8", dev),
        part_index=_dev(torch, info.partition_index, (P,), "<i8", dev),
        fan_edge=_dev(torch, info.fan_edge, (NF,), "<i8", dev),
        stats=stats_vector(st),
        c0=int(c0), c1=int(c1),
    )
    return piece, ctx


def stats_vector(st):
    v = [getattr(st, k) for k in STAT_KEYS]
    v += list(st.point2d_status_counts) + list(st.qef_rank_counts) + list(st.split_case_counts)
    v += list(st.eval_batches) + list(st.eval_evals)
    v.append(int(np.array([st.qef_max_residual]).view(np.int64)[0]))  # >= 0 doubles order like their bits
    # extras for the benchmark: kernel launches, grid-label kernel time (ns)
    v.append(int(st.n_kernel_launches))
    v.append(int(round(float(st.stage_ms[7]) * 1e6)))
    return np.asarray(v, dtype=np.int64)


def run_extras(rows):
    """(kernel launches summed over ranks, slowest rank's grid-label kernel ms)."""
    rows = np.asarray(rows)
    return int(rows[:, -2].sum()), float(rows[:, -1].max()) / 1e6


def rank_label_work(rows):
    """Per rank: (grid-label evaluations incl. the halo layer, grid-label
    kernel ms) -- for the slowest rank's roofline."""
    rows = np.asarray(rows)
    nk = len(STAT_KEYS)
    return rows[:, nk + 18].astype(np.int64), rows[:, -1].astype(np.float64) / 1e6


def probe_bytes(grid, nxy=17, nz_max=129, analytic=False):
    """Host<->device bytes of layer_work's probe per rank: (H2D points, D2H
    labels), or for an analytic field the surface probe's (0, its counts)."""
    R = int(grid.resolution)
    if analytic:
        return 0, 8 * -(-R // max(4, R // 64))
    zs = max(1, -(-R // (nz_max - 1)))
    nz = len(range(0, R + 1, zs)) + (0 if R % zs == 0 else 1)
    n = nz * nxy * nxy
    return 24 * n, n


def check_ranges(allc, R=None):
    """Every rank computes its slab bounds on its own; rank 0 checks that the
    gathered [c0, c1) ranges tile [0, R) in rank order (overlaps or gaps
    would silently corrupt the global ids)."""
    c0, c1 = allc[:, 3], allc[:, 4]
    ok = c0[0] == 0 and bool(np.all(c1[:-1] == c0[1:])) and bool(np.all(c1 > c0))
    if R is not None:
        ok = ok and c1[-1] == R
    if not ok:
        raise RuntimeError(f"slab ranges do not tile the grid: {list(zip(c0.tolist(), c1.tolist()))}")


def stitch(piece, rank, world, dist, device, R=None):
    """Collectives + assembly.  Returns the assembled arrays on rank 0
    (vertices, triangles (global int32), kind, ref, n_partitions_total,
    per-rank stats) and None elsewhere.  One all-gather of the counts and
    stats, then one grouped point-to-point exchange (every rank's six
    payload tensors to rank 0 in a single batch_isend_irecv, i.e. one
    ncclGroupStart/End on the NCCL backend).  With the gloo backend and
    device tensors (several ranks sharing one GPU in the tests) the payload
    is staged through host memory."""
    import torch

    stage = dist.get_backend() == "gloo" and torch.device(device).type == "cuda"
    wire = torch.device("cpu") if stage else device
    P, NF, T = piece.part_vertices.shape[0], piece.fan_vertices.shape[0], piece.triangles.shape[0]
    head = torch.tensor([P, NF, T, piece.c0, piece.c1], dtype=torch.int64)
    sv = torch.cat([head, torch.as_tensor(piece.stats, dtype=torch.int64)]).to(wire)
    gathered = [torch.zeros_like(sv) for _ in range(world)]
    dist.all_gather(gathered, sv)
    rows = torch.stack(gathered).cpu().numpy()
    allc, stats_rows = rows[:, :5], rows[:, 5:]
    if rank == 0:
        check_ranges(allc, R)
    part_base, P_tot, fan_base = global_offsets(allc[:, :3], rank)
    tris = globalize(piece, part_base, P_tot, fan_base, device)
    payload = [piece.part_vertices.contiguous(), piece.fan_vertices.contiguous(), tris.contiguous(),
               piece.part_cell.contiguous(), piece.part_index.contiguous(), piece.fan_edge.contiguous()]
    if stage and rank != 0:
        payload = [t.cpu() for t in payload]
    if rank != 0:
        ops = [dist.P2POp(dist.isend, t, 0) for t in payload if t.numel()]
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        return None
    parts = [[p] for p in payload]
    ops = []
    for r in range(1, world):
        Pr, NFr, Tr = (int(x) for x in allc[r, :3])
        bufs = [torch.empty((Pr, 3), dtype=torch.float64, device=wire),
                torch.empty((NFr, 3), dtype=torch.float64, device=wire),
                torch.empty((Tr, 3), dtype=torch.int32, device=wire),
                torch.empty((Pr,), dtype=torch.int64, device=wire),
                torch.empty((Pr,), dtype=torch.int64, device=wire),
                torch.empty((NFr,), dtype=torch.int64, device=wire)]
        ops += [dist.P2POp(dist.irecv, b, r) for b in bufs if b.numel()]
        for i, b in enumerate(bufs):
            parts[i].append(b)
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    if stage:
        parts = [[p[0]] + [b.to(device) for b in p[1:]] for p in parts]
    verts, tr, kind, ref = assemble([[p[r] for p in parts] for r in range(world)], device)
    return verts, tr, kind, ref, P_tot, stats_rows


def _torch_sync(device):
    """libodc runs on its context's own stream: tensors torch just wrote (or a
    block the caching allocator just recycled) must be complete before the
    library touches them."""
    import torch

    torch.cuda.current_stream(device).synchronize()


def globalize(piece, part_base, P_tot, fan_base, device):
    import torch

    T = piece.triangles.shape[0]
    out = torch.empty((T, 3), dtype=torch.int32, device=device)
    if T == 0:
        return out
    if piece.triangles.is_cuda:
        ctx = _lib.context(piece.triangles.device.index or 0)
        _torch_sync(out.device)
        rc = _lib.load().odc_slab_globalize(ctx.handle, part_base, P_tot, fan_base, out.data_ptr())
        if rc != _lib.ODC_OK:
            raise RuntimeError(_lib.load().odc_last_error(ctx.handle).decode())
        return out
    g = globalize_ids(piece.triangles.numpy(), piece.n_halo, piece.n_window, part_base, P_tot, fan_base)
    return torch.as_tensor(g.astype(np.int32))


def aggregate_stats(rows, options):
    """Sum per-rank stats vectors into the reference's stats dict."""
    from .pipeline import STATUS_NAMES

    rows = np.asarray(rows)
    nk = len(STAT_KEYS)
    tot = rows[:, :nk].sum(axis=0)
    d = dict(zip(STAT_KEYS, (int(x) for x in tot)))
    status = rows[:, nk:nk + 4].sum(axis=0)
    ranks = rows[:, nk + 4:nk + 8].sum(axis=0)
    split = rows[:, nk + 8:nk + 12].sum(axis=0)
    batches = rows[:, nk + 12:nk + 18].max(axis=0)
    evals = rows[:, nk + 18:nk + 24].sum(axis=0)
    resid = float(np.array([rows[:, nk + 24].max()], dtype=np.int64).view(np.float64)[0])
    return d, status, ranks, split, batches, evals, resid


def _p2p(dist, sends, recvs):
    """One grouped exchange: sends = [(tensor, peer)], recvs = [(tensor, peer)]."""
    ops = [dist.P2POp(dist.isend, t, r) for t, r in sends if t.numel()]
    ops += [dist.P2POp(dist.irecv, t, r) for t, r in recvs if t.numel()]
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()


def finish_distributed(piece, ctx, rank, world, dist, device, R=None):
    """Finish the mesh on the ranks that produced it (odc.h "Distributed
    finish"): seam triangles go one rank down, every rank marks/compacts its
    used partitions and checks that all its vertices' fans are closed discs.
    Returns None on every rank when some fan is not (the caller then runs
    the central finish, which repairs); else this rank's final piece
    [partition vertices, fan vertices, triangles (global ids), partition
    cell, partition index, fan edge] and the all-gathered count/stat rows."""
    import torch

    L = _lib.load()
    device = torch.device(device)
    stage = dist.get_backend() == "gloo" and device.type == "cuda"
    wire = torch.device("cpu") if stage else device
    _torch_sync(device)  # torch-allocated buffers below are written on libodc's stream
    n = ctypes.c_int64()
    _lib.check(L.odc_slab_seam(ctx.handle, None, ctypes.byref(n)), ctx.handle)
    seam = torch.empty((n.value, 3), dtype=torch.int32, device=device)
    if n.value:
        _lib.check(L.odc_slab_seam(ctx.handle, seam.data_ptr(), ctypes.byref(n)), ctx.handle)
    P, NF, T = piece.part_vertices.shape[0], piece.fan_vertices.shape[0], piece.triangles.shape[0]
    head = torch.tensor([P, NF, T, piece.c0, piece.c1, piece.n_halo, seam.shape[0]], dtype=torch.int64)
    sv = torch.cat([head, torch.as_tensor(piece.stats, dtype=torch.int64)]).to(wire)
    gathered = [torch.zeros_like(sv) for _ in range(world)]
    dist.all_gather(gathered, sv)
    rows = torch.stack(gathered).cpu().numpy()
    allc, stats_rows = rows[:, :7], rows[:, 7:]
    if rank == 0:
        check_ranges(allc[:, :5], R)
    # seam exchange: this rank's seam to the rank below, the next rank's to here
    nxt = rank + 1 < world
    recv = torch.empty((int(allc[rank + 1, 6]) if nxt else 0, 3), dtype=torch.int32, device=wire)
    send = seam.to(wire) if stage else seam
    _p2p(dist, [(send, rank - 1)] if rank > 0 else [], [(recv, rank + 1)] if nxt else [])
    recv = recv.to(device)
    torch.cuda.current_stream(device).synchronize()
    U, nd = ctypes.c_int64(), ctypes.c_int64()
    _lib.check(L.odc_slab_local_finish(ctx.handle, recv.data_ptr() if recv.numel() else None, recv.shape[0],
                                       int(allc[rank + 1, 5]) if nxt else 0, ctypes.byref(U), ctypes.byref(nd)),
               ctx.handle)
    fin = torch.tensor([U.value, nd.value], dtype=torch.int64, device=wire)
    got = [torch.zeros_like(fin) for _ in range(world)]
    dist.all_gather(got, fin)
    un = torch.stack(got).cpu().numpy()
    if un[:, 1].sum() > 0:
        return None
    Us, NFs = un[:, 0], allc[:, 1]
    part_base, P_tot = int(Us[:rank].sum()), int(Us.sum())
    fan_base = P_tot + int(NFs[:rank].sum())
    # global ids of this rank's top-layer partitions to the next rank (its halo)
    top = torch.empty((int(allc[rank + 1, 5]) if nxt else 0,), dtype=torch.int32, device=device)
    if top.numel():
        _lib.check(L.odc_slab_top_ids(ctx.handle, part_base, top.shape[0], top.data_ptr()), ctx.handle)
    halo = torch.empty((piece.n_halo,), dtype=torch.int32, device=wire)
    _p2p(dist, [(top.to(wire) if stage else top, rank + 1)] if nxt else [], [(halo, rank - 1)] if rank > 0 else [])
    halo = halo.to(device)
    torch.cuda.current_stream(device).synchronize()
    u = int(Us[rank])
    tris = torch.empty((T, 3), dtype=torch.int32, device=device)
    pv = torch.empty((u, 3), dtype=torch.float64, device=device)
    pc = torch.empty((u,), dtype=torch.int64, device=device)
    pi = torch.empty((u,), dtype=torch.int64, device=device)
    ptr = lambda t: t.data_ptr() if t.numel() else None  # noqa: E731
    _lib.check(L.odc_slab_final(ctx.handle, part_base, fan_base, ptr(halo), ptr(tris), ptr(pv), ptr(pc), ptr(pi)),
               ctx.handle)
    final = [pv, piece.fan_vertices.contiguous(), tris, pc, pi, piece.fan_edge.contiguous()]
    return final, allc, stats_rows, Us


def gather_final(final, Us, allc, rank, world, dist, device):
    """Rank 0 receives every rank's final piece (one grouped exchange) and
    concatenates it in the reference's order; None on the other ranks."""
    import torch

    device = torch.device(device)
    stage = dist.get_backend() == "gloo" and device.type == "cuda"
    wire = torch.device("cpu") if stage else device
    if rank != 0:
        _p2p(dist, [(t.to(wire) if stage else t, 0) for t in final], [])
        return None
    parts = [[t] for t in final]
    recvs = []
    for r in range(1, world):
        u, nf, t = int(Us[r]), int(allc[r, 1]), int(allc[r, 2])
        bufs = [torch.empty((u, 3), dtype=torch.float64, device=wire),
                torch.empty((nf, 3), dtype=torch.float64, device=wire),
                torch.empty((t, 3), dtype=torch.int32, device=wire),
                torch.empty((u,), dtype=torch.int64, device=wire),
                torch.empty((u,), dtype=torch.int64, device=wire),
                torch.empty((nf,), dtype=torch.int64, device=wire)]
        recvs += [(b, r) for b in bufs]
        for i, b in enumerate(bufs):
            parts[i].append(b)
    _p2p(dist, [], recvs)
    if stage:
        parts = [[p[0]] + [b.to(device) for b in p[1:]] for p in parts]
    return assemble([[p[r] for p in parts] for r in range(world)], device)


def contour_slab(field, grid, options=None, *, rank, world, dist, device=0, to_host=True, distributed=True):
    """One rank of a z-slab extraction over ``world`` ranks (one per GPU).
    Returns the ContourResult on rank 0 and None on the other ranks; with
    ``to_host=False`` the finished mesh stays on rank 0's device (read it with
    odc_mesh_device) and only the stats are returned.

    ``distributed``: finish on the ranks (finish_distributed) whenever every
    vertex fan is a closed disc -- then ``to_host=False`` returns as soon as
    every rank holds its final piece (the mesh stays distributed) and
    ``to_host=True`` gathers the pieces to rank 0; otherwise (or with
    ``distributed=False``) the pieces are gathered and rank 0 finishes and
    repairs the whole mesh."""
    import torch

    from .pipeline import ContourOptions, ContourResult, EvalCounter, _copy_mesh, _raise, _raw_from_repaired

    options = options or ContourOptions()
    options.validate()
    t0 = time.perf_counter()
    from .pipeline import DeviceField

    with DeviceField(_lib.context(device), field) as df:  # one upload for the probe and the slab
        c0, c1 = balanced_slab_ranges(field, grid, world, device, dfield=df)[rank]
        piece, ctx = extract_piece(field, grid, options, c0, c1, device, dfield=df)
    if distributed and options.repair and world > 1:
        dres = finish_distributed(piece, ctx, rank, world, dist, torch.device("cuda", device),
                                  R=int(grid.resolution))
        if dres is not None:
            return _distributed_result(field, options, dres, rank, world, dist, device, to_host, t0)
    out = stitch(piece, rank, world, dist, torch.device("cuda", device), R=int(grid.resolution))
    if out is None:
        return None
    verts, tris, kind, ref, P_tot, rows = out
    L = _lib.load()
    st = _lib.Stats()
    _torch_sync(verts.device)
    rc = L.odc_mesh_finish(ctx.handle, verts.data_ptr(), verts.shape[0], tris.data_ptr(), tris.shape[0], P_tot,
                           kind.data_ptr(), ref.data_ptr(), int(bool(options.repair)), ctypes.byref(st))
    if rc != _lib.ODC_OK:
        _raise(rc, ctx)
    if not to_host:
        launches, k_ms = run_extras(rows)
        ev, kms = rank_label_work(rows)
        return {"finish": st, "n_kernel_launches": launches + int(st.n_kernel_launches), "labels_kernel_ms": k_ms,
                "rank_label_evals": ev.tolist(), "rank_label_ms": kms.tolist()}
    mesh = _copy_mesh(ctx, 0, st) if st.n_triangles else TriangleMesh(np.zeros((0, 3)), np.zeros((0, 3), np.int64))
    raw = mesh if st.repair_added_vertices == 0 else _raw_from_repaired(ctx, mesh, st)
    stats = slab_stats(rows, options, st)
    counter = EvalCounter(field)
    _, _, _, _, batches, evals, _ = aggregate_stats(rows, options)
    for c, name in enumerate(_lib.CATEGORIES):
        if evals[c] or (batches[c] and c == 0):
            counter.record(name, int(batches[c]), int(evals[c]))
    stats["wall_time_s"] = time.perf_counter() - t0
    stats["eval_counts"] = counter.snapshot()
    stats["slabs"] = world
    launches, k_ms = run_extras(rows)
    stats["n_kernel_launches"] = launches + int(st.n_kernel_launches)
    stats["labels_kernel_ms"] = k_ms
    return ContourResult(mesh, raw, counter, stats)


def _distributed_result(field, options, dres, rank, world, dist, device, to_host, t0):
    import torch

    from .pipeline import ContourResult, EvalCounter

    final, allc, rows, Us = dres
    if not to_host:
        torch.cuda.synchronize(device)
        if rank != 0:
            return None
        launches, k_ms = run_extras(rows)
        ev, kms = rank_label_work(rows)
        return {"finish": None, "distributed": True, "n_kernel_launches": launches, "labels_kernel_ms": k_ms,
                "rank_label_evals": ev.tolist(), "rank_label_ms": kms.tolist()}
    out = gather_final(final, Us, allc, rank, world, dist, device)
    if out is None:
        return None
    verts, tris, kind, ref = out
    if tris.shape[0] == 0:  # pipeline.py:174-179: the empty mesh carries no provenance
        mesh = TriangleMesh(np.zeros((0, 3)), np.zeros((0, 3), dtype=np.int64))
    else:
        mesh = TriangleMesh(verts.cpu().numpy(), tris.cpu().numpy().astype(np.int64),
                            provenance_kind=kind.cpu().numpy(), provenance_ref=ref.cpu().numpy())

    class _NoRepair:
        repair_added_vertices = 0

    stats = slab_stats(rows, options, _NoRepair())
    counter = EvalCounter(field)
    _, _, _, _, batches, evals, _ = aggregate_stats(rows, options)
    for c, name in enumerate(_lib.CATEGORIES):
        if evals[c] or (batches[c] and c == 0):
            counter.record(name, int(batches[c]), int(evals[c]))
    stats["wall_time_s"] = time.perf_counter() - t0
    stats["eval_counts"] = counter.snapshot()
    stats["slabs"] = world
    stats["distributed_finish"] = True
    launches, k_ms = run_extras(rows)
    stats["n_kernel_launches"] = launches
    stats["labels_kernel_ms"] = k_ms
    return ContourResult(mesh, mesh, counter, stats)


def assemble(pieces_global, device):
    """Concatenate per-rank (part_vertices, fan_vertices, triangles_global,
    part_cell, part_index, fan_edge) in rank order: partitions of all ranks,
    then fans of all ranks (the reference's vertex order)."""
    import torch

    pv, fv, tr, pc, pi, fe = (torch.cat([p[i] for p in pieces_global]) for i in range(6))
    verts = torch.cat([pv, fv])
    kind = torch.cat([torch.zeros(pv.shape[0], dtype=torch.int64, device=device),
                      torch.ones(fv.shape[0], dtype=torch.int64, device=device)])
    ref = torch.cat([torch.stack([pc, pi], dim=1), torch.stack([fe, torch.full_like(fe, -1)], dim=1)])
    return verts, tr, kind, ref


def contour_slabs_serial(field, grid, n_slabs, options=None, device=0, ranges=None):
    """All slabs of an n-way decomposition run one after another on one GPU
    (the same kernels and id arithmetic as the multi-GPU path, without the
    collectives) and finished into one mesh -- used to check that slab
    decomposition reproduces the single-extraction result exactly."""
    import torch

    from .pipeline import ContourOptions, _copy_mesh, _raise

    options = options or ContourOptions()
    dev = torch.device("cuda", device)
    ranges = ranges or slab_ranges(grid.resolution, n_slabs)
    pieces = [extract_piece(field, grid, options, c0, c1, device)[0] for c0, c1 in ranges]
    counts = np.array([[p.part_vertices.shape[0], p.fan_vertices.shape[0], p.triangles.shape[0]] for p in pieces])
    glob = []
    for k, p in enumerate(pieces):
        part_base, P_tot, fan_base = global_offsets(counts, k)
        t = globalize_ids(p.triangles.cpu().numpy(), p.n_halo, p.n_window, part_base, P_tot, fan_base)
        glob.append([p.part_vertices, p.fan_vertices, torch.as_tensor(t.astype(np.int32), device=dev), p.part_cell,
                     p.part_index, p.fan_edge])
    verts, tris, kind, ref = assemble(glob, dev)
    ctx = _lib.context(device)
    st = _lib.Stats()
    _torch_sync(dev)
    rc = _lib.load().odc_mesh_finish(ctx.handle, verts.data_ptr(), verts.shape[0], tris.data_ptr(), tris.shape[0],
                                     int(counts[:, 0].sum()), kind.data_ptr(), ref.data_ptr(),
                                     int(bool(options.repair)), ctypes.byref(st))
    if rc != _lib.ODC_OK:
        _raise(rc, ctx)
    return _copy_mesh(ctx, 0, st), pieces, np.stack([p.stats for p in pieces])


def slab_stats(rows, options, st_finish):
    from .pipeline import STATUS_NAMES

    d, status, ranks, split, batches, evals, resid = aggregate_stats(rows, options)
    stats = {"options": options, "warnings": []}
    bi = d["boundary_inside_vertices"]
    stats["boundary_inside_vertices"] = bi
    if bi:
        stats["warnings"].append(f"{bi} boundary grid vertices are inside; the output will have an open boundary")
    stats["n_crossing_edges"] = d["n_crossing_edges"]
    stats["n_crossing_cells"] = d["n_crossing_cells"]
    if d["n_crossing_edges"] == 0:
        stats["n_2d_points"] = 0
        stats["open_boundary"] = False
        return stats
    stats["n_partitions"] = d["n_partitions"]
    stats["n_2d_points"] = d["n_2d_points"]
    if options.normals == "two-d-points":
        stats["point2d_status_counts"] = {STATUS_NAMES[c]: int(status[c]) for c in range(4) if status[c]}
    stats["normal_fallbacks"] = d["normal_fallbacks"]
    stats["qef_rank_counts"] = {r: int(ranks[r]) for r in range(4) if ranks[r]}
    stats["qef_max_residual"] = float(resid)
    stats["split_case_counts"] = {c: int(split[c]) for c in range(1, 4) if split[c]}
    stats["open_boundary"] = d["skipped_boundary_edges"] > 0
    stats["skipped_boundary_edges"] = d["skipped_boundary_edges"]
    stats["repair_added_vertices"] = int(st_finish.repair_added_vertices)
    return stats
