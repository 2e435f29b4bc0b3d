"""The z-slab multi-GPU step emulated on one GPU, assembly included.

For each slab count N (balanced bounds, paper_2409_13418_b200.slab):
  * every rank's slab extraction (odc_extract_slab, halo included) runs in
    turn: its device time is that rank's share of the step;
  * rank 0's assembly is then run for real on the same GPU: global ids
    (odc_slab_globalize), concatenation in rank order, unused-vertex removal
    and repair of the whole mesh (odc_mesh_finish) -- each timed on the device;
  * the gather itself (ranks 1..N-1 send vertices, triangles and provenance to
    rank 0 over NVLink) cannot be run on one GPU: its bytes are counted and
    its time estimated at --gather-gbs (default 300 GB/s, a conservative
    NCCL point-to-point rate on NVLink 5 / NVSwitch, 900 GB/s per direction).

step(N) = max over ranks of the slab time + gather estimate + rank 0's
globalize/concatenate/finish; efficiency = t(1 GPU) / (N step(N)).

Distributed finish (slab.finish_distributed, used when every fan is a
closed disc): per rank the slab extraction, its seam, the local finish with
the next rank's seam and the final ids, all timed on the device; the two
neighbour exchanges (seam triangles, top-layer ids) are a few MB and are
estimated at the same rate.  The mesh then stays on the ranks; gathering it
to rank 0 is the end-to-end part (reported separately).

    python scripts/slab_emulation.py mlp_512 thin_shell_1024
"""
import argparse
import ctypes
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from bench import workload  # noqa: E402
from paper_2409_13418_b200 import GridSpec, _lib  # noqa: E402
from paper_2409_13418_b200.pipeline import ContourOptions, DeviceField, _grid_args, make_options  # noqa: E402
from paper_2409_13418_b200.slab import (assemble, balanced_slab_ranges, extract_piece, global_offsets,  # noqa: E402
                                        globalize)


def timed(torch, fn, reps=3):
    best = None
    for _ in range(reps):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        out = fn()
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b)
        best = ms if best is None else min(best, ms)
    return out, best


def main():
    import torch

    ap = argparse.ArgumentParser()
    ap.add_argument("workloads", nargs="*", default=["mlp_512"])
    ap.add_argument("--gather-gbs", type=float, default=300.0)
    ap.add_argument("--worlds", default="2,4,8")
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    L = _lib.load()
    ctx = _lib.context(0)
    o = make_options(ContourOptions())
    for name in a.workloads:
        field, lo, hi, R, desc = workload(name)
        g = GridSpec(lo, hi, R)
        lo_c, hi_c, RR = _grid_args(g)
        with DeviceField(ctx, field) as df:
            st = _lib.Stats()
            for _ in range(3):
                assert L.odc_extract(ctx.handle, df.handle, lo_c, hi_c, RR, ctypes.byref(o), ctypes.byref(st)) == 0
            one = float(st.device_ms)
            print(f"{name}: 1 GPU {one:.2f} ms (device, whole extraction)")
            for world in (int(x) for x in a.worlds.split(",")):
                rr = balanced_slab_ranges(field, g, world, dfield=df)
                times, pieces = [], []
                for c0, c1 in rr:
                    sts = _lib.Stats()
                    info = _lib.SlabInfo()
                    for _ in range(2):
                        assert L.odc_extract_slab(ctx.handle, df.handle, lo_c, hi_c, RR, ctypes.byref(o), int(c0),
                                                  int(c1), ctypes.byref(sts), ctypes.byref(info)) == 0
                    times.append(float(sts.device_ms))
                    pieces.append(extract_piece(field, g, ContourOptions(), c0, c1, 0, dfield=df)[0])
                counts = np.array([[p.part_vertices.shape[0], p.fan_vertices.shape[0], p.triangles.shape[0]]
                                   for p in pieces])
                # rank 0's assembly: globalize every piece (on its own rank in
                # the real run: counted once, the max), concatenate, finish
                glob, gl_ms = [], []
                for k, p in enumerate(pieces):
                    extract_piece(field, g, ContourOptions(), *rr[k], 0, dfield=df)  # the context's last slab = k
                    pb, ptot, fb = global_offsets(counts, k)
                    t, ms = timed(torch, lambda: globalize(p, pb, ptot, fb, dev), reps=1)
                    gl_ms.append(ms)
                    glob.append([p.part_vertices, p.fan_vertices, t, p.part_cell, p.part_index, p.fan_edge])
                (verts, tris, kind, ref), cat_ms = timed(torch, lambda: assemble(glob, dev))
                fst = _lib.Stats()

                def finish():
                    torch.cuda.current_stream(dev).synchronize()
                    rc = L.odc_mesh_finish(ctx.handle, verts.data_ptr(), verts.shape[0], tris.data_ptr(),
                                           tris.shape[0], int(counts[:, 0].sum()), kind.data_ptr(), ref.data_ptr(),
                                           1, ctypes.byref(fst))
                    assert rc == 0, L.odc_last_error(ctx.handle)
                _, fin_wall = timed(torch, finish)
                fin_ms = float(fst.device_ms) if fst.device_ms > 0 else fin_wall
                # bytes that ranks 1.. send to rank 0: vertices (24 B), triangles
                # (12 B), provenance (kind 8 B + ref 16 B per vertex)
                sent = 0
                for p in pieces[1:]:
                    nv = p.part_vertices.shape[0] + p.fan_vertices.shape[0]
                    sent += nv * (24 + 24) + p.triangles.shape[0] * 12
                gather_ms = sent / (a.gather_gbs * 1e9) * 1e3
                step = max(times) + max(gl_ms) + gather_ms + cat_ms + fin_ms
                print(f"  {world} balanced slabs: per-rank slab ms {np.round(times, 2).tolist()}")
                # distributed finish, ranks from the top down (rank k needs rank k+1's seam);
                # run twice and keep the second (the first carries one-time allocations, like
                # the bench's warm-up steps)
                for _rep in range(2):
                    dist_ms, nondisc, seam_next, xbytes = [0.0] * world, 0, None, 0
                    fin_parts = [None] * world
                    for k in reversed(range(world)):
                        c0, c1 = rr[k]
                        sts = _lib.Stats()
                        info = _lib.SlabInfo()
                        assert L.odc_extract_slab(ctx.handle, df.handle, lo_c, hi_c, RR, ctypes.byref(o), int(c0),
                                                  int(c1), ctypes.byref(sts), ctypes.byref(info)) == 0
                        n = ctypes.c_int64()

                        def seam_fn():
                            L.odc_slab_seam(ctx.handle, None, ctypes.byref(n))
                            t = torch.empty((n.value, 3), dtype=torch.int32, device=dev)
                            if n.value:
                                L.odc_slab_seam(ctx.handle, t.data_ptr(), ctypes.byref(n))
                            return t
                        seam, t_seam = timed(torch, seam_fn, reps=1)
                        nh_next = int(pieces[k + 1].n_halo) if k + 1 < world else 0
                        U, nd = ctypes.c_int64(), ctypes.c_int64()
                        sn = seam_next if seam_next is not None else torch.empty((0, 3), dtype=torch.int32, device=dev)

                        def local_fn():
                            assert L.odc_slab_local_finish(ctx.handle, sn.data_ptr() if sn.numel() else None,
                                                           sn.shape[0], nh_next, ctypes.byref(U), ctypes.byref(nd)) == 0
                        _, t_local = timed(torch, local_fn, reps=1)
                        nondisc += nd.value
                        u = U.value
                        T_k = int(counts[k, 2])
                        top = torch.zeros((nh_next,), dtype=torch.int32, device=dev)
                        halo = torch.zeros((int(pieces[k].n_halo),), dtype=torch.int32, device=dev)
                        tri = torch.empty((T_k, 3), dtype=torch.int32, device=dev)
                        pv = torch.empty((u, 3), dtype=torch.float64, device=dev)
                        pc = torch.empty((u,), dtype=torch.int64, device=dev)
                        pi = torch.empty((u,), dtype=torch.int64, device=dev)
                        ptr = lambda t: t.data_ptr() if t.numel() else None  # noqa: E731

                        def final_fn():
                            if nh_next:
                                assert L.odc_slab_top_ids(ctx.handle, 0, nh_next, top.data_ptr()) == 0
                            assert L.odc_slab_final(ctx.handle, 0, 0, ptr(halo), ptr(tri), ptr(pv), ptr(pc), ptr(pi)) == 0
                        _, t_final = timed(torch, final_fn, reps=1)
                        dist_ms[k] = times[k] + t_seam + t_local + t_final
                        fin_parts[k] = (round(t_seam, 3), round(t_local, 3), round(t_final, 3))
                        xbytes = max(xbytes, seam.numel() * 4 + nh_next * 4)
                        seam_next = seam
                xchg_ms = 2 * xbytes / (a.gather_gbs * 1e9) * 1e3 + 0.05  # two neighbour exchanges + all-gathers
                dstep = max(dist_ms) + xchg_ms
                print(f"    distributed finish: per-rank ms {np.round(dist_ms, 2).tolist()} + exchanges "
                      f"{xchg_ms:.3f} (est) = {dstep:.2f} ms -> speedup {one / dstep:.2f} "
                      f"({one / dstep / world * 100:.0f} % of linear); non-disc fans {nondisc} "
                      f"({'fallback to the central finish' if nondisc else 'distributed path taken'})")
                print(f"    per-rank finish (seam, local, final) ms: {fin_parts}")
                print(f"    max slab {max(times):.2f} + globalize {max(gl_ms):.3f} + gather {gather_ms:.3f} "
                      f"({sent / 1e6:.1f} MB at {a.gather_gbs:.0f} GB/s, estimated) + concat {cat_ms:.3f} "
                      f"+ finish {fin_ms:.3f} (V={verts.shape[0]}, T={tris.shape[0]}, +{fst.repair_added_vertices} "
                      f"repair) = {step:.2f} ms -> speedup {one / step:.2f} ({one / step / world * 100:.0f} % of linear)")


if __name__ == "__main__":
    main()
