"""Per-rank device time of the z-slab path, emulated on one GPU: each rank's
slab extraction (odc_extract_slab, halo included) run in turn.  The slowest
rank bounds the N-GPU step (before the count all-gather and rank 0's
assembly), so max(rank) vs the 1-GPU extraction estimates strong scaling."""
import ctypes
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from bench import workload  # noqa: E402
from paper_2409_13418_b200 import GridSpec, _lib, contour  # noqa: E402
from paper_2409_13418_b200.pipeline import ContourOptions, DeviceField, _grid_args, make_options  # noqa: E402
from paper_2409_13418_b200.slab import balanced_slab_ranges, slab_ranges  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "mlp_512"
field, lo, hi, R, desc = workload(name)
g = GridSpec(lo, hi, R)
ctx = _lib.Context(0)
L = _lib.load()
lo_c, hi_c, RR = _grid_args(g)
o = make_options(ContourOptions())
with DeviceField(ctx, field) as df:
    st = _lib.Stats()
    for _ in range(3):
        assert L.odc_extract(ctx.handle, df.handle, lo_c, hi_c, RR, ctypes.byref(o), ctypes.byref(st)) == 0
    one = st.device_ms
    print(f"{name}: 1 GPU {one:.2f} ms")
    for world, kind in ((2, "equal"), (4, "equal"), (8, "equal"), (2, "balanced"), (4, "balanced"), (8, "balanced")):
        times = []
        rr = slab_ranges(R, world) if kind == "equal" else balanced_slab_ranges(field, g, world)
        for c0, c1 in rr:
            st = _lib.Stats()
            info = _lib.SlabInfo()
            for _ in range(2):
                assert L.odc_extract_slab(ctx.handle, df.handle, lo_c, hi_c, RR, ctypes.byref(o), int(c0), int(c1),
                                          ctypes.byref(st), ctypes.byref(info)) == 0
            times.append(st.device_ms)
        mx = max(times)
        print(f"  {world} {kind} slabs: per-rank ms {np.round(times, 2).tolist()}  max {mx:.2f}  "
              f"-> speedup {one / mx:.2f} ({one / mx / world * 100:.0f} % of linear, before assembly)")
