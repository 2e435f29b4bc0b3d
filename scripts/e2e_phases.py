"""Time the phases of the public contour() call (field upload, extraction,
mesh copy-back, free) over several calls, to find host-side overhead."""
import ctypes
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from bench import workload  # noqa: E402
from paper_2409_13418_b200 import GridSpec, _lib, contour  # noqa: E402
from paper_2409_13418_b200 import pipeline as P  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "mlp_512"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 8
field, lo, hi, R, desc = workload(name)
g = GridSpec(lo, hi, R)
ctx = _lib.context(0)
L = _lib.load()
for i in range(reps):
    t = [time.perf_counter()]
    df = P.DeviceField(ctx, field)
    t.append(time.perf_counter())
    st = _lib.Stats()
    lo_c, hi_c, RR = P._grid_args(g)
    o = P.make_options(P.ContourOptions())
    rc = L.odc_extract(ctx.handle, df.handle, lo_c, hi_c, RR, ctypes.byref(o), ctypes.byref(st))
    t.append(time.perf_counter())
    m, raw = P._copy_meshes(ctx, st, True)
    t.append(time.perf_counter())
    t.append(time.perf_counter())
    df.free()
    t.append(time.perf_counter())
    res = contour(field, g)
    t.append(time.perf_counter())
    d = np.diff(t) * 1e3
    print(f"upload {d[0]:6.1f}  extract {d[1]:6.1f} (device {st.device_ms:6.1f})  copy {d[2]:6.1f}  raw {d[3]:5.1f}  "
          f"free {d[4]:5.1f}  | contour() {d[5]:6.1f} (device {res.stats['device_ms']:6.1f})")
