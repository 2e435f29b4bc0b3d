"""Dynamic (default) vs static round-robin pair schedule (mlp_debug bit 8),
same box, alternating, burst launches with cool-downs."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2409_13418_b200 import MlpField, _lib  # noqa: E402
from paper_2409_13418_b200.pipeline import DeviceField  # noqa: E402

ctx = _lib.Context(0)
L = _lib.load()
L.odc_set_param(ctx.handle, b"mlp_impl", 3)
tr = np.zeros(1024, dtype=np.int64)
pts = int(sys.argv[1]) if len(sys.argv) > 1 else 0
with DeviceField(ctx, MlpField()) as f:
    for n in (1_190_588, 2_381_176, 8_000_000, 30_000_000):
        res = {64: [], 72: []}
        for rep in range(6):
            for dbg in (64, 72):
                L.odc_set_param(ctx.handle, b"mlp_debug", dbg | pts)
                time.sleep(0.15)
                assert L.odc_profile_mlp(ctx.handle, f.handle, n, tr.ctypes.data, len(tr)) == 0
                res[dbg].append(tr[-1] / 1e6)
        d, st = np.median(res[64]), np.median(res[72])
        print(f"n={n:9d} dynamic {d:.3f} ms  static {st:.3f} ms  ({(st / d - 1) * 100:+.1f}% static slower)")
