"""Burst (short, below the power cap) MLP evaluator timing with and without
the L2 weight stream (mlp_debug bit 1)."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2409_13418_b200 import MlpField, _lib  # noqa: E402
from paper_2409_13418_b200.pipeline import DeviceField  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4_000_000
ctx = _lib.Context(0)
L = _lib.load()
L.odc_set_param(ctx.handle, b"mlp_impl", 3)
tr = np.zeros(1024, dtype=np.int64)
with DeviceField(ctx, MlpField()) as f:
    for dbg in (64, 65, 64, 65):
        L.odc_set_param(ctx.handle, b"mlp_debug", dbg)
        ms = []
        for _ in range(5):
            time.sleep(0.3)  # cool down between launches: stay below the power cap
            assert L.odc_profile_mlp(ctx.handle, f.handle, n, tr.ctypes.data, len(tr)) == 0
            ms.append(tr[-1] / 1e6)
        tf = 937984 * n / (np.median(ms) * 1e-3) / 1e12
        print(f"debug {dbg}: median {np.median(ms):.3f} ms -> {tf:.0f} TFLOP/s")
