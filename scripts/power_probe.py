"""Sustained MLP evaluator throughput under the power cap, with and without
the weight stream from L2 (mlp_debug bit 1: stale weights, timing only)."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2409_13418_b200 import MlpField, _lib  # noqa: E402
from paper_2409_13418_b200.pipeline import DeviceField  # noqa: E402

impl = int(sys.argv[1]) if len(sys.argv) > 1 else 3
n = int(sys.argv[2]) if len(sys.argv) > 2 else 100_000_000
ctx = _lib.Context(0)
L = _lib.load()
L.odc_set_param(ctx.handle, b"mlp_impl", impl)
tr = np.zeros(1024, dtype=np.int64)
with DeviceField(ctx, MlpField()) as f:
    for dbg in (64, 65, 64, 65):
        L.odc_set_param(ctx.handle, b"mlp_debug", dbg)
        ms = []
        t_end = time.time() + 3.0
        while time.time() < t_end:
            assert L.odc_profile_mlp(ctx.handle, f.handle, n, tr.ctypes.data, len(tr)) == 0
            ms.append(tr[-1] / 1e6)
        tf = 937984 * n / (np.median(ms[2:]) * 1e-3) / 1e12
        print(f"impl {impl} debug {dbg}: median {np.median(ms[2:]):.2f} ms over {len(ms)} runs -> {tf:.0f} TFLOP/s")
