"""Grid-vertex vs explicit-point MLP evaluator timing (mlp_debug bit 128) at
the batch sizes of the lock-step searches; burst launches with cool-downs."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2409_13418_b200 import MlpField, _lib  # noqa: E402
from paper_2409_13418_b200.pipeline import DeviceField  # noqa: E402

ctx = _lib.Context(0)
L = _lib.load()

tr = np.zeros(1024, dtype=np.int64)
extra = int(sys.argv[1]) if len(sys.argv) > 1 else 0
with DeviceField(ctx, MlpField()) as f:
    for n in (595_294, 1_190_588, 2_381_176, 8_000_000):
        row = []
        for dbg in (64 | extra, 192 | extra):
            L.odc_set_param(ctx.handle, b"mlp_debug", dbg)
            ms = []
            for _ in range(7):
                time.sleep(0.15)
                assert L.odc_profile_mlp(ctx.handle, f.handle, n, tr.ctypes.data, len(tr)) == 0
                ms.append(tr[-1] / 1e6)
            row.append(np.median(ms))
        tf = [937984 * n / (x * 1e-3) / 1e12 for x in row]
        print(f"n={n:9d} grid {row[0]:.3f} ms ({tf[0]:.0f} TF)  points {row[1]:.3f} ms ({tf[1]:.0f} TF)")
