"""Back-to-back evaluator launches (no cool-down, as inside an extraction):
per-launch time vs batch size, to expose the fixed per-launch cost."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2409_13418_b200 import MlpField, _lib  # noqa: E402
from paper_2409_13418_b200.pipeline import DeviceField  # noqa: E402

ctx = _lib.Context(0)
L = _lib.load()
L.odc_set_param(ctx.handle, b"mlp_impl", 3)
tr = np.zeros(2048, dtype=np.int64)
dbg = int(sys.argv[1]) if len(sys.argv) > 1 else 192  # 64 no trace | 128 explicit points
with DeviceField(ctx, MlpField()) as f:
    L.odc_set_param(ctx.handle, b"mlp_debug", dbg)
    for _ in range(int(sys.argv[2]) if len(sys.argv) > 2 else 30):  # heat up to the sustained state
        L.odc_profile_mlp(ctx.handle, f.handle, 8_000_000, tr.ctypes.data, len(tr))
    res = {}
    for n in (37_888, 297_647, 595_294, 1_190_588, 2_381_176, 8_000_000):
        ms = []
        for _ in range(12):
            assert L.odc_profile_mlp(ctx.handle, f.handle, n, tr.ctypes.data, len(tr)) == 0
            ms.append(tr[-1] / 1e6)
        res[n] = np.median(ms)
    rate = res[8_000_000] / 8_000_000
    for n, t in res.items():
        print(f"n={n:9d} {t * 1e3:8.1f} us   at the 8M rate {rate * n * 1e3:8.1f} us   overhead {(t - rate * n) * 1e3:6.1f} us")
