"""CTA-0 timeline of the CTA-pair N=256 evaluator (mlp_impl 3)."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2409_13418_b200 import MlpField, _lib  # noqa: E402
from paper_2409_13418_b200.pipeline import DeviceField  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2_000_000
ctx = _lib.Context(0)
L = _lib.load()
L.odc_set_param(ctx.handle, b"mlp_impl", 3)
L.odc_set_param(ctx.handle, b"mlp_debug", int(sys.argv[2]) if len(sys.argv) > 2 else 0)
tr = np.zeros(256 * 4, dtype=np.int64)
with DeviceField(ctx, MlpField()) as f:
    for _ in range(2):
        assert L.odc_profile_mlp(ctx.handle, f.handle, n, tr.ctypes.data, len(tr)) == 0
t = tr[:256].reshape(2, 8, 16).astype(np.float64)
base = t[0, 0, 0]
names = ["m0_wait", "m0_ok", "m1_wait", "m1_ok", "iss0", "iss1", "e0_wait", "e1_wait", "e0_ok", "e1_ok", "e0_rel",
         "e1_rel"]
print("pair layer " + " ".join(f"{x:>8s}" for x in names))
for ti in range(2):
    for l in range(8):
        row = [(t[ti, l, e] - base) if t[ti, l, e] else float("nan") for e in range(12)]
        print(f"{ti:4d} {l:5d} " + " ".join(f"{x:8.0f}" for x in row))
ww = tr[256:320].reshape(2, 8, 4)
print("weight waits [pair][layer][k]:", ww.tolist())
print("layer 7 head done (rel. e_ok):", [[t[i, 7, 12 + u] - t[i, 7, 8 + u] for u in range(2)] for i in range(2)],
      "released:", [[t[i, 7, 10 + u] - t[i, 7, 8 + u] for u in range(2)] for i in range(2)])
print("epilogue sched_get cycles per pair:", tr[320:328].tolist())
print("piece ends:", [[t[i, l, 14] - (t[i, l, 11]) for l in range(1, 7)] for i in range(2)])
per = [t[0, l + 1, 0] - t[0, l, 0] for l in range(1, 6)]
print(f"mean layer period {np.mean(per):.0f} cycles; pair {t[1, 0, 0] - t[0, 0, 0]:.0f}; kernel {tr[-1] / 1e6:.3f} ms")
