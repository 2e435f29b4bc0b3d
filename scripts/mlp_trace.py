"""Print the per-layer event timeline of the MLP kernel's CTA 0 (odc_profile_mlp)."""
import ctypes
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2409_13418_b200 import MlpField, _lib  # noqa: E402
from paper_2409_13418_b200.pipeline import DeviceField  # noqa: E402

impl = int(sys.argv[1]) if len(sys.argv) > 1 else 0
n = int(sys.argv[2]) if len(sys.argv) > 2 else 2_000_000
ctx = _lib.Context(0)
L = _lib.load()
L.odc_set_param(ctx.handle, b"mlp_impl", impl)
dbg = int(sys.argv[3]) if len(sys.argv) > 3 else 0
L.odc_set_param(ctx.handle, b"mlp_debug", dbg)
tr = np.zeros(256 * 4, dtype=np.int64)
field = MlpField()
if len(sys.argv) > 4 and sys.argv[4] == "zero":  # power experiment: all-zero weights
    field.weights = [np.zeros_like(w) for w in field.weights]
elif len(sys.argv) > 4 and sys.argv[4] == "tiny":  # weights scaled so activations stay tiny
    field.weights = [w * 1e-3 for w in field.weights]
with DeviceField(ctx, field) as f:
    for _ in range(2):
        rc = L.odc_profile_mlp(ctx.handle, f.handle, n, tr.ctypes.data, len(tr))
        assert rc == 0, L.odc_last_error(ctx.handle)
t = tr[:256].reshape(2, 8, 16).astype(np.float64)
base = t[0, 0, 0]
names = ["mma_start", "a0_ok", "wait_a1", "a1_ok", "iss_nh0", "iss_nh1", "e0_wait", "e1_wait", "e0_acc", "e1_acc",
         "e0_done", "e1_done", "w_full"]
print("tile layer " + " ".join(f"{x:>9s}" for x in names))
for ti in range(2):
    for l in range(8):
        row = [(t[ti, l, e] - base) if t[ti, l, e] else float("nan") for e in range(12)]
        row.append(t[ti, l, 12])
        if t[ti, l, 13]:
            row.append(t[ti, l, 13] - base)
            row.append(t[ti, l, 14] - base)  # cycles the MMA warp waited on weight stages in this layer (single-CTA kernel)
        print(f"{ti:4d} {l:5d} " + " ".join(f"{x:9.0f}" for x in row))
print(f"kernel {tr[-1] / 1e6:.3f} ms for {n} points")
if dbg & 64:
    sys.exit(0)
per = [t[0, l + 1, 0] - t[0, l, 0] for l in range(1, 6)]
print(f"debug={dbg}: mean layer period (layers 1-5) {np.mean(per):.0f} cycles; tile pair {t[1, 0, 0] - t[0, 0, 0]:.0f}")
