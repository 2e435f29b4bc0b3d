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
tr = np.zeros(256 * 4, dtype=np.int64)
with DeviceField(ctx, MlpField()) as f:
    for _ in range(2):
        rc = L.odc_profile_mlp(ctx.handle, f.handle, n, tr.ctypes.data, len(tr))
        assert rc == 0, L.odc_last_error(ctx.handle)
t = tr[:256].reshape(2, 8, 16).astype(np.float64)
base = t[0, 0, 0]
names = ["mma_start", "a0_ok", "wait_a1", "a1_ok", "iss_nh0", "iss_nh1", "e0_wait", "e1_wait", "e0_acc", "e1_acc",
         "e0_done", "e1_done"]
print("tile layer " + " ".join(f"{x:>9s}" for x in names))
for ti in range(2):
    for l in range(8):
        row = [(t[ti, l, e] - base) if t[ti, l, e] else float("nan") for e in range(12)]
        print(f"{ti:4d} {l:5d} " + " ".join(f"{x:9.0f}" for x in row))
