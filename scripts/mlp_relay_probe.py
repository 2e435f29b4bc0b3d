"""a_ready path timing (globaltimer, ns): each epilogue warp's release of A(0)
in both CTAs of cluster 0, the peer relay's a_loc completion and the
leader's a_ready completion, per release index (1 + 8 per pair)."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2409_13418_b200 import MlpField, _lib  # noqa: E402
from paper_2409_13418_b200.pipeline import DeviceField  # noqa: E402

ctx = _lib.Context(0)
L = _lib.load()
L.odc_set_param(ctx.handle, b"mlp_impl", 3)
tr = np.zeros(1400, dtype=np.int64)
with DeviceField(ctx, MlpField()) as f:
    for _ in range(2):
        assert L.odc_profile_mlp(ctx.handle, f.handle, 4_000_000, tr.ctypes.data, len(tr)) == 0
rel0 = tr[800:800 + 8 * 24].reshape(8, 24)
rel1 = tr[1000:1000 + 8 * 24].reshape(8, 24)
loc = tr[700:724]
rdy = tr[750:774]
base = rdy[1]
print("idx  leader warps (max-min)   peer warps (max-min)   peer a_loc  leader a_ready   [ns rel. to leader's last warp]")
for i in range(2, 20):
    lm = rel0[:, i].max()
    print(f"{i:3d}  {rel0[:, i].max() - rel0[:, i].min():6d}                {rel1[:, i].max() - rel1[:, i].min():6d}"
          f"   peer_last {rel1[:, i].max() - lm:6d}  a_loc {loc[i] - lm:6d}  a_ready {rdy[i] - lm:6d}")
