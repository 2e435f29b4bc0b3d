"""Per-CTA start/end (globaltimer) of one evaluator launch vs its CUDA-event
time: where the fixed per-launch cost goes."""
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
with DeviceField(ctx, MlpField()) as f:
    for n in (595_294, 2_381_176, 8_000_000):
        for dbg in (0, 128):
            L.odc_set_param(ctx.handle, b"mlp_debug", dbg)
            for rep in range(3):
                time.sleep(0.15)
                assert L.odc_profile_mlp(ctx.handle, f.handle, n, tr.ctypes.data, len(tr)) == 0
            nct = 2 * min(74, (n + 511) // 512)
            st = tr[400:400 + 2 * nct:2].astype(np.float64)
            en = tr[401:401 + 2 * nct:2].astype(np.float64)
            t0 = st.min()
            print(f"n={n:8d} dbg={dbg:3d} event {tr[-1] / 1e3:8.1f} us | starts spread {st.max() - t0:6.1f} ns"
                  f" | ends {np.percentile(en - t0, 0) / 1e3:7.1f} .. {np.percentile(en - t0, 50) / 1e3:7.1f} .. {(en.max() - t0) / 1e3:7.1f} us")
