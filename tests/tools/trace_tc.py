"""Run one C2 step with SAGIPS_TRACE=1 and summarise the per-tile timeline of
each tensor-core layer launch (CTA 0): producer-done / MMA-start /
epilogue-start / epilogue-done intervals."""
import ctypes
import os
import sys

os.environ["SAGIPS_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2407_00051_b200 import _lib as L  # noqa: E402
from paper_2407_00051_b200 import runtime  # noqa: E402

cfg = L.config_init(L.PRESET_PAPER)
ctx = runtime.make_context(cfg)
sp = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
ctx.train_step(0, 0, sp)
L.debug_trace()  # discard warm-up
ctx.train_step(1, 0, sp)
tr = L.debug_trace().astype(np.int64)
names = ["fwd-first", "fwd-mid", "fwd-head", "bwd-L3", "bwd-L2", "bwd-L1", "G fwd-first", "G fwd-mid", "G fwd-head",
         "G bwd-L3", "G bwd-L2", "G bwd-dy"]
for li in range(12):
    t = tr[li, 0]
    n = int((t[:, 0] > 0).sum())
    if n < 3:
        continue
    t = t[:n]
    t0 = t[0, 0]
    prod = np.diff(t[:, 0]).mean()
    mma_wait = (t[:, 1] - t[:, 0]).mean()
    mma_to_epi = (t[:, 2] - t[:, 1]).mean()
    epi = (t[:, 3] - t[:, 2]).mean()
    print(f"{names[li]:12s} tiles {n:3d} span {(t[-1, 3] - t0) / 1e3:8.1f} us  per-tile producer {prod:7.0f} ns  "
          f"full->mma {mma_wait:7.0f}  mma->epi {mma_to_epi:7.0f}  epi {epi:7.0f}")
