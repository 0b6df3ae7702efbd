"""Run one C2 step with SAGIPS_TRACE=1 and summarise the per-tile timeline of
each tensor-core layer launch (CTA 0): producer-done / MMA-start /
epilogue-start / epilogue-done intervals, and the per-CTA wait times per role
(summed over the timed threads: the loader / MMA threads, lane 0 of each
producer / epilogue warp)."""
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
tr, ctas = L.debug_trace(with_ctas=True)
tr = tr.astype(np.int64)
ctas = ctas.astype(np.int64)
# launch order of the traced tensor-core layer kernels (k_tc_layers.cu): with the
# fused kernels (default) only the D step's three backward passes; with
# SAGIPS_FUSED=0 all twelve layer passes
if os.environ.get("SAGIPS_FUSED", "1") != "0":
    names = ["d_bwd_last", "d_bwd_mid", "d_bwd_first"]
else:
    names = ["fwd-first", "fwd-mid", "fwd-head", "bwd-L3", "bwd-L2", "bwd-L1", "G fwd-first", "G fwd-mid",
             "G fwd-head", "G bwd-L3", "G bwd-L2", "G bwd-dy"]
g0 = min(int(tr[li, 0][tr[li, 0][:, 0] > 0, 0].min()) for li in range(len(names)) if (tr[li, 0][:, 0] > 0).sum() >= 3)
for li in range(len(names)):
    t = tr[li, 0]
    n = int((t[:, 0] > 0).sum())
    if n < 3:
        continue
    t = t[:n]
    t0 = t[0, 0]
    prod = np.diff(t[:, 0]).mean()
    period = np.diff(t[:, 3]).mean()
    mma_wait = (t[:, 1] - t[:, 0]).mean()
    mma_to_epi = (t[:, 2] - t[:, 1]).mean()
    epi = (t[:, 3] - t[:, 2]).mean()
    print(f"{names[li]:12s} tiles {n:3d} start {(t0 - g0) / 1e3:7.1f} us span {(t[-1, 3] - t0) / 1e3:8.1f} us  "
          f"period {period:6.0f} ns  staged {prod:6.0f}  staged->mma {mma_wait:6.0f}  mma->epi {mma_to_epi:6.0f}  "
          f"epi {epi:6.0f}")
    c = ctas[li]
    c = c[c[:, 0] > 0]
    if len(c):
        st, en = c[:, 0], c[:, 1]
        print(f"{'':12s} CTAs {len(c)}: start spread {(st.max() - st.min()) / 1e3:6.1f} us, end spread "
              f"{(en.max() - en.min()) / 1e3:6.1f} us, first start -> first tile {(t0 - st.min()) / 1e3:6.1f} us, "
              f"kernel {(en.max() - st.min()) / 1e3:7.1f} us, CTA0 last tile -> last CTA end {(en.max() - t[-1, 3]) / 1e3:6.1f} us")
        # summed waits per CTA (mean over CTAs; one timed thread per role / warp)
        wn = {1: "loader-slot", 2: "mma-operands", 3: "mma-acc", 4: "producer-slot", 5: "epi-acc(warp0..)",
              6: "mask-flag", 7: "epi-X"}
        w = c[:, 4:12].mean(axis=0) / 1e3
        print(f"{'':12s} waits (us per CTA): " + ", ".join(f"{wn[k]} {w[k]:.0f}" for k in wn if w[k] > 0.5))
        # the slowest CTAs: end time after the first start, with their SM id (bwd launches record it)
        idx = np.argsort(en)[::-1][:12]
        print(f"{'':12s} slowest CTAs (end us, sm): " + ", ".join(f"{(en[k] - st.min()) / 1e3:.0f}/{c[k, 2]}" for k in idx))
        q = np.percentile((en - st.min()) / 1e3, [0, 10, 50, 90, 100])
        print(f"{'':12s} CTA end percentiles (us): " + " ".join(f"{v:.0f}" for v in q))

