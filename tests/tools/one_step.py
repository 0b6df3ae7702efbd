"""One training step at a chosen size (debugging aid): python one_step.py [k] [m]"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_2407_00051_b200 import _lib as L  # noqa: E402
from paper_2407_00051_b200 import runtime  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 256
m = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
cfg = L.config_init(L.PRESET_PAPER, param_samples=k, events_per_sample=m, reference_rows=2 * k * m, shard_rows=k * m)
ctx = runtime.make_context(cfg)
sp = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
for t in range(2):
    ctx.train_step(t, 0, sp)
torch.cuda.synchronize()
s = ctx.get(L.T_STATS)
print("ok", s.loss_d, s.loss_g)
