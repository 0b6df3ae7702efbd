"""One sagips_sample_events launch at 2^24 events (with / without histograms),
for ncu: python tests/tools/sampler_once.py [hist|nohist]"""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2407_00051_b200 import _lib as L  # noqa: E402

sp = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
n, k = 1 << 24, 1024
cs = torch.rand(k, 6, device="cuda") * 0.5 + 0.25
ev = torch.empty(2 * n, dtype=torch.float32, device="cuda")
hs = torch.zeros(2 * 66, dtype=torch.int32, device="cuda")
hist = len(sys.argv) < 2 or sys.argv[1] == "hist"
for i in range(3):
    L.sample_events(cs.data_ptr(), k, n // k, 1, i, 0, 5, ev.data_ptr(), hs.data_ptr() if hist else None, 64,
                    (0.0, 0.0), (4.0, 4.0), sp)
torch.cuda.synchronize()
print("ok")
