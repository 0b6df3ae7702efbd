"""Time sagips_sample_events at 2^20 and 2^24 events, with and without
histograms (CUDA events, 20 launches each)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_2407_00051_b200 import _lib as L  # noqa: E402

sp = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
for n in (1 << 20, 1 << 24):
    k = 1024
    cs = torch.rand(k, 6, device="cuda") * 0.5 + 0.25
    ev = torch.empty(2 * n, dtype=torch.float32, device="cuda")
    hs = torch.zeros(2 * 66, dtype=torch.int32, device="cuda")
    for with_hist in (True, False):
        hp = hs.data_ptr() if with_hist else None
        for _ in range(3):
            L.sample_events(cs.data_ptr(), k, n // k, 1, 0, 0, 5, ev.data_ptr(), hp, 64, (0.0, 0.0), (4.0, 4.0), sp)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(20):
            L.sample_events(cs.data_ptr(), k, n // k, 1, i, 0, 5, ev.data_ptr(), hp, 64, (0.0, 0.0), (4.0, 4.0), sp)
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / 20 * 1e-3
        print(f"n=2^{n.bit_length() - 1} hist={with_hist}: {t * 1e6:8.1f} us  {8 * n / t / 1e9:7.0f} GB/s")
