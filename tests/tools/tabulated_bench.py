"""Time the tabulated-CDF sampler variant (R32) at C2 size (k = 1024 parameter
samples, m = 1024 events each, G grid nodes): forward and backward, CUDA
events around 20 launches each, after 3 warm-up launches."""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_2407_00051_b200 import _lib as L  # noqa: E402

sp = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
k, m = 1024, 1024
raw = (torch.randn(k, 6, device="cuda") * 0.9).contiguous()
ev = torch.empty(k * m, 2, device="cuda")
dy = torch.randn(k * m, 2, device="cuda")
draw = torch.empty(k, 6, device="cuda")
out = {}
for G in (256, 1024, 2048):
    for name, fn in (("fwd", lambda i: L.sample_tabulated(raw.data_ptr(), k, m, G, 1, i, 0, 5, ev.data_ptr(), sp)),
                     ("bwd", lambda i: L.sample_tabulated_bwd(raw.data_ptr(), k, m, G, 1, i, 0, 5, dy.data_ptr(),
                                                              draw.data_ptr(), sp))):
        for i in range(3):
            fn(i)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(20):
            fn(i)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 20
        out[f"{name}_G{G}"] = {"ms": ms, "events_per_s": k * m / (ms * 1e-3)}
        print(f"G={G:5d} {name}: {ms * 1e3:8.1f} us  {k * m / (ms * 1e-3) / 1e9:6.2f} G events/s")
print(json.dumps({"workload": "k=1024 m=1024 (2^20 events)", "results": out}))
