"""Standalone timing of the fused sampler (a4-a6) through the C ABI:
sagips_sample_events (fake rows + histograms) at 2^20 and 2^24 events, and
with / without histograms.  CUDA events over 50 launches after 5 warm-ups;
the 2^24 output (128 MiB) exceeds L2, the 2^20 one does not (reported as
such).  Prints one JSON line per case."""
import ctypes
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2407_00051_b200 import _lib as L  # noqa: E402


def main():
    sp = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    peaks = json.load(open(os.path.join(os.path.dirname(__file__), "..", "..", "MEASURED_PEAKS.json")))
    for n in (1 << 20, 1 << 24):
        k = 1024
        cs = torch.rand(k, 6, device="cuda") * 0.5 + 0.25
        ev = torch.empty(2 * n, dtype=torch.float32, device="cuda")
        hs = torch.zeros(2 * 66, dtype=torch.int32, device="cuda")
        for hist in (True, False):
            hp = hs.data_ptr() if hist else None
            for i in range(5):
                L.sample_events(cs.data_ptr(), k, n // k, 1, i, 0, 5, ev.data_ptr(), hp, 64, (0.0, 0.0), (4.0, 4.0), sp)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for i in range(50):
                L.sample_events(cs.data_ptr(), k, n // k, 1, i, 0, 5, ev.data_ptr(), hp, 64, (0.0, 0.0), (4.0, 4.0), sp)
            e1.record()
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) / 50 * 1e3
            gbs = 8 * n / (us * 1e-6) / 1e9
            print(json.dumps({"events": n, "hist": hist, "us": us, "GBps_written": gbs,
                              "frac_hbm": gbs / peaks["hbm_gbs"]}), flush=True)


if __name__ == "__main__":
    main()
