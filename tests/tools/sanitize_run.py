"""A small workload for compute-sanitizer (one tool per run): the standalone
sampler with histograms, a desk-size and a paper-width (fused kernels)
training step, and two emulated ranks exchanging through the one-sided
windows (one-hop all-gather and pass-along ring).
  compute-sanitizer --tool memcheck python tests/tools/sanitize_run.py
  compute-sanitizer --tool racecheck python tests/tools/sanitize_run.py"""
import ctypes
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_2407_00051_b200 import _lib as L  # noqa: E402
from paper_2407_00051_b200 import runtime  # noqa: E402


def main():
    sp = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    # sampler
    k, m = 16, 100
    cs = torch.rand(k, 6, device="cuda") * 0.5 + 0.25
    ev = torch.empty(2 * k * m, dtype=torch.float32, device="cuda")
    hs = torch.zeros(2 * 66, dtype=torch.int32, device="cuda")
    L.sample_events(cs.data_ptr(), k, m, 1, 0, 0, 5, ev.data_ptr(), hs.data_ptr(), 64, (0.0, 0.0), (4.0, 4.0), sp)
    # steps: desk, paper widths (fused tcgen05 kernels, ragged tiles)
    for preset, kw in ((L.PRESET_DESK, {}), (L.PRESET_PAPER, dict(param_samples=8, events_per_sample=40))):
        ctx = runtime.make_context(L.config_init(preset, **kw))
        for t in range(2):
            ctx.train_step(t, 0, sp)
        torch.cuda.synchronize()
        ctx.close()
    # exchange: two emulated ranks, one stream each
    for mode in (L.MODE_RMA_ALLGATHER, L.MODE_RMA_ARAR_ARAR):
        ctxs, streams = [], []
        for r in range(2):
            st = torch.cuda.Stream()
            streams.append(st)
            with torch.cuda.stream(st):
                ctxs.append(runtime.make_context(L.config_init(L.PRESET_DESK, world=2, rank=r, mode=mode, group_size=2,
                                                               staleness=1, exchange_timeout_ms=60000)))
        ptrs = [c.window_ptr() for c in ctxs]
        for c in ctxs:
            c.connect_peers_local(ptrs)
        sps = [ctypes.c_void_p(s.cuda_stream) for s in streams]
        for t in range(3):
            for r in range(2):
                ctxs[r].train_step(t, L.STEP_LOCAL_ONLY, sps[r])
            for r in range(2):
                ctxs[r].push_generator_grad(t, sps[r])
            for r in range(2):
                ctxs[r].pull_generator_grad(t, sps[r])
        torch.cuda.synchronize()
        for c in ctxs:
            c.close()
    print("SANITIZE_RUN_OK")


if __name__ == "__main__":
    main()
