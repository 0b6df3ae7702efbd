"""Where the end-to-end (host-input) step time goes at C2: device-input
steps (eager / graph) vs sagips_train_step_host, waiting for every step or
one step in flight.  Each variant runs 40 steps, twice, interleaved; prints
the wall-clock ms per step and the GPU's own (CUDA events around the 40
steps) so that host-issue limits show as wall > GPU."""
import ctypes
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2407_00051_b200 import _lib as L  # noqa: E402
from paper_2407_00051_b200 import runtime  # noqa: E402


def main():
    timing = int(os.environ.get("PROBE_TIMING", "1"))
    cfg = L.config_init(L.PRESET_PAPER)
    cfg.phase_timing = timing
    ctx = runtime.make_context(cfg)
    cur = torch.cuda.current_stream()
    sp = ctypes.c_void_p(cur.cuda_stream)
    N = cfg.param_samples * cfg.events_per_sample
    st = {"step": 0}
    for _ in range(3):
        ctx.train_step(st["step"], 0, sp)
        st["step"] += 1
    torch.cuda.synchronize()
    noise_h = torch.randn(cfg.param_samples, cfg.noise_dim).pin_memory()
    real_h = torch.from_numpy(ctx.get(L.T_EVENTS).reshape(-1, 2)[:N].copy()).pin_memory()
    stats_h = [torch.empty(ctypes.sizeof(L.StepStats), dtype=torch.uint8).pin_memory() for _ in range(2)]
    done = [torch.cuda.Event(), torch.cuda.Event()]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    K = 40

    def run(name, fn, pipelined):
        for _ in range(3):
            fn(0)
            st["step"] += 1
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e0.record(cur)
        for i in range(K):
            fn(i)
            done[i & 1].record(cur)
            st["step"] += 1
            if pipelined:
                if i > 0:
                    done[(i - 1) & 1].synchronize()
            else:
                done[i & 1].synchronize()
        e1.record(cur)
        torch.cuda.synchronize()
        ms = (time.perf_counter() - t0) * 1e3 / K
        print(f"timing={timing} {name:30s} wall {ms:7.3f}  gpu {e0.elapsed_time(e1) / K:7.3f} ms/step", flush=True)

    dev = lambda i: ctx.train_step(st["step"], 0, sp)
    dev_g = lambda i: ctx.train_step(st["step"], L.STEP_GRAPH, sp)
    host = lambda i: ctx.train_step_host(st["step"], 0, noise_h.data_ptr(), real_h.data_ptr(),
                                         stats_h[i & 1].data_ptr(), sp)
    for rep in range(2):
        run("device eager, wait each", dev, False)
        run("device eager, pipelined", dev, True)
        run("device graph, pipelined", dev_g, True)
        run("host inputs, wait each", host, False)
        run("host inputs, pipelined", host, True)
    runtime.close(ctx)


if __name__ == "__main__":
    main()
