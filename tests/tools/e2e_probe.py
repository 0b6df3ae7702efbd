"""Where the end-to-end (host-input) step time goes at C2: device-input
steps vs sagips_train_step_host, with and without waiting for every step,
phase timing on and off.  Prints one line per variant (ms per step, wall
clock over 20 steps after 3 warm-ups)."""
import ctypes
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2407_00051_b200 import _lib as L  # noqa: E402
from paper_2407_00051_b200 import runtime  # noqa: E402


def main():
    for timing in (1, 0):
        cfg = L.config_init(L.PRESET_PAPER)
        cfg.phase_timing = timing
        ctx = runtime.make_context(cfg)
        cur = torch.cuda.current_stream()
        sp = ctypes.c_void_p(cur.cuda_stream)
        N = cfg.param_samples * cfg.events_per_sample
        step = 0
        for _ in range(3):
            ctx.train_step(step, 0, sp)
            step += 1
        torch.cuda.synchronize()
        noise_h = torch.randn(cfg.param_samples, cfg.noise_dim).pin_memory()
        real_h = torch.from_numpy(ctx.get(L.T_EVENTS).reshape(-1, 2)[:N].copy()).pin_memory()
        stats_h = [torch.empty(ctypes.sizeof(L.StepStats), dtype=torch.uint8).pin_memory() for _ in range(2)]
        done = [torch.cuda.Event(), torch.cuda.Event()]

        def run(name, fn, pipelined):
            nonlocal step
            for _ in range(3):
                fn(0)
                step += 1
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for i in range(20):
                fn(i)
                done[i & 1].record(cur)
                step += 1
                if pipelined:
                    if i > 0:
                        done[(i - 1) & 1].synchronize()
                else:
                    done[i & 1].synchronize()
            torch.cuda.synchronize()
            ms = (time.perf_counter() - t0) * 1e3 / 20
            print(f"timing={timing} {name:34s} {ms:7.3f} ms/step", flush=True)

        dev = lambda i: ctx.train_step(step, 0, sp)
        dev_g = lambda i: ctx.train_step(step, L.STEP_GRAPH, sp)
        host = lambda i: ctx.train_step_host(step, 0, noise_h.data_ptr(), real_h.data_ptr(), stats_h[i & 1].data_ptr(), sp)
        host_n = lambda i: ctx.train_step_host(step, 0, noise_h.data_ptr(), None, stats_h[i & 1].data_ptr(), sp)
        run("device, wait each", dev, False)
        run("device, pipelined", dev, True)
        run("device graph, pipelined", dev_g, True)
        run("host noise+real, wait each", host, False)
        run("host noise+real, pipelined", host, True)
        run("host noise only, pipelined", host_n, True)
        runtime.close(ctx)


if __name__ == "__main__":
    main()
