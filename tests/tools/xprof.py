"""Kernel timeline of the exchange alone (push + pull + Adam(G)) on every
rank, from the CUDA activity trace of torch.profiler (CUPTI; not ncu, which
must not run multi-rank).  Diagnostic only.

    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tests/tools/xprof.py [--mode rma]
"""
import argparse
import ctypes
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
from paper_2407_00051_b200 import _lib as L  # noqa: E402
from paper_2407_00051_b200 import runtime  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--mode", default="rma")
p.add_argument("--iters", type=int, default=5)
args = p.parse_args()
rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
cfg = L.config_init(L.PRESET_PAPER)
cfg.world, cfg.rank, cfg.group_size = world, rank, world
cfg.mode = {"rma": L.MODE_RMA_ARAR_ARAR, "rma-ag": L.MODE_RMA_ALLGATHER, "arar": L.MODE_ARAR,
            "sync": L.MODE_SYNC_ALLREDUCE}[args.mode]
cfg.staleness = 0
ctx = runtime.make_context(cfg)
runtime.connect(ctx)
sp = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
step = 0
for _ in range(3):
    ctx.train_step(step, 0, sp)
    step += 1
torch.cuda.synchronize()
prof = torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA])
rows = []
for it in range(args.iters):
    ctx.train_step(step, L.STEP_LOCAL_ONLY, sp)
    torch.cuda.synchronize()
    dist.barrier()
    torch.cuda._sleep(200_000)
    if it == args.iters - 1:
        prof.start()
    ctx.push_generator_grad(step, sp)
    ctx.pull_generator_grad(step, sp)
    torch.cuda.synchronize()
    step += 1
prof.stop()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
evs.sort(key=lambda e: e.time_range.start)
t0 = evs[0].time_range.start if evs else 0
out = [f"rank {rank} mode {args.mode}: {len(evs)} device activities"]
for e in evs:
    out.append(f"  {e.time_range.start - t0:9.2f} us  dur {e.time_range.elapsed_us():8.2f} us  {e.name[:90]}")
allout = [None] * world
dist.all_gather_object(allout, "\n".join(out))
if rank == 0:
    print("\n".join(allout), flush=True)
dist.destroy_process_group()
