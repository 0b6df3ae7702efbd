"""Convergence of the asynchronous grouped ring vs the synchronous all-reduce
(BASELINE.json configs[4], C5: 2^24 events per rank, bf16 discriminator
GEMMs).  Run under torchrun, one process per GPU:

    python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 \\
        tests/tools/convergence.py --steps 400 --mode rma --group-size 2 --outer-every 10 --out gpurun_out/conv_rma.json

Every rank trains its own discriminator on its own bootstrap shard
and exchanges generator weight gradients in the given mode (Tab. III).  Rank
0 records, every --every steps, the losses of every rank (device stats) and
the generator's ensemble estimate of the constrained parameters: the mean of
c over the step's k parameter samples, averaged over ranks, compared with p*
(the loop-closure target, R3) as the normalised residual of Eq. 6
r = (c_mean - p*) / p*.  Diagnostic tool (not a parity test)."""
import argparse
import ctypes
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2407_00051_b200 import _lib as L  # noqa: E402
from paper_2407_00051_b200 import runtime  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--steps", type=int, default=400)
    p.add_argument("--every", type=int, default=10)
    p.add_argument("--mode", choices=["rma", "rma-ag", "rma-chunked", "arar", "arar-arar", "sync", "none"], default="rma")
    p.add_argument("--group-size", type=int, default=0)
    p.add_argument("--staleness", type=int, default=1)
    p.add_argument("--outer-every", type=int, default=10)
    p.add_argument("--events-per-sample", type=int, default=16384)
    p.add_argument("--precision", choices=["bf16", "fp32"], default="bf16")
    p.add_argument("--out", default="gpurun_out/convergence.json")
    a = p.parse_args()
    rank, world, local = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), \
        int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    modes = {"rma": L.MODE_RMA_ARAR_ARAR, "rma-ag": L.MODE_RMA_ALLGATHER, "rma-chunked": L.MODE_RMA_CHUNKED,
             "arar": L.MODE_ARAR, "arar-arar": L.MODE_ARAR_ARAR, "sync": L.MODE_SYNC_ALLREDUCE, "none": L.MODE_NONE}
    cfg = L.config_init(L.PRESET_PAPER)
    m = a.events_per_sample
    cfg.events_per_sample = m
    cfg.reference_rows = 2 * cfg.param_samples * m
    cfg.shard_rows = cfg.param_samples * m
    cfg.precision = L.PREC_BF16 if a.precision == "bf16" else L.PREC_FP32
    cfg.world, cfg.rank = world, rank
    cfg.mode = modes[a.mode] if world > 1 else L.MODE_NONE
    cfg.group_size = a.group_size if (a.group_size and world > 1) else world
    cfg.outer_every = a.outer_every
    cfg.staleness = a.staleness if (world > 1 and a.mode not in ("sync", "rma-chunked")) else 0
    ctx = runtime.make_context(cfg)
    if world > 1:
        runtime.connect(ctx)
    sp = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    p_star = np.array(list(cfg.true_params), dtype=np.float64)
    rec = []
    t0 = time.perf_counter()
    for t in range(a.steps):
        ctx.train_step(t, 0, sp)
        if (t + 1) % a.every == 0 or t == 0:
            s = ctx.get(L.T_STATS)
            c = ctx.get(L.T_C).reshape(-1, 6).astype(np.float64).mean(axis=0)
            row = torch.tensor([s.loss_d, s.loss_g] + list(c), dtype=torch.float64, device="cuda")
            if world > 1:
                allr = [torch.zeros_like(row) for _ in range(world)]
                dist.all_gather(allr, row)
                allr = torch.stack(allr).cpu().numpy()
            else:
                allr = row.cpu().numpy()[None]
            c_ens = allr[:, 2:].mean(axis=0)
            rec.append({"step": t + 1, "loss_d": allr[:, 0].tolist(), "loss_g": allr[:, 1].tolist(),
                        "c_mean": c_ens.tolist(), "residual": ((c_ens - p_star) / p_star).tolist()})
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    if rank == 0:
        out = {"mode": a.mode, "world": world, "group_size": cfg.group_size, "staleness": cfg.staleness,
               "outer_every": cfg.outer_every, "events_per_rank_per_step": cfg.param_samples * m,
               "precision": a.precision, "steps": a.steps, "wall_s": wall, "p_star": p_star.tolist(), "records": rec}
        os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
        with open(a.out, "w") as f:
            json.dump(out, f)
        last = rec[-1]
        print(f"{a.mode} world {world}: {a.steps} steps in {wall:.1f} s; final mean L_D {np.mean(last['loss_d']):.4f} "
              f"L_G {np.mean(last['loss_g']):.4f}; |r| mean {np.mean(np.abs(last['residual'])):.4f}")
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
