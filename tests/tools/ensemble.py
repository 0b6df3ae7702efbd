"""Ensemble analysis vs training time (§8(f) rows 2 and 4; P:319-332,
P:391-453): every rank trains one GAN; at step 0 and every --every steps
(timestamped checkpoints) each rank predicts the constrained
parameters for one shared noise batch (sagips_predict_params), rank 0
gathers the M = world predictions and computes the ensemble response
(Eq. 7/8, averaged over the batch) and normalised residuals (Eq. 6)
with sagips_ensemble_stats.  Training time excludes the checkpoints.

Modes: --mode none = an ensemble of independent GANs (option (i), P:131;
--seed-per-rank gives each its own init and data draw); rma / arar (with
--group-size) = one distributed training whose per-rank generators are the
members.  --split-batch applies Eq. 10: param_samples =
floor(1024 / N(ranks)).  Run under torchrun, one process per GPU:

    python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 \\
        tests/tools/ensemble.py --mode none --seed-per-rank --steps 100000 --every 5000 \\
        --out gpurun_out/ensemble_none.json

Diagnostic tool (not a parity test)."""
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
    p.add_argument("--steps", type=int, default=20000)
    p.add_argument("--every", type=int, default=1000)
    p.add_argument("--mode", choices=["rma", "rma-ag", "arar", "arar-arar", "sync", "none"], default="none")
    p.add_argument("--group-size", type=int, default=0)
    p.add_argument("--outer-every", type=int, default=10)
    p.add_argument("--seed-per-rank", action="store_true")
    p.add_argument("--split-batch", action="store_true", help="Eq. 10: param_samples = 1024 // world")
    p.add_argument("--events-per-sample", type=int, default=100)  # Tab. IV
    p.add_argument("--k-eval", type=int, default=1024, help="noise vectors of the ensemble evaluation")
    p.add_argument("--sampler", choices=["quadratic", "tabulated"], default="quadratic")
    p.add_argument("--out", default="gpurun_out/ensemble.json")
    a = p.parse_args()
    rank, world, local = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), \
        int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    modes = {"rma": L.MODE_RMA_ARAR_ARAR, "rma-ag": L.MODE_RMA_ALLGATHER, "arar": L.MODE_ARAR, "arar-arar": L.MODE_ARAR_ARAR,
             "sync": L.MODE_SYNC_ALLREDUCE, "none": L.MODE_NONE}
    cfg = L.config_init(L.PRESET_PAPER)
    k = 1024 // world if a.split_batch else 1024  # Eq. 10
    cfg.param_samples = k
    cfg.events_per_sample = a.events_per_sample
    cfg.shard_rows = max(cfg.shard_rows, k * a.events_per_sample)
    cfg.reference_rows = max(cfg.reference_rows, 2 * cfg.shard_rows)
    cfg.world, cfg.rank = world, rank
    cfg.mode = modes[a.mode] if world > 1 else L.MODE_NONE
    cfg.group_size = a.group_size if (a.group_size and world > 1) else world
    cfg.outer_every = a.outer_every
    cfg.staleness = 1 if (world > 1 and a.mode not in ("sync", "none")) else 0
    if a.seed_per_rank:
        cfg.seed = cfg.seed + 7919 * rank
    if a.sampler == "tabulated":  # R32: true (w, b, c) per observable, histograms on [0, 1]
        cfg.sampler, cfg.sampler_grid = L.SAMPLER_TABULATED, 1024
        for j, v in enumerate((0.3, 2.0, 1.2, 0.7, 1.5, 3.0)):
            cfg.true_params[j] = v
        for o in range(2):
            cfg.hist_lo[o], cfg.hist_hi[o] = 0.0, 1.0
    ctx = runtime.make_context(cfg)
    if world > 1 and cfg.mode != L.MODE_NONE:
        runtime.connect(ctx)
    sp = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    p_star = np.array(list(cfg.true_params), dtype=np.float64)
    k_eval = min(a.k_eval, k)
    gen = torch.Generator().manual_seed(20240629)  # the same evaluation noise on every rank
    noise = torch.randn(k_eval, cfg.noise_dim, generator=gen).cuda()
    c_out = torch.empty(k_eval, 6, device="cuda")
    gathered = torch.empty(world, k_eval, 6, device="cuda") if rank == 0 else None
    rec = []
    train_s = 0.0

    def checkpoint(step):
        ctx.predict_params(noise.data_ptr(), k_eval, c_out.data_ptr(), sp)
        if world > 1:
            parts = list(gathered.unbind(0)) if rank == 0 else None
            dist.gather(c_out, parts, dst=0)
        elif rank == 0:
            gathered[0].copy_(c_out)
        if rank == 0:
            p_hat, sigma, r_hat = L.ensemble_stats(gathered.data_ptr(), world, k_eval, 6, p_star, sp)
            s = ctx.get(L.T_STATS)
            rec.append({"step": step, "train_s": train_s, "p_hat": p_hat.tolist(), "sigma": sigma.tolist(),
                        "r_hat": r_hat.tolist(), "r_mean": float(np.mean(r_hat)),
                        "r_abs_mean": float(np.mean(np.abs(r_hat))),
                        "r_sigma_mean": float(np.mean(sigma / np.abs(p_star))),  # sigma of r_hat, averaged
                        "loss_d": float(s.loss_d), "loss_g": float(s.loss_g)})

    checkpoint(0)
    t = 0
    while t < a.steps:
        n = min(a.every, a.steps - t)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(n):
            ctx.train_step(t, 0, sp)
            t += 1
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        train_s += time.perf_counter() - t0
        checkpoint(t)
    if rank == 0:
        out = {"mode": a.mode, "sampler": a.sampler, "world": world, "group_size": cfg.group_size, "split_batch": a.split_batch,
               "param_samples": k, "events_per_sample": a.events_per_sample, "k_eval": k_eval,
               "seed_per_rank": a.seed_per_rank, "steps": a.steps, "every": a.every, "p_star": p_star.tolist(),
               "train_s": train_s, "records": rec}
        os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
        with open(a.out, "w") as f:
            json.dump(out, f)
        first, last = rec[0], rec[-1]
        print(f"{a.mode} world {world} k {k} ({'split' if a.split_batch else 'full'} batch): {a.steps} steps, "
              f"{train_s:.1f} s training; |r_hat| mean {first['r_abs_mean']:.4f} -> {last['r_abs_mean']:.4f}, "
              f"sigma/p mean {first['r_sigma_mean']:.4f} -> {last['r_sigma_mean']:.4f}")
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
