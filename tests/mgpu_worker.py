"""torchrun worker for the multi-GPU exchange parity test (tests/test_gpu_multi.py).

Every rank runs the library step on its own GPU; every rank also runs the
oracle's lockstep simulation of all ranks (desk preset, seconds) and checks,
after every step, its own reduced packet and generator weights against the
oracle (exchange).  Exit code 0 = parity held on this rank.

usage: torchrun --nproc-per-node N tests/mgpu_worker.py MODE GROUP STALENESS STEPS [OUTER_EVERY [PACKET_BIASES [GRAPH]]]
"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from oracle import exchange as xc  # noqa: E402
from oracle import gan  # noqa: E402
from tests.gpu_util import flat, grad_close, oracle_config, sync_params  # noqa: E402

MODES = {"none": 0, "arar": 1, "arar-arar": 2, "rma": 3, "sync": 4, "rma-ag": 5, "rma-chunked": 6}


def main():
    mode_name, group, stale, steps = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
    outer = int(sys.argv[5]) if len(sys.argv) > 5 else 0
    fused = int(sys.argv[6]) if len(sys.argv) > 6 else 0  # packet_biases
    graph = int(sys.argv[7]) if len(sys.argv) > 7 else 0  # CUDA-graph steps (SAGIPS_STEP_GRAPH)
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2407_00051_b200 import _lib as L
    from paper_2407_00051_b200 import runtime
    cfg = L.config_init(L.PRESET_DESK, world=world, rank=rank, mode=MODES[mode_name], group_size=group,
                        staleness=stale, outer_every=outer, seed=21, exchange_timeout_ms=20000, packet_biases=fused)
    ctx = runtime.make_context(cfg)
    runtime.connect(ctx)
    ocfg = oracle_config(cfg)
    states = [gan.RankState(ocfg, r) for r in range(world)]
    sync_params(ctx, states[rank])
    for r in range(world):  # every rank rounds its oracle replicas the same way
        if r != rank:
            for name in ("gW", "gb", "dW", "db"):
                setattr(states[r], name, [np.asarray(w, dtype=np.float32).astype(np.float64) for w in getattr(states[r], name)])
    sp = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    history = {}
    ok = True
    for t in range(steps):
        ctx.train_step(t, L.STEP_GRAPH if graph else 0, sp)
        outs = [gan.local_step(ocfg, states[r], t) for r in range(world)]
        history[t] = [o["packet"] for o in outs]
        R = xc.reduce_step(ocfg.mode, world, group, outer, stale, ocfg.reduce_mean, t, history)
        for r in range(world):
            gan.apply_generator(ocfg, states[r], R[r], outs[r]["db_g"])
        red = ctx.get(L.T_REDUCED)
        good, nbad, worst = grad_close(red, R[rank], 1e-3)
        # weights: within 2 lr per step of the oracle (Adam sign flips on tiny grads)
        dw = np.max(np.abs(ctx.get(L.T_GEN_W) - flat(states[rank].gW)))
        if fused:  # the biases follow the reduced bias gradients
            dw = max(dw, np.max(np.abs(ctx.get(L.T_GEN_B) - flat(states[rank].gb))))
        if not good or dw > 2.0 * ocfg.gen_lr * (t + 1) + 1e-7:
            print(f"rank {rank} step {t} mode {mode_name}: reduced {nbad} bad (worst {worst:.3g}), |dW| {dw:.3g}",
                  flush=True)
            ok = False
        s = ctx.get(L.T_STATS)
        if outer and xc.outer_fires(t, outer) and rank % group == 0 and world // group > 1 and s.outer_fired != 1:
            print(f"rank {rank} step {t}: outer ring did not fire", flush=True)
            ok = False
    # replica invariant (mode ARAR / sync, s = 0): generator weights identical across ranks
    if mode_name in ("arar", "sync", "rma", "rma-ag", "rma-chunked", "arar-arar") and stale == 0 and group == world and not outer:
        w = torch.tensor(ctx.get(L.T_GEN_W), device="cuda")
        w0 = w.clone()
        dist.broadcast(w0, 0)
        if mode_name != "sync" and not torch.equal(w, w0):
            print(f"rank {rank}: generator weights differ from rank 0 under a synchronous ring", flush=True)
            ok = False
    flag = torch.tensor([0 if ok else 1], device="cuda")
    dist.all_reduce(flag)
    if rank == 0:
        print("MGPU_OK" if flag.item() == 0 else "MGPU_FAIL", mode_name, group, stale, flush=True)
    dist.destroy_process_group()
    return 0 if flag.item() == 0 else 1


if __name__ == "__main__":
    sys.exit(main())
