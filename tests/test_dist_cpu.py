"""CPU (gloo) tests of the multi-rank host logic, world_size 2: the
rendezvous in paper_2407_00051_b200.runtime.connect exchanges every rank's
IPC handle in rank order and broadcasts rank 0's NCCL id, and the oracle's
multi-rank driver agrees with per-rank runs."""
import os
import tempfile

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


class FakeCtx:
    """Stands in for a library context: records what connect() hands it."""

    def __init__(self, rank):
        self.rank = rank
        self.peers = None
        self.uid = None

    def ipc_handle(self):
        return bytes([self.rank]) * 64

    def connect_peers(self, handles):
        self.peers = handles

    def connect_nccl(self, uid):
        self.uid = uid


def _worker(rank, world, path, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    dist.init_process_group("gloo", init_method=f"file://{path}", rank=rank, world_size=world)
    import paper_2407_00051_b200._lib as L
    from paper_2407_00051_b200 import runtime
    L.nccl_unique_id = lambda: b"ID-FROM-RANK-0".ljust(128, b"\0")  # no NCCL on the CPU box
    ctx = FakeCtx(rank)
    runtime.connect(ctx)
    q.put((rank, [h[0] for h in ctx.peers], ctx.uid[:14]))
    dist.destroy_process_group()


def test_connect_rendezvous_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "rdv")
        procs = [ctx.Process(target=_worker, args=(r, world, path, q)) for r in range(world)]
        for p in procs:
            p.start()
        res = sorted(q.get(timeout=120) for _ in range(world))
        for p in procs:
            p.join(timeout=60)
            assert p.exitcode == 0
    for rank, peers, uid in res:
        assert peers == [0, 1]            # handles gathered in rank order
        assert uid == b"ID-FROM-RANK-0"   # every rank got rank 0's id


def _oracle_worker(rank, world, path, q):
    """Each process runs the oracle for its own rank in a 2-rank ARAR ring,
    exchanging packets with gloo; the result must equal the lockstep driver."""
    import numpy as np
    dist.init_process_group("gloo", init_method=f"file://{path}", rank=rank, world_size=world)
    import torch
    from oracle import exchange as xc
    from oracle import gan
    cfg = gan.Config(world=world, group_size=world, mode=xc.MODE_ARAR, noise_dim=3, gen_hidden=8, disc_hidden=8,
                     param_samples=6, events_per_sample=5, reference_rows=60, shard_rows=30, seed=3)
    st = gan.RankState(cfg, rank)
    for t in range(3):
        o = gan.local_step(cfg, st, t)
        pk = torch.tensor(o["packet"])
        gathered = [torch.zeros_like(pk) for _ in range(world)]
        dist.all_gather(gathered, pk)
        R = xc.fold_ascending({r: gathered[r].numpy() for r in range(world)}, range(world)) / world
        gan.apply_generator(cfg, st, R, o["db_g"])
    q.put((rank, np.concatenate([w.reshape(-1) for w in st.gW])))
    dist.destroy_process_group()


def test_distributed_oracle_matches_lockstep_driver():
    import numpy as np
    from oracle import exchange as xc
    from oracle import gan
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "rdv")
        procs = [ctx.Process(target=_oracle_worker, args=(r, world, path, q)) for r in range(world)]
        for p in procs:
            p.start()
        res = dict(q.get(timeout=180) for _ in range(world))
        for p in procs:
            p.join(timeout=60)
            assert p.exitcode == 0
    cfg = gan.Config(world=world, group_size=world, mode=xc.MODE_ARAR, noise_dim=3, gen_hidden=8, disc_hidden=8,
                     param_samples=6, events_per_sample=5, reference_rows=60, shard_rows=30, seed=3)
    states, _ = gan.run(cfg, 3)
    for r in range(world):
        assert np.array_equal(res[r], np.concatenate([w.reshape(-1) for w in states[r].gW]))
