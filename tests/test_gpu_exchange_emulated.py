"""The asynchronous ring exchange on ONE GPU: W ranks
emulated as W rank contexts of one process, their exchange windows wired by
raw device address (sagips_connect_peers_local; CUDA IPC cannot open a
handle in the process that exported it).  The kernels, tags and waits are
the ones a multi-GPU run uses -- only the peer addresses point into the same
HBM instead of a peer's over NVLink.

Every rank context has its own CUDA stream (as a rank process has), so a
waiting pull never blocks a peer's push or forwarding agent.  Per step t:
all contexts run the local step (LOCAL_ONLY), then all push(t), then all
pull(t) (wait + ascending fold + Adam(G)).

Checks per step and rank (Alg. 1, RMA P:192-194, grouping
P:207-228, weights-only packet P:305, fused packet P:306):
* bit-exact: the reduced packet equals oracle.exchange.reduce_step applied to
  the GPU contexts' own packets in fp32 (the exchange moves and folds fp32
  values in a fixed ascending order, R10, so nothing but the order of the
  additions is involved);
* a13: the generator weights and biases after the pull equal one oracle
  Adam(G) step (oracle.gan.apply_generator, fp64) from the context's
  pre-step generator state with that reduced packet, to fp32 rounding;
* against the independent oracle trajectory (every rank simulated from step
  0: oracle.gan local steps + reduce_step + apply_generator): generator
  weights within 2 lr per step, L_D within 2%.  (The reduced packets are not
  compared with the trajectory's elementwise: after the first Adam(D) step a
  near-zero D gradient of the other sign moves that weight by 2 lr, which the
  G-step gradients are sensitive to -- the single-step parity tests compare
  them through the GPU's own updated D, tests/test_gpu_parity.py.)
"""
import ctypes
import time

import numpy as np
import pytest

from oracle import exchange as xc
from oracle import gan
from tests.gpu_util import flat, lib, oracle_config, sync_params, unflat

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

MODES = {"rma": 3, "rma-ag": 5, "rma-chunked": 6}


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.init()


def _packet(ctx, L, fused):
    p = ctx.get(L.T_GEN_DW)
    return np.concatenate([p, ctx.get(L.T_GEN_DB)]) if fused else p


def make_world(mode, W, g, s, outer=0, fused=0, outer_rma=1, timeout_ms=20000, **kw):
    from paper_2407_00051_b200 import runtime
    L = lib()
    ctxs, streams = [], []
    for r in range(W):
        st = torch.cuda.Stream()
        streams.append(st)
        cfg = L.config_init(L.PRESET_DESK, world=W, rank=r, mode=MODES[mode], group_size=g, staleness=s,
                            outer_every=outer, seed=21, exchange_timeout_ms=timeout_ms, packet_biases=fused,
                            outer_rma=outer_rma, **kw)
        with torch.cuda.stream(st):
            ctxs.append(runtime.make_context(cfg))
    ptrs = [c.window_ptr() for c in ctxs]
    assert all(ptrs)
    for c, st in zip(ctxs, streams):
        c.connect_peers_local(ptrs)
        c.stream_keepalive = st  # the rank's stream lives as long as its context
    return ctxs, [ctypes.c_void_p(st.cuda_stream) for st in streams]


def _load_generator(st, ctx, L, ocfg):
    """The oracle rank's generator weights and Adam(G) moments := the GPU
    context's (fp32 values), so one apply_generator can be compared."""
    gW, gb = ctx.get(L.T_GEN_W), ctx.get(L.T_GEN_B)
    adam = ctx.get(L.T_GEN_ADAM)
    pw, pb = gW.size, gb.size
    st.gW, st.gb = unflat(gW, st.gW), unflat(gb, st.gb)
    st.g_mW, st.g_vW = unflat(adam[:pw], st.gW), unflat(adam[pw:2 * pw], st.gW)
    st.g_mb, st.g_vb = unflat(adam[2 * pw:2 * pw + pb], st.gb), unflat(adam[2 * pw + pb:], st.gb)


def run_emulated(mode, W, g, s, steps=6, outer=0, fused=0):
    L = lib()
    ctxs, sps = make_world(mode, W, g, s, outer, fused)
    ocfg = oracle_config(ctxs[0].cfg)
    states = [gan.RankState(ocfg, r) for r in range(W)]
    for r in range(W):
        sync_params(ctxs[r], states[r])
    apply_st = [gan.RankState(ocfg, r) for r in range(W)]  # one-step Adam(G) replicas
    hist_gpu, hist_ora = {}, {}
    failures = []
    for t in range(steps):
        for r in range(W):
            _load_generator(apply_st[r], ctxs[r], L, ocfg)
            apply_st[r].g_tau = t
            ctxs[r].train_step(t, L.STEP_LOCAL_ONLY, sps[r])
        hist_gpu[t] = [_packet(c, L, fused) for c in ctxs]          # syncs the device
        db_local = [ctxs[r].get(L.T_GEN_DB) for r in range(W)]
        for r in range(W):
            ctxs[r].push_generator_grad(t, sps[r])
        for r in range(W):
            ctxs[r].pull_generator_grad(t, sps[r])
        torch.cuda.synchronize()
        # a12 alone, bit-exact: reduce_step over the GPU contexts' own fp32 packets
        R_exact = xc.reduce_step(ocfg.mode, W, g, outer, s, ocfg.reduce_mean, t, hist_gpu)
        # the independent oracle trajectory (every rank simulated from step 0)
        outs = [gan.local_step(ocfg, states[r], t) for r in range(W)]
        hist_ora[t] = [o["packet"] for o in outs]
        R = xc.reduce_step(ocfg.mode, W, g, outer, s, ocfg.reduce_mean, t, hist_ora)
        for r in range(W):
            gan.apply_generator(ocfg, states[r], R[r], outs[r]["db_g"])
        for r in range(W):
            red = ctxs[r].get(L.T_REDUCED)
            exact = np.asarray(R_exact[r], dtype=np.float32)
            if not np.array_equal(red, exact):
                nb = int(np.sum(red != exact))
                failures.append(f"step {t} rank {r}: reduced differs from the fp32 fold of the GPU packets in {nb}")
            # a13 on the reduced packet: one oracle Adam(G) step from the GPU's
            # pre-step generator state with the same reduced packet
            gan.apply_generator(ocfg, apply_st[r], exact.astype(np.float64), unflat(db_local[r], apply_st[r].gb))
            for which, ref in ((L.T_GEN_W, flat(apply_st[r].gW)), (L.T_GEN_B, flat(apply_st[r].gb))):
                got = ctxs[r].get(which).astype(np.float64)
                bad = np.abs(got - ref) > 4e-7 * np.abs(ref) + 1e-3 * ocfg.gen_lr
                if bad.any():
                    failures.append(f"step {t} rank {r}: Adam(G) of the reduced packet off in {int(bad.sum())}")
            # the whole trajectory: weights within 2 lr per step of the oracle's
            dw = np.max(np.abs(ctxs[r].get(L.T_GEN_W) - flat(states[r].gW)))
            if fused:
                dw = max(dw, np.max(np.abs(ctxs[r].get(L.T_GEN_B) - flat(states[r].gb))))
            if dw > 2.0 * ocfg.gen_lr * (t + 1) + 1e-7:
                failures.append(f"step {t} rank {r}: generator weights {dw:.3g} from the oracle")
            st = ctxs[r].get(L.T_STATS)
            fires = bool(outer) and xc.outer_fires(t, outer) and r % g == 0 and (W + g - 1) // g > 1
            if st.outer_fired != int(fires):
                failures.append(f"step {t} rank {r}: outer_fired {st.outer_fired}, expected {int(fires)}")
            if abs(st.loss_d - outs[r]["loss_d"]) > 0.02 * abs(outs[r]["loss_d"]):
                failures.append(f"step {t} rank {r}: L_D {st.loss_d} vs oracle {outs[r]['loss_d']} (> 2%)")
    assert not failures, "\n".join(failures[:12])
    return ctxs


@pytest.mark.parametrize("mode", ["rma", "rma-ag"])
@pytest.mark.parametrize("W,g", [(2, 2), (4, 4), (8, 8), (8, 4), (8, 2)])
@pytest.mark.parametrize("s", [0, 1])
def test_emulated_exchange(mode, W, g, s):
    run_emulated(mode, W, g, s)


@pytest.mark.parametrize("W,g,outer", [(2, 2, 0), (4, 4, 0), (8, 8, 0), (8, 4, 0), (8, 2, 3), (6, 4, 2), (4, 4, 0)])
def test_emulated_chunked_ring(W, g, outer):
    """The chunked reduce-scatter + all-gather (SAGIPS_MODE_RMA_CHUNKED, the
    paper's future work P:180; staleness 0): member q folds chunk q of every
    packet in ascending origin order, so the reduced packets are bit-identical
    to the pass-along ring's (the oracle's reduce_step)."""
    run_emulated("rma-chunked", W, g, 0, outer=outer)


def test_emulated_chunked_fused_bias_packet():
    run_emulated("rma-chunked", 4, 4, 0, fused=1)


@pytest.mark.parametrize("mode", ["rma", "rma-ag"])
@pytest.mark.parametrize("s", [0, 1])
def test_emulated_fused_bias_packet(mode, s):
    """Tensor fusion: the packet is [weights | biases]."""
    run_emulated(mode, 4, 4, s, fused=1)


@pytest.mark.parametrize("mode,W,g,outer", [("rma", 8, 2, 2), ("rma-ag", 8, 4, 3), ("rma", 6, 4, 2),
                                             ("rma-ag", 5, 2, 1), ("rma", 4, 1, 2)])
@pytest.mark.parametrize("s", [0, 1])
def test_emulated_grouping_outer_ring(mode, W, g, outer, s):
    """Grouping: inner groups every step, the leaders' outer ring
    every h steps (one-sided, cfg.outer_rma); (6, 4) and (5, 2) have a smaller
    last group; g = 1 makes every rank a leader."""
    run_emulated(mode, W, g, s, outer=outer)


def test_writer_never_waits_for_a_slow_peer():
    """RMA: "a given rank does not have to wait for an other rank to
    finish its current task before gradients can be sent".  Rank 1's stream
    is held by a long device spin; rank 0's push(t) must complete (its stream
    drains) while rank 1 is still busy, and rank 0's pull completes as soon
    as rank 1 pushes."""
    L = lib()
    for mode in ("rma", "rma-ag"):
        ctxs, sps = make_world(mode, 2, 2, 0)
        s0 = torch.cuda.ExternalStream(sps[0].value)
        s1 = torch.cuda.ExternalStream(sps[1].value)
        for r in range(2):
            ctxs[r].train_step(0, L.STEP_LOCAL_ONLY, sps[r])
        torch.cuda.synchronize()
        with torch.cuda.stream(s1):
            torch.cuda._sleep(1_500_000_000)  # ~0.75 s of device time on rank 1's stream
        t0 = time.perf_counter()
        ctxs[0].push_generator_grad(0, sps[0])
        s0.synchronize()                        # rank 0's push completed ...
        t_push = time.perf_counter() - t0
        assert not s1.query(), "rank 1 should still be busy"  # ... while rank 1 still computes
        ctxs[1].push_generator_grad(0, sps[1])
        ctxs[0].pull_generator_grad(0, sps[0])
        ctxs[1].pull_generator_grad(0, sps[1])
        torch.cuda.synchronize()
        assert t_push < 0.5, f"{mode}: push waited {t_push:.3f} s for the busy peer"
        a, b = ctxs[0].get(L.T_REDUCED), ctxs[1].get(L.T_REDUCED)
        assert np.array_equal(a, b)  # s = 0, one group: both ranks fold the same packets in the same order


def test_timeout_skips_the_update_and_is_reported():
    """A pull whose peer never pushes times out (bounded wait); the step's
    fold and Adam(G) are skipped (the weights stay as they were) and the next
    call returns TIMEOUT without a device sync."""
    L = lib()
    ctxs, sps = make_world("rma-ag", 2, 2, 0, timeout_ms=200)
    ctxs[0].train_step(0, L.STEP_LOCAL_ONLY, sps[0])
    w0 = ctxs[0].get(L.T_GEN_W)
    ctxs[0].push_generator_grad(0, sps[0])
    ctxs[0].pull_generator_grad(0, sps[0])     # rank 1 never pushes
    torch.cuda.synchronize()
    with pytest.raises(L.SagipsError) as e:
        ctxs[0].train_step(1, 0, sps[0])
    assert e.value.status == 7  # TIMEOUT
    w1 = np.empty_like(w0)
    L.lib.sagips_get(ctxs[0].h, L.T_GEN_W, w1.ctypes.data, w1.nbytes)  # reports TIMEOUT too; copies first
    assert np.array_equal(w1, w0), "the generator must keep its weights when the exchange failed"


def test_overrun_slot_is_a_protocol_error():
    """A peer that runs more than the slot depth (4 versions) ahead
    overwrites the packet a slow rank still needs: the slow rank's wait sees
    a newer version in the slot (not a stale one), skips the fold and
    Adam(G), and the next call returns PROTOCOL."""
    L = lib()
    ctxs, sps = make_world("rma-ag", 2, 2, 0, timeout_ms=2000)
    for t in range(5):                          # rank 1: versions 0..4 (4 lands in version 0's slot)
        ctxs[1].train_step(t, L.STEP_LOCAL_ONLY, sps[1])
        ctxs[1].push_generator_grad(t, sps[1])
    torch.cuda.synchronize()
    ctxs[0].train_step(0, L.STEP_LOCAL_ONLY, sps[0])
    w0 = ctxs[0].get(L.T_GEN_W)
    ctxs[0].push_generator_grad(0, sps[0])
    ctxs[0].pull_generator_grad(0, sps[0])      # needs rank 1's version 0: overwritten
    torch.cuda.synchronize()
    with pytest.raises(L.SagipsError) as e:
        ctxs[0].train_step(1, 0, sps[0])
    assert e.value.status == 5  # PROTOCOL
    w1 = np.empty_like(w0)
    L.lib.sagips_get(ctxs[0].h, L.T_GEN_W, w1.ctypes.data, w1.nbytes)
    assert np.array_equal(w1, w0), "the generator must keep its weights when the exchange failed"
