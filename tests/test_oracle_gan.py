"""Pins for oracle/gan.py: the whole step against PyTorch CPU autograd (an
independent library differentiation of the same forward definition) and
against central finite differences; replica / grouping invariants over
several steps."""
import copy
import time

import numpy as np
import pytest
import torch
import torch.nn.functional as F

from oracle import exchange as xc
from oracle import gan, mlp, proxy


def tiny_config(**kw):
    base = dict(noise_dim=3, gen_hidden=8, gen_depth=2, disc_hidden=8, disc_depth=2,
                param_samples=6, events_per_sample=5, reference_rows=60, shard_rows=30, seed=3)
    base.update(kw)
    return gan.Config(**base)


def _torch_mlp(Ws, bs, x):
    h = x
    for l in range(len(Ws)):
        h = F.linear(h, Ws[l], bs[l])
        if l < len(Ws) - 1:
            h = F.leaky_relu(h, 0.01)
    return h


def test_full_step_matches_torch_autograd():
    cfg = tiny_config()
    st = gan.RankState(cfg, 0)
    d_before = ([w.copy() for w in st.dW], [b.copy() for b in st.db])
    out = gan.local_step(cfg, st, 0)
    N = cfg.n_events
    # D step: loss on [x; y] with the D parameters before the update
    tW = [torch.tensor(w, requires_grad=True) for w in d_before[0]]
    tb = [torch.tensor(b, requires_grad=True) for b in d_before[1]]
    X = torch.tensor(np.concatenate([out["x"], out["y"]]))
    lab = torch.cat([torch.ones(N, dtype=torch.float64), torch.zeros(N, dtype=torch.float64)])
    ld = F.binary_cross_entropy_with_logits(_torch_mlp(tW, tb, X)[:, 0], lab)
    ld.backward()
    assert ld.item() == pytest.approx(out["loss_d"], rel=1e-13)
    for l in range(len(tW)):
        assert np.allclose(tW[l].grad.numpy(), out["dW_d"][l], rtol=1e-11, atol=1e-14)
        assert np.allclose(tb[l].grad.numpy(), out["db_d"][l], rtol=1e-11, atol=1e-14)
    # G step: generator -> softplus(threshold 20) -> quantile -> updated D -> loss
    gW = [torch.tensor(w, requires_grad=True) for w in gan.RankState(cfg, 0).gW]
    gb = [torch.tensor(b, requires_grad=True) for b in gan.RankState(cfg, 0).gb]
    raw = _torch_mlp(gW, gb, torch.tensor(out["z"])).reshape(-1, 2, 3)
    c0 = raw[:, :, 0]
    c1 = F.softplus(raw[:, :, 1], beta=1, threshold=20)
    c2 = F.softplus(raw[:, :, 2], beta=1, threshold=20)
    u = torch.tensor(out["u"])
    s = torch.arange(N) // cfg.events_per_sample
    y = c0[s] + c1[s] * u + c2[s] * u * u
    assert np.allclose(y.detach().numpy(), out["y"], rtol=1e-14, atol=1e-14)
    dW = [torch.tensor(w) for w in st.dW]
    db = [torch.tensor(b) for b in st.db]
    lg = F.binary_cross_entropy_with_logits(_torch_mlp(dW, db, y)[:, 0], torch.ones(N, dtype=torch.float64))
    lg.backward()
    assert lg.item() == pytest.approx(out["loss_g"], rel=1e-13)
    for l in range(len(gW)):
        assert np.allclose(gW[l].grad.numpy(), out["dW_g"][l], rtol=1e-10, atol=1e-15)
        assert np.allclose(gb[l].grad.numpy(), out["db_g"][l], rtol=1e-10, atol=1e-15)


def test_generator_gradient_finite_differences():
    cfg = tiny_config(seed=8)
    st0 = gan.RankState(cfg, 0)
    st = copy.deepcopy(st0)
    out = gan.local_step(cfg, st, 0)
    dW_upd = [w.copy() for w in st.dW]
    db_upd = [b.copy() for b in st.db]
    z, u, N, m = out["z"], out["u"], cfg.n_events, cfg.events_per_sample

    def lg(gW):
        raw, _ = mlp.forward(gW, st0.gb, z)
        y = proxy.sample_events(proxy.constrain(raw), m, u)
        zz, _ = mlp.forward(dW_upd, db_upd, y)
        return mlp.bce_with_logits(zz[:, 0], np.ones(N))

    rng = np.random.default_rng(0)
    h = 1e-6
    for l in range(len(st0.gW)):
        for _ in range(6):
            idx = tuple(rng.integers(0, d) for d in st0.gW[l].shape)
            Wp = [w.copy() for w in st0.gW]; Wp[l][idx] += h
            Wm = [w.copy() for w in st0.gW]; Wm[l][idx] -= h
            fd = (lg(Wp) - lg(Wm)) / (2 * h)
            assert abs(fd - out["dW_g"][l][idx]) <= 1e-9 + 1e-5 * abs(fd)


def test_packet_layout_weights_only():
    cfg = tiny_config()
    out = gan.local_step(cfg, gan.RankState(cfg, 0), 0)
    assert out["packet"].size == mlp.count_weights(cfg.gen_sizes())
    assert np.array_equal(out["packet"][:out["dW_g"][0].size], out["dW_g"][0].reshape(-1))


def test_fused_packet_carries_the_biases_and_syncs_them():
    # P:306 tensor fusion: the packet is [weights | biases]; under a
    # synchronous ring the replicas then agree in the biases too (with the
    # paper's weights-only packet they diverge through the local bias grads)
    cfg = tiny_config(packet_biases=1)
    out = gan.local_step(cfg, gan.RankState(cfg, 0), 0)
    nw, nb = mlp.count_weights(cfg.gen_sizes()), sum(b.size for b in out["db_g"])
    assert out["packet"].size == nw + nb
    np.testing.assert_array_equal(out["packet"][nw:], np.concatenate([b.reshape(-1) for b in out["db_g"]]))
    for fused in (0, 1):
        cfgw = tiny_config(world=2, group_size=2, mode=xc.MODE_ARAR, staleness=0, packet_biases=fused)
        states, _ = gan.run(cfgw, 3)
        same_b = all(np.array_equal(states[1].gb[l], states[0].gb[l]) for l in range(len(states[0].gb)))
        assert same_b == bool(fused)
        assert all(np.array_equal(states[1].gW[l], states[0].gW[l]) for l in range(len(states[0].gW)))


def test_step_basic_properties():
    cfg = tiny_config()
    out = gan.local_step(cfg, gan.RankState(cfg, 1), 4)
    assert out["x"].shape == out["y"].shape == (cfg.n_events, 2)   # equal batch sizes
    assert out["loss_d"] > 0 and out["loss_g"] > 0
    assert out["hist"][0].sum() == 2 * cfg.n_events and out["hist"][1].sum() == 2 * cfg.n_events


def test_replicas_identical_in_W_under_sync_ring():
    cfg = tiny_config(world=4, group_size=4, mode=xc.MODE_ARAR, staleness=0)
    states, _ = gan.run(cfg, 4)
    for r in range(1, 4):
        for l in range(len(states[0].gW)):
            assert np.array_equal(states[r].gW[l], states[0].gW[l])
        assert not np.array_equal(states[r].dW[0], states[0].dW[0])   # private discriminators


def test_grouped_non_leaders_identical():
    cfg = tiny_config(world=4, group_size=2, outer_every=2, mode=xc.MODE_RMA_ARAR_ARAR)
    states, _ = gan.run(cfg, 3)
    # groups {0,1}, {2,3}; leaders diverge only via outer fires, non-leaders
    # hold their group's inner result -> ranks 1 and 3 differ (different groups)
    assert not np.array_equal(states[1].gW[0], states[3].gW[0])


def test_group_size_one_equals_independent_runs():
    cfg = tiny_config(world=3, group_size=1, mode=xc.MODE_ARAR_ARAR, outer_every=0)
    states, _ = gan.run(cfg, 3)
    for r in range(3):
        solo = tiny_config(world=1, group_size=1, mode=xc.MODE_NONE)
        st = gan.RankState(solo, r)
        for t in range(3):
            o = gan.local_step(solo, st, t)
            gan.apply_generator(solo, st, o["packet"], o["db_g"])
        for l in range(len(st.gW)):
            assert np.array_equal(st.gW[l], states[r].gW[l])


def test_desk_config_runs_in_seconds():
    cfg = gan.desk_config()
    t0 = time.time()
    _, log = gan.run(cfg, 5)
    assert time.time() - t0 < 30
    assert all(np.isfinite(e["loss_d"][0]) and np.isfinite(e["loss_g"][0]) for e in log)


def test_trajectory_matches_torch_autograd_and_adam():
    """Multi-step pin of the training loop (S:Alg. GAN step, P:305 Adam(G)):
    T steps of the oracle at N=1 against the same loop written with PyTorch
    autograd and torch.optim.Adam (library routines), fed the same seeded
    draws (noise, uniforms, real-row indices).  Learning rates raised so the
    parameters move by O(1e-2) per step and a wrong Adam moment carry-over,
    bias-correction index or D-before-G ordering shows up."""
    cfg = tiny_config(seed=5, gen_lr=1e-2, disc_lr=1e-2)
    st = gan.RankState(cfg, 0)
    init = copy.deepcopy(st)
    T = 5
    _, log = gan.run(cfg, T, states=[st])
    N, m = cfg.n_events, cfg.events_per_sample
    gW = [torch.tensor(w, requires_grad=True) for w in init.gW]
    gb = [torch.tensor(b, requires_grad=True) for b in init.gb]
    dW = [torch.tensor(w, requires_grad=True) for w in init.dW]
    db = [torch.tensor(b, requires_grad=True) for b in init.db]
    optG = torch.optim.Adam(gW + gb, lr=cfg.gen_lr, betas=(0.9, 0.999), eps=1e-8)
    optD = torch.optim.Adam(dW + db, lr=cfg.disc_lr, betas=(0.9, 0.999), eps=1e-8)
    s = torch.arange(N) // m
    lab = torch.cat([torch.ones(N, dtype=torch.float64), torch.zeros(N, dtype=torch.float64)])
    for t in range(T):
        z = torch.tensor(gan.noise(cfg, t, 0))
        u = torch.tensor(proxy.fake_uniforms(cfg.seed, t, 0, N))
        x = torch.tensor(init.shard[proxy.real_indices(cfg.seed, t, 0, cfg.shard_rows, N)])
        raw = _torch_mlp(gW, gb, z).reshape(-1, 2, 3)
        c0 = raw[:, :, 0]
        c1 = F.softplus(raw[:, :, 1], beta=1, threshold=20)
        c2 = F.softplus(raw[:, :, 2], beta=1, threshold=20)
        y = c0[s] + c1[s] * u + c2[s] * u * u
        optD.zero_grad()
        ld = F.binary_cross_entropy_with_logits(_torch_mlp(dW, db, torch.cat([x, y.detach()]))[:, 0], lab)
        ld.backward()
        optD.step()
        optG.zero_grad()
        lg = F.binary_cross_entropy_with_logits(_torch_mlp(dW, db, y)[:, 0], torch.ones(N, dtype=torch.float64))
        lg.backward()
        optG.step()
        assert ld.item() == pytest.approx(log[t]["loss_d"][0], rel=1e-10)
        assert lg.item() == pytest.approx(log[t]["loss_g"][0], rel=1e-10)
    for a, b in zip(gW + gb + dW + db, st.gW + st.gb + st.dW + st.db):
        assert np.allclose(a.detach().numpy(), b, rtol=1e-9, atol=1e-12)
    # the loop moved the parameters (the pin is not vacuous)
    assert max(np.abs(a - b).max() for a, b in zip(st.gW, init.gW)) > 1e-3


@pytest.mark.parametrize("mode,staleness,W,gs,h", [(xc.MODE_SYNC_ALLREDUCE, 0, 2, 2, 0),
                                                   (xc.MODE_ARAR, 0, 2, 2, 0),
                                                   (xc.MODE_RMA_ARAR_ARAR, 1, 2, 2, 0),
                                                   (xc.MODE_RMA_ARAR_ARAR, 1, 4, 2, 2),
                                                   (xc.MODE_ARAR_ARAR, 0, 5, 2, 3)])
def test_multi_rank_trajectory_matches_torch_loop(mode, staleness, W, gs, h):
    """Multi-rank pin: two ranks, each its own
    D and shard; after every step rank r's generator weight gradient is
    replaced by (g_r(t) + sum_{o != r} g_o(t - s)) / 2 -- s = 0: the ring's
    fold equals the all-reduce up to summation order; s = 1: the RMA ring's
    one-step-stale peer packets, zero before step 0 -- biases keep their
    local gradients; written with PyTorch autograd + torch.optim.Adam.
    Grouped cases: inner groups of gs contiguous ranks (the last
    may be smaller) average within the group; at the end of step t with
    (t + 1) mod h == 0 the group leaders (first rank of each group) replace
    theirs by the mean of the leaders' inner results."""
    cfg = tiny_config(seed=6, gen_lr=1e-2, disc_lr=1e-2, world=W, mode=mode,
                      group_size=gs, staleness=staleness, outer_every=h)
    if mode == xc.MODE_SYNC_ALLREDUCE or mode == xc.MODE_ARAR:
        gs, h = W, 0
    groups = [list(range(a, min(a + gs, W))) for a in range(0, W, gs)]
    leaders = [g[0] for g in groups]
    states = [gan.RankState(cfg, r) for r in range(W)]
    init = copy.deepcopy(states)
    T = 4
    _, log = gan.run(cfg, T, states=states)
    N, m = cfg.n_events, cfg.events_per_sample
    s = torch.arange(N) // m
    lab = torch.cat([torch.ones(N, dtype=torch.float64), torch.zeros(N, dtype=torch.float64)])
    P = []
    for r in range(W):
        gW = [torch.tensor(w, requires_grad=True) for w in init[r].gW]
        gb = [torch.tensor(b, requires_grad=True) for b in init[r].gb]
        dW = [torch.tensor(w, requires_grad=True) for w in init[r].dW]
        db = [torch.tensor(b, requires_grad=True) for b in init[r].db]
        P.append(dict(gW=gW, gb=gb, dW=dW, db=db,
                      optG=torch.optim.Adam(gW + gb, lr=cfg.gen_lr, eps=1e-8),
                      optD=torch.optim.Adam(dW + db, lr=cfg.disc_lr, eps=1e-8)))
    hist = {}
    for t in range(T):
        for r, p in enumerate(P):
            z = torch.tensor(gan.noise(cfg, t, r))
            u = torch.tensor(proxy.fake_uniforms(cfg.seed, t, r, N))
            x = torch.tensor(init[r].shard[proxy.real_indices(cfg.seed, t, r, cfg.shard_rows, N)])
            raw = _torch_mlp(p["gW"], p["gb"], z).reshape(-1, 2, 3)
            c0 = raw[:, :, 0]
            c1 = F.softplus(raw[:, :, 1], beta=1, threshold=20)
            c2 = F.softplus(raw[:, :, 2], beta=1, threshold=20)
            y = c0[s] + c1[s] * u + c2[s] * u * u
            p["optD"].zero_grad()
            ld = F.binary_cross_entropy_with_logits(
                _torch_mlp(p["dW"], p["db"], torch.cat([x, y.detach()]))[:, 0], lab)
            ld.backward()
            p["optD"].step()
            p["optG"].zero_grad()
            lg = F.binary_cross_entropy_with_logits(
                _torch_mlp(p["dW"], p["db"], y)[:, 0], torch.ones(N, dtype=torch.float64))
            lg.backward()
            assert ld.item() == pytest.approx(log[t]["loss_d"][r], rel=1e-10)
            assert lg.item() == pytest.approx(log[t]["loss_g"][r], rel=1e-10)
        hist[t] = [[g.grad.clone() for g in p["gW"]] for p in P]
        for l in range(len(P[0]["gW"])):
            R = {}
            for g in groups:
                for r in g:
                    tot = hist[t][r][l].clone()
                    for o in g:
                        if o != r and t - staleness >= 0:
                            tot = tot + hist[t - staleness][o][l]
                    R[r] = tot / len(g)
            if h > 0 and (t + 1) % h == 0 and len(leaders) > 1:
                outer = sum(R[q] for q in leaders) / len(leaders)
                for q in leaders:
                    R[q] = outer
            for r, p in enumerate(P):
                p["gW"][l].grad = R[r]
        for p in P:
            p["optG"].step()
    for r, p in enumerate(P):
        for a, b in zip(p["gW"] + p["gb"] + p["dW"] + p["db"],
                        states[r].gW + states[r].gb + states[r].dW + states[r].db):
            assert np.allclose(a.detach().numpy(), b, rtol=1e-9, atol=1e-12)
    # ranks 0 and 1 (one group) share G weights iff the exchange is
    # synchronous and no outer step has given the leader a different R
    same = all(np.array_equal(a, b) for a, b in zip(states[0].gW, states[1].gW))
    assert same == (staleness == 0 and (h == 0 or len(leaders) == 1))
    assert not np.allclose(states[0].dW[0], states[1].dW[0])
