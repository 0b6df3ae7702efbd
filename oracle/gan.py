"""The per-rank SAGIPS training step and a lockstep multi-rank driver.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Paper: "Each GPU has a copy of the generator network, but trains
its own discriminator locally. [...] Every rank randomly draws training
sub-samples (via bootstrapping) from its data and feeds them through the GAN.
The discriminator gradients are updated right away whereas the generator
gradients are transferred to neighbouring ranks."  Generator gradients are
exchanged (oracle/exchange.py) and then applied.

One step t of rank r, in the order of DESIGN.md R8 (the paper does not fix
it):
  1  noise z[k, d] ~ N(0, 1)                         (stream NOISE)
  2  raw = G(z)
  3  c = constrain(raw)                              (R1)
  4  fake y[N, 2] = Q(u; c), u from stream FAKE
  5  real x[N, 2] = shard[bootstrap idx]             (stream REAL)
  6  histograms of x and y                           (diagnostic, R22)
  7  D step on [x; y] with labels (1, 0), Adam(D)
  8  G loss on y through the *updated* D, backprop to dy, dc, draw, and
     through G to dW_G, db_G
  9  packet = weights-only dW_G, layer order
 10  exchange -> R (oracle/exchange.py)
 11  Adam(G) with W-grad R and the local bias grads

The multi-step trajectory has no closed form; at N=1 it is pinned against
the same loop written with PyTorch autograd + torch.optim.Adam (tests/
test_oracle_gan.py::test_trajectory_matches_torch_autograd_and_adam).  Each
ingredient is pinned separately (tests/test_oracle_*.py), a full single step
by finite differences of both losses, and the exchange by the ring
invariants; multi-rank trajectories (sync, ARAR, stale RMA, grouped with
the outer leader ring) are pinned the same way (test_multi_rank_trajectory_
matches_torch_loop).
"""
from dataclasses import dataclass, field
from typing import List

import numpy as np

from . import exchange as xc
from . import mlp
from . import philox as px
from . import proxy
from . import tabulated as tab

SAMPLER_QUADRATIC, SAMPLER_TABULATED = 0, 1


@dataclass
class Config:
    world: int = 1
    group_size: int = 1
    outer_every: int = 0
    mode: int = xc.MODE_NONE
    staleness: int = 0
    reduce_mean: int = 1
    noise_dim: int = 8
    gen_hidden: int = 64
    gen_depth: int = 2          # number of hidden layers
    disc_hidden: int = 64
    disc_depth: int = 2
    param_samples: int = 64     # k
    events_per_sample: int = 16  # m
    reference_rows: int = 2048  # N_ref
    shard_rows: int = 1024      # n_s
    gen_lr: float = 1e-5
    disc_lr: float = 1e-4
    leaky_slope: float = 0.01
    true_params: List[float] = field(default_factory=lambda: [1.0, 1.0, 0.5, 2.0, 0.5, 1.0])
    hist_bins: int = 64
    hist_lo: List[float] = field(default_factory=lambda: [0.0, 0.0])
    hist_hi: List[float] = field(default_factory=lambda: [4.0, 4.0])
    seed: int = 1
    # a3-a9 sampler: the quadratic quantile (R1) or the tabulated CDF (R32;
    # true_params then hold (w, b, c) per observable)
    sampler: int = SAMPLER_QUADRATIC
    sampler_grid: int = 1024
    # tensor fusion: the packet also carries the
    # bias gradients and Adam(G) applies their reduction (default: P:305)
    packet_biases: int = 0

    @property
    def n_events(self):
        return self.param_samples * self.events_per_sample

    def gen_sizes(self):
        return [self.noise_dim] + [self.gen_hidden] * self.gen_depth + [6]

    def disc_sizes(self):
        return [2] + [self.disc_hidden] * self.disc_depth + [1]


def desk_config(**kw):
    """C1: G [8,64,64,6], D [2,64,64,1], k=64, m=16 (SPEC desk preset)."""
    return Config(**kw)


def paper_config(**kw):
    """C2: G [6,128,128,128,128,6], D [2,128,128,128,128,1] (R4/R5),
    k = 1024, m = 1024, N_ref = 2N, n_s = N."""
    base = dict(noise_dim=6, gen_hidden=128, gen_depth=4, disc_hidden=128, disc_depth=4,
                param_samples=1024, events_per_sample=1024,
                reference_rows=2 * 1024 * 1024, shard_rows=1024 * 1024)
    base.update(kw)
    return Config(**base)


class RankState:
    def __init__(self, cfg: Config, rank: int):
        self.rank = rank
        a = cfg.leaky_slope
        self.gW, self.gb = mlp.kaiming_init(cfg.seed, px.STREAM_INIT_G, 0, cfg.gen_sizes(), a)
        self.dW, self.db = mlp.kaiming_init(cfg.seed, px.STREAM_INIT_D, rank, cfg.disc_sizes(), a)
        z = lambda arrs: [np.zeros_like(x) for x in arrs]
        self.g_mW, self.g_vW, self.g_mb, self.g_vb = z(self.gW), z(self.gW), z(self.gb), z(self.gb)
        self.d_mW, self.d_vW, self.d_mb, self.d_vb = z(self.dW), z(self.dW), z(self.db), z(self.db)
        self.g_tau = 0
        self.d_tau = 0
        self.shard_idx = proxy.shard_indices(cfg.seed, rank, cfg.reference_rows, cfg.shard_rows)
        if cfg.sampler == SAMPLER_TABULATED:
            # the reference drawn by the tabulated sampler at the true (w, b, c),
            # whose raw values the library passes in fp32 (R32)
            ref = tab.sample_events(tabulated_raw_true(cfg)[None, :], cfg.reference_rows,
                                    proxy.reference_uniforms(cfg.seed, cfg.reference_rows), cfg.sampler_grid)
            ref32 = ref.astype(np.float32)
        else:
            ref = proxy.make_reference(cfg.seed, cfg.true_params, cfg.reference_rows)
            ref32 = proxy.make_reference_f32(cfg.seed, cfg.true_params, cfg.reference_rows)
        self.shard = ref[self.shard_idx]
        self.shard32 = ref32[self.shard_idx]


def tabulated_raw_true(cfg):
    """(logit w, log expm1 b, log expm1 c) per observable, rounded to fp32 (R32)."""
    r = []
    for o in range(2):
        w, b, c = (float(np.float32(v)) for v in cfg.true_params[3 * o:3 * o + 3])
        r += [np.log(w / (1.0 - w)), b if b > 20.0 else np.log(np.expm1(b)), c if c > 20.0 else np.log(np.expm1(c))]
    return np.array(r, dtype=np.float32).astype(np.float64)


def noise(cfg, step, rank):
    return px.normals(cfg.seed, px.STREAM_NOISE, step, rank,
                      cfg.param_samples * cfg.noise_dim).reshape(cfg.param_samples, cfg.noise_dim)


def local_step(cfg: Config, st: RankState, t: int):
    """Steps 1-9 for one rank; applies Adam(D).  Returns every intermediate."""
    a = cfg.leaky_slope
    k, m, N = cfg.param_samples, cfg.events_per_sample, cfg.n_events
    out = {}
    # 1-3 generator forward and constraint
    z = noise(cfg, t, st.rank)
    raw, g_cache = mlp.forward(st.gW, st.gb, z, a)
    tabulated = cfg.sampler == SAMPLER_TABULATED
    if tabulated:
        c = np.array([[tab.constrain(r[3 * o:3 * o + 3]) for o in range(2)] for r in raw])
    else:
        c = proxy.constrain(raw)
    # 4 synthetic events
    u = proxy.fake_uniforms(cfg.seed, t, st.rank, N)
    y = tab.sample_events(raw, m, u, cfg.sampler_grid) if tabulated else proxy.sample_events(c, m, u)
    # 5 real batch
    ridx = proxy.real_indices(cfg.seed, t, st.rank, cfg.shard_rows, N)
    x = st.shard[ridx]
    # 6 histograms (fp32 decision: real rows from the fp32 reference; fake
    #   rows from the fp32 evaluation of the oracle's c -- see R22)
    if tabulated:  # the kernel's decision from fp32 raw (fp64 tables, fp32 events)
        y32 = tab.sample_events(raw.astype(np.float32).astype(np.float64), m, u, cfg.sampler_grid).astype(np.float32)
    else:
        y32 = proxy.sample_events_f32(c.astype(np.float32), m, u)
    x32 = st.shard32[ridx]
    hist = np.zeros((2, 2, cfg.hist_bins + 2), dtype=np.int64)
    for o in range(2):
        hist[0, o] = proxy.histogram_f32(x32[:, o], cfg.hist_lo[o], cfg.hist_hi[o], cfg.hist_bins)
        hist[1, o] = proxy.histogram_f32(y32[:, o], cfg.hist_lo[o], cfg.hist_hi[o], cfg.hist_bins)
    # 7 discriminator step: rows real-first then fake (R9)
    X = np.concatenate([x, y], axis=0)
    labels = np.concatenate([np.ones(N), np.zeros(N)])
    zD, d_cache = mlp.forward(st.dW, st.db, X, a)
    zD = zD[:, 0]
    loss_d = mlp.bce_with_logits(zD, labels)
    dzD = mlp.bce_grad(zD, labels)
    dWd, dbd, _ = mlp.backward(st.dW, d_cache, dzD[:, None], a)
    st.d_tau += 1
    for l in range(len(st.dW)):
        st.dW[l], st.d_mW[l], st.d_vW[l] = mlp.adam_update(st.dW[l], dWd[l], st.d_mW[l], st.d_vW[l], st.d_tau, cfg.disc_lr)
        st.db[l], st.d_mb[l], st.d_vb[l] = mlp.adam_update(st.db[l], dbd[l], st.d_mb[l], st.d_vb[l], st.d_tau, cfg.disc_lr)
    # 8-9 generator step through the updated discriminator
    out.update(z=z, raw=raw, c=c, u=u, y=y, real_idx=ridx, x=x, hist=hist,
               logits_d=zD, loss_d=loss_d, dW_d=dWd, db_d=dbd)
    out.update(generator_step(cfg, st.dW, st.db, st.gW, g_cache, raw, u, y))
    return out


def generator_step(cfg: Config, dW, db, gW, g_cache, raw, u, y):
    """Steps 8-9: the non-saturating generator loss L_G = mean softplus(-D(y))
    through the given (updated) discriminator, backprop to dy, through the
    sampler (dc, draw) and the generator (dW_G, db_G); the weights-only
    packet."""
    a = cfg.leaky_slope
    N, m = cfg.n_events, cfg.events_per_sample
    zG, g_d_cache = mlp.forward(dW, db, y, a)
    zG = zG[:, 0]
    loss_g = mlp.bce_with_logits(zG, np.ones(N))
    dzG = mlp.bce_grad(zG, np.ones(N))
    _, _, dy = mlp.backward(dW, g_d_cache, dzG[:, None], a)
    if cfg.sampler == SAMPLER_TABULATED:
        dc, draw = None, tab.sampler_backward(raw, m, u, dy, cfg.sampler_grid)
    else:
        dc, draw = proxy.sampler_backward(dy, u, raw, m)
    dWg, dbg, _ = mlp.backward(gW, g_cache, draw, a)
    packet = np.concatenate([w.reshape(-1) for w in dWg] + ([b.reshape(-1) for b in dbg] if cfg.packet_biases else []))
    return dict(logits_g=zG, loss_g=loss_g, dy=dy, dc=dc, draw=draw, dW_g=dWg, db_g=dbg, packet=packet)


def apply_generator(cfg: Config, st: RankState, R, db_local):
    """Step 11: unflatten R into the weight gradients; biases use the local
    gradients or, with the fused packet, R's bias part; Adam(G)."""
    st.g_tau += 1
    if cfg.packet_biases:
        nw = sum(w.size for w in st.gW)
        db_local, o = [], nw
        for b in st.gb:
            db_local.append(R[o:o + b.size].reshape(b.shape))
            o += b.size
    off = 0
    for l in range(len(st.gW)):
        n = st.gW[l].size
        gw = R[off:off + n].reshape(st.gW[l].shape)
        off += n
        st.gW[l], st.g_mW[l], st.g_vW[l] = mlp.adam_update(st.gW[l], gw, st.g_mW[l], st.g_vW[l], st.g_tau, cfg.gen_lr)
        st.gb[l], st.g_mb[l], st.g_vb[l] = mlp.adam_update(st.gb[l], db_local[l], st.g_mb[l], st.g_vb[l], st.g_tau, cfg.gen_lr)


def run(cfg: Config, steps: int, states=None, record=None):
    """Lockstep driver over cfg.world simulated ranks.  Returns (states,
    per-step list of dicts with the losses of every rank)."""
    if states is None:
        states = [RankState(cfg, r) for r in range(cfg.world)]
    history = {}
    log = []
    for t in range(steps):
        outs = [local_step(cfg, states[r], t) for r in range(cfg.world)]
        history[t] = [o["packet"] for o in outs]
        history.pop(t - 2, None)
        R = xc.reduce_step(cfg.mode, cfg.world, cfg.group_size, cfg.outer_every,
                           cfg.staleness, cfg.reduce_mean, t, history)
        for r in range(cfg.world):
            apply_generator(cfg, states[r], R[r], outs[r]["db_g"])
        entry = {"loss_d": [o["loss_d"] for o in outs], "loss_g": [o["loss_g"] for o in outs]}
        if record is not None:
            entry.update(record(t, outs, R, states))
        log.append(entry)
    return states, log
