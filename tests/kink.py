"""LeakyReLU kink ambiguity bound for gradient parity (R27).

LeakyReLU'(z) is 1 for z > 0 and alpha otherwise: a floating-point sign
decides a discrete branch.  The GPU takes it on fp32 pre-activations, the
oracle on fp64 ones, so a pre-activation within the fp32 accumulation error
of zero may take different branches on the two sides, changing that row's
gradient contribution by (1 - alpha) of itself -- not a small relative
perturbation.  This module recomputes the step's gradients with every such
ambiguous decision forced to the positive branch, then to the negative one,
using the oracle's own functions, and returns the elementwise deviation from
the oracle's gradients.  Parity tests add it to the 1e-3 tolerance.

Band: |z| <= c * 2^-24 * (|h| |W|^T + |b|), c = 16 (fp32 accumulation bound
of a K = 128 dot product with slack).  Where the two sides' *inputs* differ
by a known bound dx per row (the tabulated sampler's events, R32: the
inverse CDF amplifies the generator's fp32 rounding), the band also holds
the propagated input deviation |W_l| d_{l-1}, d_0 = dx (LeakyReLU is
1-Lipschitz).
"""
import numpy as np

from oracle import mlp, proxy

U32 = 2.0 ** -24
C_BAND = 16.0
BAND_FP32 = C_BAND * 2.0 ** -24          # CUDA-core fp32 dot products
BAND_BF16X3 = 16.0 * 2.0 ** -16          # bf16x3 tensor-core layers: ~2^-15 per layer, accumulated over three layers, x2 slack


def _forward(Ws, bs, x, alpha, band_rel=BAND_FP32, x_dev=None):
    h = np.asarray(x, dtype=np.float64)
    dev = None if x_dev is None else np.broadcast_to(np.asarray(x_dev, dtype=np.float64)[:, None], h.shape)
    cache = []
    L = len(Ws)
    for l in range(L):
        z = h @ Ws[l].T + bs[l]
        band = band_rel * (np.abs(h) @ np.abs(Ws[l]).T + np.abs(bs[l]))
        if dev is not None:
            dev = dev @ np.abs(Ws[l]).T  # input deviation bound of this layer's pre-activations
            band = band + dev
        cache.append((h, z, band))
        h = mlp.lrelu(z, alpha) if l < L - 1 else z
    return h, cache


def _backward(Ws, cache, dout, alpha, mode):
    """mode 0: the oracle's decisions; +1 / -1: band decisions forced."""
    L = len(Ws)
    dWs, dbs = [None] * L, [None] * L
    g = dout
    for l in reversed(range(L)):
        h, z, band = cache[l]
        if l == L - 1:
            dz = g
        else:
            pos = z > 0
            if mode > 0:
                pos = pos | (np.abs(z) <= band)
            elif mode < 0:
                pos = pos & ~(np.abs(z) <= band)
            dz = g * np.where(pos, 1.0, alpha)
        dWs[l] = dz.T @ h
        dbs[l] = dz.sum(axis=0)
        g = dz @ Ws[l]
    return dWs, dbs, g


def _flat(ws):
    return np.concatenate([w.reshape(-1) for w in ws])


def step_deviation(cfg, d_before, d_after, g_params, out, disc_band=BAND_FP32, fake_dev=0.0):
    """Elementwise kink deviations of the D-step grads (dW_D, db_D) and of
    the G-step quantities (dy, draw, packet, db_G) of one oracle step.
    d_before / d_after: (Ws, bs) of the discriminator before / after Adam;
    g_params: (Ws, bs) of the generator; out: gan.local_step's dict."""
    a = cfg.leaky_slope
    N, m = cfg.n_events, cfg.events_per_sample
    # D step
    X = np.concatenate([out["x"], out["y"]])
    labels = np.concatenate([np.ones(N), np.zeros(N)])
    xdev = np.concatenate([np.zeros(N), np.full(N, fake_dev)]) if fake_dev > 0 else None
    zD, cD = _forward(d_before[0], d_before[1], X, a, disc_band, xdev)
    dzD = mlp.bce_grad(zD[:, 0], labels)[:, None]
    ref = _backward(d_before[0], cD, dzD, a, 0)
    devW = np.zeros(sum(w.size for w in d_before[0]))
    devB = np.zeros(sum(b.size for b in d_before[1]))
    for mode in (1, -1):
        alt = _backward(d_before[0], cD, dzD, a, mode)
        devW = np.maximum(devW, np.abs(_flat(alt[0]) - _flat(ref[0])))
        devB = np.maximum(devB, np.abs(_flat(alt[1]) - _flat(ref[1])))
    # G step through the updated D, then the sampler and the generator
    zG, cG = _forward(d_after[0], d_after[1], out["y"], a, disc_band, np.full(N, fake_dev) if fake_dev > 0 else None)
    dzG = mlp.bce_grad(zG[:, 0], np.ones(N))[:, None]
    _, gcache = _forward(g_params[0], g_params[1], out["z"], a)
    raw = gcache[-1][1]
    res = {}
    refs = None
    for mode in (0, 1, -1):
        _, _, dy = _backward(d_after[0], cG, dzG, a, mode)
        if getattr(cfg, "sampler", 0) == 1:  # the tabulated sampler (R32)
            from oracle import tabulated as tab
            draw = tab.sampler_backward(raw, m, out["u"], dy, cfg.sampler_grid)
        else:
            _, draw = proxy.sampler_backward(dy, out["u"], raw, m)
        dWg, dbg, _ = _backward(g_params[0], gcache, draw, a, mode)
        vals = (dy.reshape(-1), draw.reshape(-1), _flat(dWg), _flat(dbg))
        if mode == 0:
            refs = vals
            res = {k: np.zeros_like(v) for k, v in zip(("dy", "draw", "packet", "db_g"), vals)}
        else:
            for k, v, r in zip(("dy", "draw", "packet", "db_g"), vals, refs):
                res[k] = np.maximum(res[k], np.abs(v - r))
    res["dW_d"] = devW
    res["db_d"] = devB
    return res
