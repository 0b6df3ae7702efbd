"""Elementwise error bounds for the bf16 discriminator path (SAGIPS_PREC_BF16,
C5's precision; R20), evaluated on the oracle's own values.

What the GPU computes in bf16 (everything else is fp32): the 128 -> 128
hidden layers' GEMMs -- forward Z = bf16(H) bf16(W)^T, dgrad with bf16(G)
bf16(W), wgrad G^T H with bf16(G) bf16(H) and the bias gradient bf16(G)^T 1
-- all with fp32 accumulation.  A round-to-nearest bf16 operand carries a
relative error uniform in [-u, u], u = 2^-9 (variance u^2 / 3).

Error model (a mixed bound, reading R33):
* inside a row's forward / backward chain the rounding errors of the K = 128
  terms of a dot product are independent, so their variances add (root sum
  of squares): var(dz) = var(dh) W^2 + (2 u^2 / 3) h^2 W^2 per bf16 layer
  (LeakyReLU is 1-Lipschitz: var(dh) <= var(dz)); the same backwards for the
  dgrad chain; a row's bound is C_SIGMA = 6 standard deviations;
* across rows -- the weight-gradient and loss sums, whose per-row errors share
  the weights' rounding and may add coherently -- the per-row bounds add
  linearly (worst case), plus the wgrad's own operand rounding 2.01 u |G|^T |h|.
* LeakyReLU' takes a branch on the sign of Z: where |Z| is within its bound
  the branch may differ; the kink deviation (tests/kink.py's forced-branch
  method, per-element bands) is added.
The tests compare GPU and oracle elementwise with these bounds plus a 1e-4
max|ref| floor.

TEST INFRASTRUCTURE (uses the oracle's functions; no GPU arithmetic).
"""
import numpy as np

from oracle import mlp, proxy

U_BF16 = 2.0 ** -9
VAR2 = 2.0 * U_BF16 ** 2 / 3.0   # variance of a product of two rounded operands (relative^2)
C2U = 2.01 * U_BF16              # worst case of that product's relative error
C_SIGMA = 6.0


def _is_bf16(Ws, l):
    """the 128 -> 128 hidden layers run on the tensor cores (paper widths)"""
    return 0 < l < len(Ws) - 1 and Ws[l].shape == (128, 128)


def forward_var(Ws, bs, x, alpha):
    """Returns (out, cache, vz, vh): cache[l] = (h_in, z); vz[l] = per-element
    variance of layer l's pre-activation error, vh[l] of its input's."""
    h = np.asarray(x, dtype=np.float64)
    v = np.zeros_like(h)
    cache, vz, vh = [], [], []
    L = len(Ws)
    for l in range(L):
        z = h @ Ws[l].T + bs[l]
        W2 = Ws[l].T ** 2
        e = v @ W2
        if _is_bf16(Ws, l):
            e = e + VAR2 * ((h * h) @ W2)
        cache.append((h, z))
        vz.append(e)
        vh.append(v)
        if l < L - 1:
            h = mlp.lrelu(z, alpha)
            v = e
        else:
            h = z
    return h, cache, vz, vh


def backward_bounds(Ws, cache, vz, vh, dout, vdout, alpha, kink_mode=0, bf16=True):
    """Reverse pass.  dout: gradient at the output, vdout: its per-row error
    variance.  kink_mode 0: the oracle's branches; +1 / -1: every branch with
    |z| <= C_SIGMA sqrt(vz) forced positive / negative.  Returns (dWs, dbs,
    dx, edWs, edbs, vdx): edW / edb are bounds (linear over rows), vdx the
    per-row variance of dx."""
    L = len(Ws)
    dWs, dbs, edWs, edbs = [None] * L, [None] * L, [None] * L, [None] * L
    g = np.asarray(dout, dtype=np.float64)
    v = np.asarray(vdout, dtype=np.float64)
    for l in reversed(range(L)):
        h, z = cache[l]
        if l == L - 1:
            dz, vdz = g, v
        else:
            pos = z > 0
            band = C_SIGMA * np.sqrt(vz[l]) if vz is not None else 0.0
            if kink_mode > 0:
                pos = pos | (np.abs(z) <= band)
            elif kink_mode < 0:
                pos = pos & ~(np.abs(z) <= band)
            slope = np.where(pos, 1.0, alpha)
            dz, vdz = g * slope, v * slope * slope
        bf = bf16 and _is_bf16(Ws, l)
        sdz = C_SIGMA * np.sqrt(vdz)
        dWs[l] = dz.T @ h
        edWs[l] = sdz.T @ np.abs(h) + (C2U * (np.abs(dz).T @ np.abs(h)) if bf else 0.0)
        if vh is not None:
            edWs[l] = edWs[l] + np.abs(dz).T @ (C_SIGMA * np.sqrt(vh[l]))
        dbs[l] = dz.sum(axis=0)
        edbs[l] = sdz.sum(axis=0) + (U_BF16 * np.abs(dz).sum(axis=0) if bf else 0.0)
        W2 = Ws[l] ** 2
        g = dz @ Ws[l]
        v = vdz @ W2 + (VAR2 * ((dz * dz) @ W2) if bf else 0.0)
    return dWs, dbs, g, edWs, edbs, v


def _flat(ws):
    return np.concatenate([w.reshape(-1) for w in ws])


def step_tolerances(cfg, d_before, d_after, g_params, out):
    """Per-element bounds for a bf16 step's dW_D, db_D (D step with d_before)
    and dy, draw, packet, db_G (G step through d_after), and the two losses.
    out: gan.local_step's dict (its x, y, z, u)."""
    a = cfg.leaky_slope
    N, m = cfg.n_events, cfg.events_per_sample
    res = {}
    # D step: logits of [x; y], BCE with labels (1, 0), backward
    X = np.concatenate([out["x"], out["y"]])
    labels = np.concatenate([np.ones(N), np.zeros(N)])
    zD, cD, vzD, vhD = forward_var(d_before[0], d_before[1], X, a)
    s_logit = C_SIGMA * np.sqrt(vzD[-1][:, 0])
    dz = mlp.bce_grad(zD[:, 0], labels)[:, None]
    vdz = ((0.25 / (2 * N)) ** 2 * vzD[-1][:, 0])[:, None]   # |sigmoid'| <= 1/4
    res["loss_d"] = float(np.mean(s_logit))                  # |softplus'| <= 1, linear over rows
    refs = None
    for mode in (0, 1, -1):
        dW, db, _, edW, edb, _ = backward_bounds(d_before[0], cD, vzD, vhD, dz, vdz, a, mode)
        if mode == 0:
            refs = (_flat(dW), _flat(db))
            res["dW_d"], res["db_d"] = _flat(edW), _flat(edb)
        else:
            res["dW_d"] = res["dW_d"] + np.abs(_flat(dW) - refs[0])
            res["db_d"] = res["db_d"] + np.abs(_flat(db) - refs[1])
    # G step through the updated D: dy, then the sampler and the generator (fp32)
    zG, cG, vzG, vhG = forward_var(d_after[0], d_after[1], out["y"], a)
    res["loss_g"] = float(np.mean(C_SIGMA * np.sqrt(vzG[-1][:, 0])))
    dzG = mlp.bce_grad(zG[:, 0], np.ones(N))[:, None]
    vdzG = ((0.25 / N) ** 2 * vzG[-1][:, 0])[:, None]
    _, gcache = mlp.forward(g_params[0], g_params[1], out["z"], a)
    raw = gcache[-1][1]
    vals0 = None
    for mode in (0, 1, -1):
        _, _, dy, _, _, vdy = backward_bounds(d_after[0], cG, vzG, vhG, dzG, vdzG, a, mode)
        _, draw = proxy.sampler_backward(dy, out["u"], raw, m)
        edy = C_SIGMA * np.sqrt(vdy)
        # the sampler backward and the generator are linear in dy with
        # |u^j| <= 1 and |softplus'| <= 1: the bound through the same
        # functions on absolute values (raw = 50: softplus' = 1; slope 1)
        _, edraw = proxy.sampler_backward(edy, out["u"], np.full_like(raw, 50.0), m)
        dWg, dbg, _ = mlp.backward(g_params[0], gcache, draw, a)
        # the generator (fp32) propagates the draw error: within a sample's
        # chain as variance, over the k samples linearly
        _, _, _, edWg, edbg, _ = backward_bounds(g_params[0], gcache, None, None, draw,
                                                 (np.abs(edraw) / C_SIGMA) ** 2, a, 0, bf16=False)
        vals = (dy.reshape(-1), draw.reshape(-1), _flat(dWg), _flat(dbg))
        if mode == 0:
            vals0 = vals
            res["dy"], res["draw"] = edy.reshape(-1), np.abs(edraw).reshape(-1)
            res["packet"], res["db_g"] = _flat(edWg), _flat(edbg)
        else:
            for k, v, r in zip(("dy", "draw", "packet", "db_g"), vals, vals0):
                res[k] = res[k] + np.abs(v - r)
    return res
