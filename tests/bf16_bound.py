"""Elementwise error bounds for the bf16 discriminator path (SAGIPS_PREC_BF16,
C5's precision; R20), evaluated on the oracle's own values.

What the GPU computes in bf16 (everything else is fp32): the 128 -> 128
hidden layers' GEMMs -- forward Z = bf16(H) bf16(W)^T, dgrad with bf16(G)
bf16(W), wgrad G^T H with bf16(G) bf16(H) and the bias gradient bf16(G)^T 1
-- all with fp32 accumulation.  A round-to-nearest bf16 operand carries a
relative error of at most u = 2^-8 (8 significant bits; the error is uniform
in [-ulp/2, ulp/2] and ulp / x <= 2^-7), taken as uniform in [-u, u]
(variance u^2 / 3, a slight over-estimate of the log-uniform average).

Error model (a mixed bound, reading R33):
* inside a row's forward / backward chain the roundings of different operand
  elements are independent, so their variances add; a row's bound is
  C_SIGMA = 6 standard deviations.  For dy (one row's whole G step) the
  variance is the exact first-order one: every rounded operand times its
  downstream sensitivity (dy_variance).  For the D step's per-row errors the
  cheaper diagonal chain var(dz) = var(dh) W^2 + (2 u^2 / 3) h^2 W^2 is used
  (LeakyReLU is 1-Lipschitz: var(dh) <= var(dz));
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

U_BF16 = 2.0 ** -8
VAR2 = 2.0 * U_BF16 ** 2 / 3.0   # variance of a product of two rounded operands (relative^2)
C2U = 2.01 * U_BF16              # worst case of that product's relative error (the wgrad's G^T h)
U_DB = U_BF16                    # the bias gradient's operand (G)
C_SIGMA = 6.0
SCHEME = "bf16"


def use_scheme(scheme):
    """'bf16' (SAGIPS_PREC_BF16, the default) or 'split' (SAGIPS_PREC_FP32 on
    the tensor cores, R28): every forward / dgrad operand x = hi + lo with
    |x - hi - lo| <= 2^-18 |x| and the lo x lo product dropped -- a product's
    relative error below 3 2^-18, modelled as u = 2^-16 per operand -- while
    the wgrad multiplies the split G by the hi plane of H only (relative
    error 2^-9, taken as 2^-8) and the bias gradient sums the split G."""
    global U_BF16, VAR2, C2U, U_DB, SCHEME
    if scheme == "bf16":
        U_BF16 = 2.0 ** -8
        C2U = 2.01 * U_BF16
    elif scheme == "split":
        U_BF16 = 2.0 ** -16
        C2U = 1.01 * 2.0 ** -8
    else:
        raise ValueError(scheme)
    VAR2 = 2.0 * U_BF16 ** 2 / 3.0
    U_DB = U_BF16
    SCHEME = scheme


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


def backward_bounds(Ws, cache, vz, vh, dout, vdout, alpha, kink_mode=0, bf16=True, values_only=False):
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
        dWs[l] = dz.T @ h
        dbs[l] = dz.sum(axis=0)
        if values_only:
            g = dz @ Ws[l]
            continue
        sdz = C_SIGMA * np.sqrt(vdz)
        edWs[l] = sdz.T @ np.abs(h) + (C2U * (np.abs(dz).T @ np.abs(h)) if bf else 0.0)
        if vh is not None:
            edWs[l] = edWs[l] + np.abs(dz).T @ (C_SIGMA * np.sqrt(vh[l]))
        edbs[l] = sdz.sum(axis=0) + (U_DB * np.abs(dz).sum(axis=0) if bf else 0.0)
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
        dW, db, _, edW, edb, _ = backward_bounds(d_before[0], cD, vzD, vhD, dz, vdz, a, mode, values_only=mode != 0)
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
    # dy: the exact first-order variance (dy_variance); the diagonal chain
    # model of backward_bounds under-estimates it (a rounded operand feeds
    # every output of its layer, so the errors of one layer's outputs are
    # correlated) -- checked by emulating the GPU's bf16 roundings in numpy
    # plus, for dy, the first-order bound of any pattern of LeakyReLU' flips
    vdy, kdy = dy_variance(d_after[0], d_after[1], out["y"], a, 1.0 / N, with_kinks=True)
    edy0 = C_SIGMA * np.sqrt(vdy) + kdy
    vals0 = None
    for mode in (0, 1, -1):
        _, _, dy, _, _, _ = backward_bounds(d_after[0], cG, vzG, vhG, dzG, vdzG, a, mode, values_only=True)
        _, draw = proxy.sampler_backward(dy, out["u"], raw, m)
        edy = edy0
        # the sampler backward and the generator are linear in dy with
        # |u^j| <= 1 and |softplus'| <= 1: the bound through the same
        # functions on absolute values (raw = 50: softplus' = 1; slope 1)
        _, edraw = proxy.sampler_backward(edy, out["u"], np.full_like(raw, 50.0), m)
        dWg, dbg, _ = mlp.backward(g_params[0], gcache, draw, a)
        # the generator (fp32) propagates the draw error: within a sample's
        # chain as variance, over the k samples linearly
        if mode == 0:
            _, _, _, edWg, edbg, _ = backward_bounds(g_params[0], gcache, None, None, draw,
                                                     (np.abs(edraw) / C_SIGMA) ** 2, a, 0, bf16=False)
        vals = (dy.reshape(-1), draw.reshape(-1), _flat(dWg), _flat(dbg))
        if mode == 0:
            vals0 = vals
            res["dy"], res["draw"] = edy.reshape(-1), np.abs(edraw).reshape(-1)
            res["dy_forced"] = np.zeros_like(res["dy"])
            res["packet"], res["db_g"] = _flat(edWg), _flat(edbg)
        else:
            for k, v, r in zip(("dy_forced", "draw", "packet", "db_g"), vals, vals0):
                res[k] = res[k] + np.abs(v - r)
    res.pop("dy_forced")  # dy carries the per-flip kink bound instead of the forced extremes
    return res


def dy_variance(Ws, bs, y, alpha, scale, with_kinks=False):
    """Exact first-order variance of the G step's dy under bf16 operand
    rounding (per row, per component), by the downstream sensitivities of
    every rounded operand: the forward layers' inputs and weights reach dy
    through the logit (dy = dz q, dz = (sigmoid(z) - 1) scale, q = the
    row's backward chain of a unit dz); the dgrad layers' inputs G and
    weights reach it through S_l = d dy / d (G_{l+1} W_l).  Independent
    roundings (relative variance u^2 / 3 each) add their variances.
    with_kinks: also the first-order bound of LeakyReLU' decisions that may
    differ (|Z| within C_SIGMA of its forward error): flipping the branch of
    element j of layer l changes dy by (1 - alpha) |P_l[j]| |S_l[j]|, P_l =
    G_{l+1} W_l before the mask; summed over a row's ambiguous elements
    (any pattern of flips)."""
    u2 = U_BF16 ** 2 / 3.0
    L = len(Ws)
    h = np.asarray(y, dtype=np.float64)
    hs, zs = [], []
    for l in range(L):
        z = h @ Ws[l].T + bs[l]
        hs.append(h)
        zs.append(z)
        h = mlp.lrelu(z, alpha) if l < L - 1 else z
    logit = h[:, 0]
    dz = (mlp.sigmoid(logit) - 1.0) * scale
    sig_p = mlp.sigmoid(logit) * (1.0 - mlp.sigmoid(logit)) * scale
    # d logit / d z_{l+1} and d logit / d h_l for the hidden layers (backward of a unit logit)
    g = np.ones((h.shape[0], 1))
    gz, gh = [None] * L, [None] * L
    for l in reversed(range(L)):
        dzl = g if l == L - 1 else g * mlp.lrelu_grad(zs[l], alpha)
        gz[l] = dzl
        g = dzl @ Ws[l]
        gh[l] = g
    var_logit = np.zeros(h.shape[0])
    for l in range(L):
        if not _is_bf16(Ws, l):
            continue
        # input rounding: sum_k (d logit / d h_k)^2 h_k^2 ; weight rounding: sum_j (d logit / d z_j)^2 sum_k h_k^2 W_jk^2
        var_logit += u2 * np.sum(gh[l] ** 2 * hs[l] ** 2, axis=1)
        var_logit += u2 * np.sum(gz[l] ** 2 * ((hs[l] ** 2) @ (Ws[l].T ** 2)), axis=1)
    # the backward chain of a unit dz: G_4 = w m_4, G_l = (G_{l+1} W_l) m_l; q = G_1 W_0
    Gs, Ps = [None] * L, [None] * L
    G = np.repeat(Ws[L - 1][0][None, :], h.shape[0], axis=0)
    Ps[L - 1] = G                                     # the head's "pre-mask" G_4 (mask of Z_4)
    G = G * mlp.lrelu_grad(zs[L - 2], alpha)
    for l in range(L - 2, 0, -1):
        Gs[l] = G  # G_{l+1}: the input of the dgrad with W_l
        Ps[l] = G @ Ws[l]
        G = Ps[l] * mlp.lrelu_grad(zs[l - 1], alpha)
    q = G @ Ws[0]                                     # [rows, 2]
    var = (sig_p ** 2 * var_logit)[:, None] * q ** 2  # through dz
    kink = np.zeros_like(var)
    if with_kinks:  # bands of the pre-activations Z_1..Z_4 (Z_1 is fp32: no band)
        _, _, vz, _ = forward_var(Ws, bs, y, alpha)
        amb = [np.abs(zs[l]) <= C_SIGMA * np.sqrt(vz[l]) for l in range(L)]
    # S[o]: [rows, 128] per output component o; S_1 = m_1 W_0[:, o], S_l = m_l (W_{l-1} S_{l-1})
    S = [mlp.lrelu_grad(zs[0], alpha) * Ws[0][:, o][None, :] for o in range(2)]
    for l in range(1, L - 1):
        Gl2 = (Gs[l] * dz[:, None]) ** 2                                  # G_{l+1}^2 of this row
        GW2 = Gl2 @ (Ws[l] ** 2)
        for o in range(2):
            WS = S[o] @ Ws[l].T                                           # d dy_o / d G_{l+1}
            var[:, o] += u2 * np.sum(Gl2 * WS ** 2, axis=1)               # G rounding
            var[:, o] += u2 * np.sum(S[o] ** 2 * GW2, axis=1)             # W rounding
            if with_kinks:  # the mask of Z_{l+1}, applied to P_{l+1} (the head's G_4 for l + 1 = 4)
                kink[:, o] += (1.0 - alpha) * np.sum(amb[l] * np.abs(Ps[l + 1] * dz[:, None]) * np.abs(WS), axis=1)
            if l + 1 < L - 1:
                S[o] = mlp.lrelu_grad(zs[l], alpha) * WS
    return (var, kink) if with_kinks else var
