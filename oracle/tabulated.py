"""Tabulated-CDF sampler (reading R32 in DESIGN.md).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Paper: the sampler "relies on the inverse CDF method, i.e. we use the
inverse of a differentiable function to sample events from a given one
dimensional distribution"; realistic pipelines are expected to be
sampler-dominated.  The closed-form quadratic quantile of R1
skips the density -> CDF -> inversion work; this variant does it on a grid.

Reading R32 (builder-chosen family, not from the paper).  Per parameter
sample s and observable o, with (r0, r1, r2) = raw[s][3o..3o+2]:
    w = sigmoid(r0), b = softplus(r1), c = softplus(r2)
    f(x) = w x^b (1-x)^c + (1-w) x^c (1-x)^b          on [0, 1]
Both mirror components integrate to B(b+1, c+1), so f / B(b+1, c+1) is a
density with E[x] = (w (b+1) + (1-w) (c+1)) / (b + c + 2).
Grid t_i = i / (G-1), i = 0..G-1, Delta = 1 / (G-1):
    S_0 = 0, S_i = S_{i-1} + (f(t_{i-1}) + f(t_i)) Delta / 2   (trapezoid)
    F_i = S_i / S_{G-1}
Inversion of u in (0, 1): i = the largest index with F_i <= u, clipped to
[0, G-2]; x = t_i + (u - F_i) / (F_{i+1} - F_i) Delta.  Events y[e][o] = x
(f = identity, R2) with u from the FAKE Philox stream as the quadratic
sampler (R-RNG, R-UNIF).  The backward is the exact derivative of this
tabulated inverse: with F'_i = dF_i/dtheta (the same trapezoid over
df/dtheta, then the quotient rule),
    dx/dtheta = -Delta [F'_i (F_{i+1} - F_i) + (u - F_i)(F'_{i+1} - F'_i)] / (F_{i+1} - F_i)^2
and dtheta/draw = (w (1-w), sigmoid(r1), sigmoid(r2)).
Everything in float64, loops in the order written.
"""
import numpy as np

from .proxy import softplus, softplus_grad


def sigmoid(x):
    return 1.0 / (1.0 + np.exp(-np.asarray(x, dtype=np.float64)))


def constrain(raw3):
    """(r0, r1, r2) -> (w, b, c)."""
    r0, r1, r2 = (float(v) for v in raw3)
    return float(sigmoid(r0)), float(softplus(r1)), float(softplus(r2))


def _pw(t, p):
    """t^p with 0^p = 0 for p > 0 (b, c = softplus > 0) and 0^0 = 1."""
    return np.where(t > 0.0, np.power(np.maximum(t, 1e-300), p), 0.0 if p > 0 else 1.0)


def _xlogx_pw(t, p):
    """t^p ln t with the limit 0 at t = 0."""
    return np.where(t > 0.0, np.power(np.maximum(t, 1e-300), p) * np.log(np.maximum(t, 1e-300)), 0.0)


def density(t, w, b, c):
    """Unnormalised f(t) = w t^b (1-t)^c + (1-w) t^c (1-t)^b."""
    t = np.asarray(t, dtype=np.float64)
    return w * _pw(t, b) * _pw(1.0 - t, c) + (1.0 - w) * _pw(t, c) * _pw(1.0 - t, b)


def density_grads(t, w, b, c):
    """(df/dw, df/db, df/dc) at t."""
    t = np.asarray(t, dtype=np.float64)
    s = 1.0 - t
    dfw = _pw(t, b) * _pw(s, c) - _pw(t, c) * _pw(s, b)
    dfb = w * _xlogx_pw(t, b) * _pw(s, c) + (1.0 - w) * _pw(t, c) * _xlogx_pw(s, b)
    dfc = w * _pw(t, b) * _xlogx_pw(s, c) + (1.0 - w) * _xlogx_pw(t, c) * _pw(s, b)
    return dfw, dfb, dfc


def trapezoid_cumsum(f, G):
    """S_0 = 0, S_i = S_{i-1} + (f_{i-1} + f_i) Delta / 2, in index order."""
    delta = 1.0 / (G - 1)
    S = np.zeros(G, dtype=np.float64)
    for i in range(1, G):
        S[i] = S[i - 1] + (f[i - 1] + f[i]) * delta / 2.0
    return S


def cdf_table(w, b, c, G):
    """F_i = S_i / S_{G-1} on t_i = i / (G-1)."""
    t = np.arange(G, dtype=np.float64) / (G - 1)
    S = trapezoid_cumsum(density(t, w, b, c), G)
    return S / S[G - 1]


def cdf_table_grads(w, b, c, G):
    """dF_i / d(w, b, c): quotient rule on the trapezoid sums."""
    t = np.arange(G, dtype=np.float64) / (G - 1)
    S = trapezoid_cumsum(density(t, w, b, c), G)
    out = []
    for df in density_grads(t, w, b, c):
        dS = trapezoid_cumsum(df, G)
        out.append((dS * S[G - 1] - S * dS[G - 1]) / S[G - 1] ** 2)
    return out


def cell(F, u):
    """The largest i with F_i <= u, clipped to [0, G-2]."""
    G = len(F)
    i = int(np.searchsorted(F, u, side="right")) - 1
    return min(max(i, 0), G - 2)


def invert(F, u):
    G = len(F)
    delta = 1.0 / (G - 1)
    i = cell(F, u)
    return i * delta + (u - F[i]) / (F[i + 1] - F[i]) * delta


def invert_grad(F, dF, u):
    """dx/dtheta of invert() for one parameter's table derivative dF."""
    G = len(F)
    delta = 1.0 / (G - 1)
    i = cell(F, u)
    d = F[i + 1] - F[i]
    return -delta * (dF[i] * d + (u - F[i]) * (dF[i + 1] - dF[i])) / (d * d)


def sample_events(raw, m, u, G):
    """raw [k][6], u [k*m][2] -> y [k*m][2]: event e of sample s = e // m."""
    raw = np.asarray(raw, dtype=np.float64).reshape(-1, 6)
    y = np.empty((len(u), 2), dtype=np.float64)
    for s in range(raw.shape[0]):
        for o in range(2):
            F = cdf_table(*constrain(raw[s, 3 * o:3 * o + 3]), G)
            for e in range(s * m, min((s + 1) * m, len(u))):
                y[e, o] = invert(F, u[e, o])
    return y


def sampler_backward(raw, m, u, dy, G):
    """dLoss/draw [k][6] from dLoss/dy [k*m][2] (events fixed by u)."""
    raw = np.asarray(raw, dtype=np.float64).reshape(-1, 6)
    draw = np.zeros_like(raw)
    for s in range(raw.shape[0]):
        for o in range(2):
            r = raw[s, 3 * o:3 * o + 3]
            w, b, c = constrain(r)
            F = cdf_table(w, b, c, G)
            dFs = cdf_table_grads(w, b, c, G)
            dth = np.zeros(3)
            for e in range(s * m, min((s + 1) * m, len(u))):
                for j in range(3):
                    dth[j] += dy[e, o] * invert_grad(F, dFs[j], u[e, o])
            chain = (w * (1.0 - w), float(softplus_grad(r[1])), float(softplus_grad(r[2])))
            draw[s, 3 * o:3 * o + 3] = dth * np.array(chain)
    return draw


def analytic_mean(w, b, c):
    """E[x] under the exact (continuous) density."""
    return (w * (b + 1.0) + (1.0 - w) * (c + 1.0)) / (b + c + 2.0)


def tabulated_mean(F):
    """E[x] of the piecewise-linear-CDF distribution: uniform within each cell."""
    G = len(F)
    t = np.arange(G, dtype=np.float64) / (G - 1)
    return float(np.sum((F[1:] - F[:-1]) * (t[1:] + t[:-1]) / 2.0))
