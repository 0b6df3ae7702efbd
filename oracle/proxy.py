"""The proxy pipeline f(x_hat(p)) of the loop-closure experiment.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Paper: six parameters p0..p5 are translated to two observables (y0, y1)
(Eq. 4); the sampler "relies on the inverse CDF method, i.e. we use
the inverse of a differentiable function to sample events from a given one
dimensional distribution"; k = 1024 parameter samples with m = 100
events each (Tab. IV); each rank bootstraps from a random 50%
sub-sample of the reference data.

The functional form is not disclosed (R1).  Reading R1/R2: per observable o
the quantile is the degree-2 polynomial Q(u; c) = c0 + c1 u + c2 u^2 with
(c0, c1, c2) = (p_{3o}, softplus(p_{3o+1}), softplus(p_{3o+2})), and f is the
identity on the sampled (x0, x1).  Everything below is float64 unless the
name ends in ``_f32``: those helpers reproduce an integer decision (a
histogram bin) in the precision the kernel takes it in, as the parity rules
require.
"""
import numpy as np

from . import philox as px

SOFTPLUS_THRESHOLD = 20.0


# ---------------------------------------------------------------- constrain
def softplus(x):
    """softplus(x) = log(1 + e^x), and x itself above the threshold 20 (R23)."""
    x = np.asarray(x, dtype=np.float64)
    return np.where(x > SOFTPLUS_THRESHOLD, x, np.log1p(np.exp(np.minimum(x, SOFTPLUS_THRESHOLD))))


def softplus_grad(x):
    """d softplus / dx = sigmoid(x), and 1 above the threshold."""
    x = np.asarray(x, dtype=np.float64)
    return np.where(x > SOFTPLUS_THRESHOLD, 1.0, 1.0 / (1.0 + np.exp(-x)))


def constrain(raw):
    """raw[k, 6] -> c[k, 2, 3]: c[s, o] = (raw[s,3o], softplus(raw[s,3o+1]),
    softplus(raw[s,3o+2])) (R1; the monotone-quantile validity c1, c2 > 0
    holds by construction)."""
    raw = np.asarray(raw, dtype=np.float64).reshape(-1, 2, 3)
    c = np.empty_like(raw)
    c[:, :, 0] = raw[:, :, 0]
    c[:, :, 1] = softplus(raw[:, :, 1])
    c[:, :, 2] = softplus(raw[:, :, 2])
    return c


# ---------------------------------------------------------------- sampler
def quantile(u, c0, c1, c2):
    """Inverse CDF Q(u; c) = c0 + c1 u + c2 u^2 (R1)."""
    return c0 + c1 * u + c2 * u * u


def fake_uniforms(seed, step, rank, n_events):
    """u[e, o] for the synthetic batch: word 2e+o of the FAKE stream."""
    w = px.words(seed, px.STREAM_FAKE, step, rank, 0, 2 * n_events)
    return px.uniform_open01(w).reshape(n_events, 2)


def sample_events(c, m, u):
    """Synthetic events y[e, o] = Q(u[e, o]; c[e // m, o]), sample-major
    (event e belongs to parameter sample s = e // m; Tab. IV)."""
    c = np.asarray(c, dtype=np.float64).reshape(-1, 2, 3)
    n = c.shape[0] * m
    s = np.arange(n) // m
    y = np.empty((n, 2), dtype=np.float64)
    for o in range(2):
        y[:, o] = quantile(u[:, o], c[s, o, 0], c[s, o, 1], c[s, o, 2])
    return y


def sample_events_f32(c32, m, u):
    """The same events evaluated the way the kernel evaluates them, in fp32
    with every operation rounded separately (no FMA contraction):
    y = c0 + u * (c1 + u * c2).  Used only where an fp32 value decides an
    integer (histogram bins)."""
    c32 = np.asarray(c32, dtype=np.float32).reshape(-1, 2, 3)
    u32 = np.asarray(u, dtype=np.float32)
    n = c32.shape[0] * m
    s = np.arange(n) // m
    y = np.empty((n, 2), dtype=np.float32)
    for o in range(2):
        a = u32[:, o] * c32[s, o, 2]
        b = c32[s, o, 1] + a
        d = u32[:, o] * b
        y[:, o] = c32[s, o, 0] + d
    return y


# ---------------------------------------------------------------- data
def reference_uniforms(seed, n_ref):
    w = px.words(seed, px.STREAM_REF, 0, 0, 0, 2 * n_ref)
    return px.uniform_open01(w).reshape(n_ref, 2)


def make_reference(seed, c_true, n_ref):
    """Loop-closure reference data: the same pipeline driven by the known
    parameters; identical on every rank (R19)."""
    c_true = np.asarray(c_true, dtype=np.float64).reshape(1, 2, 3)
    u = reference_uniforms(seed, n_ref)
    return sample_events(np.repeat(c_true, n_ref, axis=0), 1, u)


def make_reference_f32(seed, c_true, n_ref):
    c_true = np.asarray(c_true, dtype=np.float32).reshape(1, 2, 3)
    u = reference_uniforms(seed, n_ref)
    return sample_events_f32(np.repeat(c_true, n_ref, axis=0), 1, u)


def lemire_index(w, n):
    """(w * n) >> 32: a 32-bit word mapped to [0, n) (R-BOOT)."""
    return ((np.asarray(w, dtype=np.uint64) * np.uint64(n)) >> np.uint64(32)).astype(np.int64)


def shard_indices(seed, rank, n_ref, n_shard):
    """The rank's random 50% sub-sample of the reference, drawn with
    replacement (R18): shard[i] = ref[idx[i]]."""
    w = px.words(seed, px.STREAM_SHARD, 0, rank, 0, n_shard)
    return lemire_index(w, n_ref)


def real_indices(seed, step, rank, n_shard, n_events):
    """Per-step bootstrap of the real batch from the shard."""
    w = px.words(seed, px.STREAM_REAL, step, rank, 0, n_events)
    return lemire_index(w, n_shard)


# ---------------------------------------------------------------- histogram
def histogram_f32(y32, lo, hi, bins):
    """Counts of fp32 values: index 0 = underflow (incl. NaN), 1..bins the
    bins of [lo, hi), bins+1 = overflow.  t = (y - lo) * (bins / (hi - lo)),
    each operation rounded in fp32; bin = floor(t) (R22)."""
    y32 = np.asarray(y32, dtype=np.float32)
    lo32 = np.float32(lo)
    scale = np.float32(bins) / (np.float32(hi) - lo32)
    t = (y32 - lo32) * scale
    h = np.zeros(bins + 2, dtype=np.int64)
    under = ~(t >= np.float32(0.0))
    over = (t >= np.float32(bins)) & ~under
    inside = ~under & ~over
    h[0] = int(under.sum())
    h[bins + 1] = int(over.sum())
    idx = np.floor(t[inside]).astype(np.int64) + 1
    np.add.at(h, idx, 1)
    return h


# ---------------------------------------------------------------- backward
def sampler_backward(dy, u, raw, m):
    """Backprop through the sampler and the constraint.

    dy[e, o] = dL/dy[e, o].  Since dQ/dc = (1, u, u^2) exactly,
        dc[s, o, j] = sum_{e in s} dy[e, o] * u[e, o]^j ,
    and through constrain: draw[s, 3o] = dc[s,o,0],
    draw[s, 3o+1] = dc[s,o,1] * softplus'(raw[s,3o+1]), same for 3o+2.
    The per-sample sums are plain ascending loops over the m events.
    """
    raw = np.asarray(raw, dtype=np.float64).reshape(-1, 6)
    k = raw.shape[0]
    dc = np.zeros((k, 2, 3), dtype=np.float64)
    for s in range(k):
        e = slice(s * m, (s + 1) * m)
        for o in range(2):
            dc[s, o, 0] = np.sum(dy[e, o])
            dc[s, o, 1] = np.sum(dy[e, o] * u[e, o])
            dc[s, o, 2] = np.sum(dy[e, o] * u[e, o] * u[e, o])
    draw = np.empty((k, 6), dtype=np.float64)
    for o in range(2):
        draw[:, 3 * o] = dc[:, o, 0]
        draw[:, 3 * o + 1] = dc[:, o, 1] * softplus_grad(raw[:, 3 * o + 1])
        draw[:, 3 * o + 2] = dc[:, o, 2] * softplus_grad(raw[:, 3 * o + 2])
    return dc, draw
