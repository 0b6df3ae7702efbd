"""Helpers for the -m gpu parity tests: build a library context and the
matching oracle state from the same configuration, and the tolerance
metrics of DESIGN.md (Parity)."""
import numpy as np

from oracle import gan
from oracle import mlp


def lib():
    from paper_2407_00051_b200 import _lib
    return _lib


def oracle_config(c):
    """oracle.gan.Config with the same fields as a library sagips_config."""
    return gan.Config(world=c.world, group_size=c.group_size, outer_every=c.outer_every, mode=c.mode,
                      staleness=c.staleness, reduce_mean=c.reduce_mean, noise_dim=c.noise_dim,
                      gen_hidden=c.gen_hidden, gen_depth=c.gen_depth, disc_hidden=c.disc_hidden,
                      disc_depth=c.disc_depth, param_samples=c.param_samples,
                      events_per_sample=c.events_per_sample, reference_rows=c.reference_rows,
                      shard_rows=c.shard_rows, gen_lr=float(np.float32(c.gen_lr)),
                      disc_lr=float(np.float32(c.disc_lr)), leaky_slope=float(np.float32(c.leaky_slope)),
                      true_params=[float(x) for x in c.true_params], hist_bins=c.hist_bins,
                      hist_lo=[float(x) for x in c.hist_lo], hist_hi=[float(x) for x in c.hist_hi], seed=c.seed,
                      sampler=c.sampler, sampler_grid=c.sampler_grid if c.sampler_grid > 0 else 1024,
                      packet_biases=c.packet_biases)


def flat(ws):
    return np.concatenate([w.reshape(-1) for w in ws])


def unflat(v, like):
    out, off = [], 0
    for w in like:
        out.append(np.asarray(v[off:off + w.size], dtype=np.float64).reshape(w.shape))
        off += w.size
    return out


def sync_params(ctx, st):
    """Round the oracle's initial parameters to fp32 and load the same values
    into the GPU context, so both sides start from identical numbers."""
    L = lib()
    for name, which in (("gW", L.T_GEN_W), ("gb", L.T_GEN_B), ("dW", L.T_DISC_W), ("db", L.T_DISC_B)):
        ws = getattr(st, name)
        v = flat(ws).astype(np.float32)
        ctx.set(which, v)
        setattr(st, name, unflat(v.astype(np.float64), ws))


def grad_close(gpu, ref, rel=1e-3, extra=None):
    """|a - b| <= rel * max(|b|, 1e-2 * max|b|) elementwise (R24): entries
    that cancel to below 1% of the tensor's largest carry no 1e-3 relative
    information in fp32 -- a sum over R rows has error ~ sqrt(R) u sum|terms|;
    the plain fp32 CUDA-core path misses a 1e-3*max floor on db_D by 4.5x."""
    gpu = np.asarray(gpu, dtype=np.float64).reshape(-1)
    ref = np.asarray(ref, dtype=np.float64).reshape(-1)
    floor = 1e-2 * np.max(np.abs(ref)) if ref.size else 0.0
    tol = rel * np.maximum(np.abs(ref), floor)
    if extra is not None:  # LeakyReLU kink ambiguity (tests/kink.py, R27)
        tol = tol + np.asarray(extra, dtype=np.float64).reshape(-1)
    bad = np.abs(gpu - ref) > tol
    return (not bad.any()), int(bad.sum()), float(np.max(np.abs(gpu - ref) / np.maximum(tol, 1e-300)) * rel)


def assert_grad_close(gpu, ref, rel=1e-3, what="", extra=None, outliers=0):
    """outliers: how many elements may exceed the tolerance, each by at most
    max|ref| (a LeakyReLU decision flipped in a mixed pattern that the two
    forced extremes of tests/kink.py do not bound changes one row's
    contribution by at most (1 - alpha) of itself)."""
    ok, nbad, worst = grad_close(gpu, ref, rel, extra)
    if not ok and nbad <= outliers:
        g = np.asarray(gpu, dtype=np.float64).reshape(-1)
        r = np.asarray(ref, dtype=np.float64).reshape(-1)
        ok = bool(np.max(np.abs(g - r)) <= np.max(np.abs(r)))
    if not ok:
        g = np.asarray(gpu, dtype=np.float64).reshape(-1)
        r = np.asarray(ref, dtype=np.float64).reshape(-1)
        order = np.argsort(-np.abs(g - r) / np.maximum(np.abs(r), 1e-2 * np.max(np.abs(r))))[:4]
        detail = ", ".join(f"[{i}] gpu {g[i]:.6g} ref {r[i]:.6g}" for i in order)
        raise AssertionError(f"{what}: {nbad} elements outside {rel} (worst scaled err {worst:.3g}; max|ref| "
                             f"{np.max(np.abs(r)):.3g}): {detail}")


def assert_rel(gpu, ref, rel, atol=0.0, what=""):
    gpu = np.asarray(gpu, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    err = np.abs(gpu - ref)
    tol = rel * np.abs(ref) + atol
    bad = err > tol
    assert not bad.any(), f"{what}: {int(bad.sum())}/{bad.size} outside rel {rel} atol {atol}; max err {err.max():.3g}"
