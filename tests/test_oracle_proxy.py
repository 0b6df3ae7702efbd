"""Pins for oracle/proxy.py: closed forms, analytic moments / CDF, brute force,
finite differences."""
import numpy as np
import pytest
from scipy import stats

from oracle import philox as px
from oracle import proxy

P_TRUE = [1.0, 1.0, 0.5, 2.0, 0.5, 1.0]   # R3 (constrained space)


def test_constrain_zero_and_threshold():
    c = proxy.constrain(np.zeros((1, 6)))
    ln2 = np.log(2.0)
    assert np.allclose(c.reshape(-1), [0, ln2, ln2, 0, ln2, ln2], rtol=0, atol=1e-15)
    # above the threshold softplus is the identity; far below it is ~e^x > 0
    c = proxy.constrain(np.array([[3.0, 25.0, -30.0, -1.0, 20.5, 0.0]]))
    assert c[0, 0, 1] == 25.0 and c[0, 1, 1] == 20.5
    assert 0 < c[0, 0, 2] < 1e-12
    assert c[0, 0, 0] == 3.0 and c[0, 1, 0] == -1.0


def test_constrain_monotone_validity():
    rng = np.random.default_rng(0)
    c = proxy.constrain(rng.normal(scale=10, size=(10000, 6)))
    assert np.all(c[:, :, 1] >= 0) and np.all(c[:, :, 1] + 2 * c[:, :, 2] >= 0)


def test_quantile_closed_forms():
    assert proxy.quantile(0.0, 1.5, 2.0, 3.0) == 1.5          # Q(0) = c0
    u = np.linspace(0, 1, 11)
    assert np.array_equal(proxy.quantile(u, 0.0, 1.0, 0.0), u)  # uniform
    assert proxy.quantile(1.0, 1.0, 1.0, 1.0) == 3.0


def test_sample_constant_params():
    c = np.zeros((4, 2, 3))
    c[:, 0, 0] = 1.25
    c[:, 1, 0] = -3.0
    u = proxy.fake_uniforms(1, 0, 0, 4 * 5)
    y = proxy.sample_events(c, 5, u)
    assert np.all(y[:, 0] == 1.25) and np.all(y[:, 1] == -3.0)


def test_sample_is_sample_major():
    # event e uses the parameters of sample e // m
    c = np.zeros((3, 2, 3))
    c[:, :, 0] = np.array([[10.0, 20.0], [30.0, 40.0], [50.0, 60.0]])
    u = proxy.fake_uniforms(1, 0, 0, 6)
    y = proxy.sample_events(c, 2, u)
    assert np.array_equal(y[:, 0], [10, 10, 30, 30, 50, 50])


def test_analytic_moments_at_true_params():
    # mean = c0 + c1/2 + c2/3 ; var = c1^2/12 + c1 c2/6 + 4 c2^2/45
    n = 1 << 20
    ref = proxy.make_reference(11, P_TRUE, n)
    exp_mean = [5.0 / 3.0, 31.0 / 12.0]
    exp_var = [17.0 / 90.0, 139.0 / 720.0]
    for o in range(2):
        assert abs(ref[:, o].mean() - exp_mean[o]) < 5 * np.sqrt(exp_var[o] / n)
        assert abs(ref[:, o].var() - exp_var[o]) < 5 * exp_var[o] * np.sqrt(2.0 / n) * 1.5
    # support [c0, c0 + c1 + c2]
    assert ref[:, 0].min() >= 1.0 and ref[:, 0].max() <= 2.5
    assert ref[:, 1].min() >= 2.0 and ref[:, 1].max() <= 3.5


def _cdf(y, c0, c1, c2):
    # F(y) = 2 (y - c0) / (c1 + sqrt(c1^2 + 4 c2 (y - c0))), the inverse of Q
    d = np.clip(y - c0, 0, None)
    return np.clip(2 * d / (c1 + np.sqrt(c1 * c1 + 4 * c2 * d)), 0, 1)


def test_analytic_cdf_chi2():
    n = 1 << 18
    ref = proxy.make_reference(5, P_TRUE, n)
    for o in range(2):
        c0, c1, c2 = P_TRUE[3 * o:3 * o + 3]
        edges = np.linspace(c0, c0 + c1 + c2, 33)
        obs, _ = np.histogram(ref[:, o], bins=edges)
        expct = n * np.diff(_cdf(edges, c0, c1, c2))
        chi2 = ((obs - expct) ** 2 / expct).sum()
        assert stats.chi2.sf(chi2, df=31) > 1e-4


def test_f32_sampler_matches_f64():
    rng = np.random.default_rng(1)
    c = proxy.constrain(rng.normal(size=(16, 6)))
    u = proxy.fake_uniforms(2, 3, 1, 16 * 8)
    y64 = proxy.sample_events(c, 8, u)
    y32 = proxy.sample_events_f32(c.astype(np.float32), 8, u)
    assert np.allclose(y32, y64, rtol=2e-6, atol=1e-6)


def test_histogram_brute_force_and_edges():
    rng = np.random.default_rng(2)
    y = rng.uniform(-1, 5, size=5000).astype(np.float32)
    h = proxy.histogram_f32(y, 0.0, 4.0, 64)
    # brute force: per value, classify with a python loop in fp32
    hb = np.zeros(66, dtype=np.int64)
    scale = np.float32(64) / (np.float32(4.0) - np.float32(0.0))
    for v in y:
        t = (np.float32(v) - np.float32(0.0)) * scale
        if not t >= 0:
            hb[0] += 1
        elif t >= 64:
            hb[65] += 1
        else:
            hb[int(np.floor(t)) + 1] += 1
    assert np.array_equal(h, hb)
    assert h.sum() == y.size
    # explicit edges
    e = proxy.histogram_f32(np.array([0.0, 4.0, -1e-7, np.nan, 0.0625, 3.9999], dtype=np.float32), 0.0, 4.0, 64)
    assert e[1] == 1 and e[2] == 1 and e[64] == 1    # 0 -> bin 1 ; 1/16 -> bin 2 ; 3.9999 -> bin 64
    assert e[65] == 1 and e[0] == 2                  # hi -> overflow ; below lo and NaN -> underflow


def test_lemire_index_brute_force():
    w = np.array([0, 1, 2 ** 31, 2 ** 32 - 1, 123456789], dtype=np.uint64)
    for n in (1, 7, 1 << 20, 3 * 10 ** 6):
        got = proxy.lemire_index(w, n)
        assert [int(g) for g in got] == [(int(x) * n) >> 32 for x in w]
        assert got.max() <= n - 1


def test_shard_rows_are_reference_rows_and_uniform():
    n_ref, n_s = 4096, 2048
    ref = proxy.make_reference(3, P_TRUE, n_ref)
    idx = proxy.shard_indices(3, 2, n_ref, n_s)
    shard = ref[idx]
    refset = {tuple(r) for r in ref}
    assert all(tuple(r) in refset for r in shard)
    assert len(shard) == n_ref // 2
    big = proxy.shard_indices(3, 0, 64, 1 << 16)
    cnt = np.bincount(big, minlength=64)
    assert stats.chisquare(cnt).pvalue > 1e-4


def test_real_indices_uniform_and_in_range():
    idx = proxy.real_indices(9, 4, 1, 100, 1 << 16)
    assert idx.min() >= 0 and idx.max() < 100
    assert stats.chisquare(np.bincount(idx, minlength=100)).pvalue > 1e-4


def test_sampler_backward_finite_differences():
    rng = np.random.default_rng(4)
    k, m = 5, 7
    raw = rng.normal(size=(k, 6))
    u = proxy.fake_uniforms(4, 0, 0, k * m)
    dy = rng.normal(size=(k * m, 2))
    dc, draw = proxy.sampler_backward(dy, u, raw, m)

    def f(r):
        return float(np.sum(dy * proxy.sample_events(proxy.constrain(r), m, u)))

    h = 1e-6
    fd = np.zeros_like(raw)
    for s in range(k):
        for j in range(6):
            rp = raw.copy(); rp[s, j] += h
            rm = raw.copy(); rm[s, j] -= h
            fd[s, j] = (f(rp) - f(rm)) / (2 * h)
    assert np.allclose(draw, fd, rtol=1e-6, atol=1e-8)
    # dQ/dc = (1, u, u^2) exactly: dc for a single event equals dy * u^j
    dc1, _ = proxy.sampler_backward(np.array([[2.0, 3.0]]), np.array([[0.5, 0.25]]), np.zeros((1, 6)), 1)
    assert np.array_equal(dc1[0, 0], [2.0, 1.0, 0.5]) and np.array_equal(dc1[0, 1], [3.0, 0.75, 0.1875])
