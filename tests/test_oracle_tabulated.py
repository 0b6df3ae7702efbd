"""Pins of oracle/tabulated.py (reading R32) against closed forms, exact
special cases, the continuous limit and finite differences of its own
forward -- chosen so that a dropped term, a wrong index or sign, a missing
normalisation or a wrong chain factor fails one of them."""
import math

import numpy as np
import pytest
from scipy import special

from oracle import tabulated as T


def _raw_for(w, b, c):
    """Inverse of constrain: (w, b, c) -> (r0, r1, r2)."""
    return np.array([math.log(w / (1.0 - w)), math.log(math.expm1(b)), math.log(math.expm1(c))])


def test_constrain_maps_as_stated():
    w, b, c = T.constrain([0.3, -1.2, 2.5])
    assert w == pytest.approx(1.0 / (1.0 + math.exp(-0.3)))
    assert b == pytest.approx(math.log1p(math.exp(-1.2)))
    assert c == pytest.approx(math.log1p(math.exp(2.5)))
    np.testing.assert_allclose(T.constrain(_raw_for(0.25, 1.5, 3.0)), (0.25, 1.5, 3.0), rtol=1e-12)


def test_table_is_a_cdf():
    F = T.cdf_table(0.3, 0.7, 2.2, 257)
    assert F[0] == 0.0 and F[-1] == 1.0
    assert np.all(np.diff(F) > 0)


def test_density_integrates_to_the_beta_function():
    # both mirror components integrate to B(b+1, c+1) (the normaliser of R32)
    for (w, b, c) in ((0.3, 1.5, 2.0), (0.9, 2.5, 1.25), (0.5, 1.0, 1.0)):
        S = T.trapezoid_cumsum(T.density(np.linspace(0, 1, 20001), w, b, c), 20001)
        assert S[-1] == pytest.approx(special.beta(b + 1, c + 1), rel=1e-7)


def test_tabulated_mean_converges_to_the_beta_moment():
    for (w, b, c) in ((0.3, 1.5, 2.0), (0.9, 2.5, 1.25), (0.1, 3.0, 1.0)):
        m_exact = T.analytic_mean(w, b, c)
        errs = [abs(T.tabulated_mean(T.cdf_table(w, b, c, G)) - m_exact) for G in (65, 257, 1025)]
        assert errs[-1] < 5e-6
        assert errs[1] < errs[0] and errs[2] < errs[1]   # converges with the grid


def test_uniform_density_inverts_to_the_identity():
    # b = c = 0 (the density helper accepts them; softplus never returns 0): f = 1, F_i = t_i, x = u
    F = T.trapezoid_cumsum(T.density(np.linspace(0, 1, 33), 0.6, 0.0, 0.0), 33)
    F = F / F[-1]
    for u in (1e-7, 0.1, 0.5, 0.73, 1 - 1e-7):
        assert T.invert(F, u) == pytest.approx(u, abs=1e-15)


def test_linear_density_has_an_exact_table():
    # w = 1, b = 1, c = 0: f = t, the trapezoid is exact, F_i = t_i^2; at the
    # nodes the inverse is sqrt(u) exactly; in between, linear interpolation
    G = 17
    t = np.linspace(0, 1, G)
    S = T.trapezoid_cumsum(T.density(t, 1.0, 1.0, 0.0), G)
    F = S / S[-1]
    np.testing.assert_allclose(F, t * t, rtol=0, atol=1e-15)
    for i in (1, 5, 16):
        assert T.invert(F, t[i] ** 2 * (1 - 1e-15)) == pytest.approx(t[i], abs=1e-12)
    u = (t[3] ** 2 + t[4] ** 2) / 2
    assert T.invert(F, u) == pytest.approx((t[3] + t[4]) / 2, abs=1e-15)


def test_mirror_symmetry():
    # (w, b, c) and (1 - w, c, b) are the same density
    np.testing.assert_allclose(T.cdf_table(0.3, 0.8, 2.5, 129), T.cdf_table(0.7, 2.5, 0.8, 129), rtol=0, atol=1e-15)
    # and w -> 1 - w with b = c changes nothing
    np.testing.assert_allclose(T.cdf_table(0.2, 1.3, 1.3, 65), T.cdf_table(0.8, 1.3, 1.3, 65), rtol=0, atol=1e-15)


def test_table_gradients_match_finite_differences():
    w, b, c, G, h = 0.35, 1.2, 2.7, 129, 1e-6
    dF = T.cdf_table_grads(w, b, c, G)
    for j, name in enumerate("wbc"):
        p = [w, b, c]
        pp, pm = list(p), list(p)
        pp[j] += h
        pm[j] -= h
        fd = (T.cdf_table(*pp, G) - T.cdf_table(*pm, G)) / (2 * h)
        np.testing.assert_allclose(dF[j], fd, rtol=1e-6, atol=1e-9, err_msg=name)


def test_sampler_backward_matches_finite_differences():
    rng = np.random.default_rng(3)
    k, m, G, h = 2, 7, 65, 1e-6
    raw = rng.normal(0.0, 0.8, (k, 6))
    u = rng.uniform(0.01, 0.99, (k * m, 2))
    dy = rng.normal(size=(k * m, 2))
    draw = T.sampler_backward(raw, m, u, dy, G)
    loss = lambda r: float(np.sum(dy * T.sample_events(r, m, u, G)))  # noqa: E731
    for s in range(k):
        for j in range(6):
            rp, rm = raw.copy(), raw.copy()
            rp[s, j] += h
            rm[s, j] -= h
            assert draw[s, j] == pytest.approx((loss(rp) - loss(rm)) / (2 * h), rel=1e-5, abs=1e-8)


def test_events_follow_their_sample_and_observable():
    # y[e][o] inverts sample (e // m)'s table of observable o: sample 0's
    # observable 0 is the mirror pair of sample 1's (the same density, so the
    # same events), observable 1 differs between the samples
    raw = np.vstack([np.r_[_raw_for(0.2, 2.0, 0.5), _raw_for(0.5, 1.0, 1.0)],
                     np.r_[_raw_for(0.8, 0.5, 2.0), _raw_for(0.3, 3.0, 1.5)]])
    u = np.array([[0.3, 0.6], [0.05, 0.9], [0.5, 0.5]] * 2)
    G = 129
    y = T.sample_events(raw, 3, u, G)
    np.testing.assert_allclose(y[:3, 0], y[3:, 0], rtol=0, atol=1e-12)
    F1 = T.cdf_table(*T.constrain(raw[1, 3:]), G)
    np.testing.assert_array_equal(y[3:, 1], [T.invert(F1, v) for v in u[3:, 1]])
    assert np.all(np.abs(y[:3, 1] - y[3:, 1]) > 1e-3)
