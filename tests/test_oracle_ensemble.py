"""Pins of oracle/ensemble.py (Eq. 6, 7, 8, 10) against
closed forms that a slip in the oracle (a dropped 1/M, a sample instead of a
population variance, a pooled instead of a batch-averaged sigma, a flipped
residual sign) would break."""
import numpy as np
import pytest

from oracle import ensemble as E


def test_identical_generators_have_zero_spread():
    rng = np.random.default_rng(1)
    one = rng.normal(size=(7, 6))
    preds = np.stack([one] * 5)
    p_hat, sigma = E.ensemble_response(preds)
    np.testing.assert_allclose(p_hat, one.mean(axis=0), rtol=0, atol=1e-15)
    np.testing.assert_allclose(sigma, np.zeros(6), rtol=0, atol=1e-15)  # (5x)/5 rounds


def test_symmetric_pair_gives_the_half_distance():
    # two members x +- d_s: p_hat = x exactly, sigma_s = |d_s| (population form);
    # a sample (1/(M-1)) variance would give |d_s| * sqrt(2)
    x = np.array([[1.0, -2.0, 3.0], [0.5, 0.25, 4.0]])
    d = np.array([[0.5, 0.25, 1.0], [2.0, 0.125, 0.75]])
    preds = np.stack([x + d, x - d])
    np.testing.assert_array_equal(E.ensemble_mean(preds), x)
    np.testing.assert_array_equal(E.ensemble_std(preds), d)


def test_three_members_closed_form():
    # {a, a, a + 3h}: mean a + h, variance (h^2 + h^2 + (2h)^2) / 3 = 2 h^2
    a, h = 1.25, 0.5
    preds = np.array([[[a]], [[a]], [[a + 3 * h]]])
    p_hat, sigma = E.ensemble_response(preds)
    assert p_hat[0] == pytest.approx(a + h, abs=1e-15)
    assert sigma[0] == pytest.approx(h * np.sqrt(2.0), rel=1e-15)


def test_sigma_is_averaged_over_the_batch_not_pooled():
    # noise vector 0: members {0, 2} (sigma 1); vector 1: {10, 10} (sigma 0).
    # P:332 reports the batch average of sigma = 0.5; the pooled std over
    # all 4 predictions would be ~4.5
    preds = np.array([[[0.0], [10.0]], [[2.0], [10.0]]])
    p_hat, sigma = E.ensemble_response(preds)
    assert p_hat[0] == pytest.approx(5.5)
    assert sigma[0] == pytest.approx(0.5)


def test_residual_sign_and_scale():
    p = np.array([2.0, -4.0, 0.5])
    np.testing.assert_array_equal(E.normalized_residual(p, p), np.zeros(3))
    np.testing.assert_array_equal(E.normalized_residual(p, np.zeros(3)), np.ones(3))
    # over-prediction gives a negative residual (Eq. 6: (p - p_hat) / p)
    assert E.normalized_residual([2.0], [2.5])[0] == pytest.approx(-0.25)


def test_split_batch_rule():
    # Eq. 10 and the paper's two quoted batch sizes: 1024 samples x 100 events
    # = 102,400 on one GPU and 5,100 at 20 ranks (floor(1024/20) = 51)
    assert E.split_batch_samples(1) == 1024
    assert E.split_batch_samples(20) == 51
    assert E.split_batch_samples(20) * 100 == 5100
    assert E.split_batch_samples(3) == 341
