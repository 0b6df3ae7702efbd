"""Ensemble response, normalised residuals and the split-batch rule.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Paper:
  Eq. 6  r_hat_i = (p_i - p_hat_i) / p_i
  Eq. 7  p_hat = (1/M) sum_{i=1..M} G_i(n)
  Eq. 8  sigma = sqrt((1/M) sum_{i=1..M} [G_i(n) - p_hat]^2)
  P:332              "For a batch of k noise vectors we simply report the
                     average of p_hat and sigma across the batch dimension k"
  Eq. 10 # predicted parameter samples = floor(1024 / N(ranks))

G_i(n) is generator i's prediction for noise vector n, here the constrained
parameters c of the proxy (R1); p is the loop-closure truth p* (P:272).
Everything in float64, written as the equations read, loops over the
ensemble members in order.
"""
import numpy as np


def ensemble_mean(preds):
    """Eq. 7 for every noise vector: preds [M][k][P] -> p_hat [k][P]."""
    preds = np.asarray(preds, dtype=np.float64)
    M = preds.shape[0]
    acc = np.zeros(preds.shape[1:], dtype=np.float64)
    for i in range(M):
        acc += preds[i]
    return acc / M


def ensemble_std(preds):
    """Eq. 8 for every noise vector (population form, 1/M): -> sigma [k][P]."""
    preds = np.asarray(preds, dtype=np.float64)
    M = preds.shape[0]
    mean = ensemble_mean(preds)
    acc = np.zeros(preds.shape[1:], dtype=np.float64)
    for i in range(M):
        acc += (preds[i] - mean) ** 2
    return np.sqrt(acc / M)


def ensemble_response(preds):
    """Eq. 7 and Eq. 8 averaged over the k noise vectors -> (p_hat [P], sigma [P])."""
    return ensemble_mean(preds).mean(axis=0), ensemble_std(preds).mean(axis=0)


def normalized_residual(p, p_hat):
    """Eq. 6: r_hat_i = (p_i - p_hat_i) / p_i."""
    p = np.asarray(p, dtype=np.float64)
    return (p - np.asarray(p_hat, dtype=np.float64)) / p


def split_batch_samples(n_ranks, total=1024):
    """Eq. 10: the predicted parameter samples per rank, floor(1024 / N(ranks))."""
    return total // n_ranks
