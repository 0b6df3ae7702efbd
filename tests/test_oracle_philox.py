"""Pins for oracle/philox.py against external known answers and closed forms."""
import os

import numpy as np
import pytest
from scipy import stats

from oracle import philox as px

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "philox_kat.txt")


def _kats():
    rows = []
    with open(GOLDEN) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            v = [int(t, 16) for t in line.split()]
            rows.append((v[:4], v[4:6], v[6:10]))
    return rows


@pytest.mark.parametrize("ctr,key,expect", _kats())
def test_philox_known_answers(ctr, key, expect):
    out = px.philox4x32_10(*[np.uint64(c) for c in ctr], key[0], key[1])
    assert [int(o) for o in out] == expect


def test_word_stream_numbering():
    # word i is word (i % 4) of Philox(ctr = (i // 4, step, rank, stream))
    seed = 0x0123456789ABCDEF
    w = px.words(seed, 5, 7, 3, 2, 11)  # words 2..12
    k0, k1 = px.seed_key(seed)
    for j, i in enumerate(range(2, 13)):
        out = px.philox4x32_10(np.uint64(i // 4), np.uint64(7), np.uint64(3), np.uint64(5), k0, k1)
        assert int(w[j]) == int(out[i % 4])


def test_uniform_endpoints_exact():
    u = px.uniform_open01(np.array([0, 511, 512, 2 ** 31, 2 ** 32 - 1], dtype=np.uint64))
    assert u[0] == 2.0 ** -24
    assert u[1] == 2.0 ** -24            # the 9 low bits are dropped
    assert u[2] == 3 * 2.0 ** -24
    assert u[3] == 0.5 + 2.0 ** -24
    assert u[4] == 1.0 - 2.0 ** -24
    # exactly representable in fp32
    assert np.all(u.astype(np.float32).astype(np.float64) == u)


def test_box_muller_closed_form():
    # ua = e^{-1/2} -> r = 1 ; ub = 1/4 -> theta = pi/2 -> (0, 1)
    zc, zs = px.box_muller(np.array([np.exp(-0.5)]), np.array([0.25]))
    assert abs(zc[0]) < 1e-15 and abs(zs[0] - 1.0) < 1e-15
    # ub = 1/2 -> theta = pi -> (-r, 0); ua = e^{-2} -> r = 2
    zc, zs = px.box_muller(np.array([np.exp(-2.0)]), np.array([0.5]))
    assert abs(zc[0] + 2.0) < 1e-14 and abs(zs[0]) < 1e-14


def test_normals_are_standard_normal():
    n = 1 << 18
    z = px.normals(7, px.STREAM_NOISE, 0, 0, n)
    assert abs(z.mean()) < 4.0 / np.sqrt(n)
    assert abs(z.var() - 1.0) < 4.0 * np.sqrt(2.0 / n)
    # Kolmogorov-Smirnov against the library normal CDF
    assert stats.kstest(z, "norm").pvalue > 1e-3


def test_uniform_words_are_uniform():
    w = px.words(3, px.STREAM_FAKE, 0, 0, 0, 1 << 18)
    u = px.uniform_open01(w)
    assert stats.kstest(u, "uniform").pvalue > 1e-3


def test_streams_are_distinct():
    a = px.words(1, px.STREAM_FAKE, 0, 0, 0, 64)
    b = px.words(1, px.STREAM_REAL, 0, 0, 0, 64)
    c = px.words(1, px.STREAM_FAKE, 0, 1, 0, 64)
    d = px.words(1, px.STREAM_FAKE, 1, 0, 0, 64)
    assert not np.array_equal(a, b) and not np.array_equal(a, c) and not np.array_equal(a, d)
