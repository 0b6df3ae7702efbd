"""Philox4x32-10 and the maps from its 32-bit words to uniforms and normals.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The paper draws its randomness through PyTorch, whose CUDA generator
is Philox4x32-10 (Salmon et al., "Parallel random numbers: as easy as 1, 2,
3", SC'11).  The counter layout is a reading (DESIGN.md R-RNG):

    key = (seed & 0xffffffff, seed >> 32)
    ctr = (index, step, rank, stream)

and a stream of 32-bit words is numbered so that word i is word (i % 4) of
Philox(ctr = (i // 4, step, rank, stream)).

Pinned by tests/test_oracle_philox.py against the Random123 known-answer
vectors (tests/golden/philox_kat.txt).
"""
import numpy as np

M0 = 0xD2511F53
M1 = 0xCD9E8D57
W0 = 0x9E3779B9
W1 = 0xBB67AE85
MASK32 = 0xFFFFFFFF

# stream identifiers (DESIGN.md R-RNG)
STREAM_REF = 0
STREAM_SHARD = 1
STREAM_INIT_G = 2
STREAM_INIT_D = 3
STREAM_NOISE = 4
STREAM_FAKE = 5
STREAM_REAL = 6


def _mulhilo(a, b):
    """Full 64-bit product of two 32-bit words -> (hi32, lo32)."""
    p = a.astype(np.uint64) * np.uint64(b)
    return (p >> np.uint64(32)) & np.uint64(MASK32), p & np.uint64(MASK32)


def philox4x32_10(c0, c1, c2, c3, k0, k1):
    """Ten Philox4x32 rounds (SC'11, Sec. 3.2), vectorised over the counters.

    One round:  (hi0, lo0) = M0 * c0 ; (hi1, lo1) = M1 * c2
                c <- (hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0)
                k <- k + (W0, W1)   (mod 2^32)
    Returns four uint32 arrays.
    """
    shape = np.broadcast(c0, c1, c2, c3).shape
    c = [np.broadcast_to(np.asarray(x, dtype=np.uint64), shape).copy() for x in (c0, c1, c2, c3)]
    k0 = np.uint64(int(k0) & MASK32)
    k1 = np.uint64(int(k1) & MASK32)
    for _ in range(10):
        hi0, lo0 = _mulhilo(c[0], M0)
        hi1, lo1 = _mulhilo(c[2], M1)
        c = [hi1 ^ c[1] ^ k0, lo1, hi0 ^ c[3] ^ k1, lo0]
        k0 = np.uint64((int(k0) + W0) & MASK32)
        k1 = np.uint64((int(k1) + W1) & MASK32)
    return tuple(x.astype(np.uint32) for x in c)


def seed_key(seed):
    seed = int(seed) & 0xFFFFFFFFFFFFFFFF
    return seed & MASK32, seed >> 32


def words(seed, stream, step, rank, first, count):
    """Words [first, first+count) of the (step, rank, stream) word stream."""
    k0, k1 = seed_key(seed)
    if count <= 0:
        return np.zeros(0, dtype=np.uint32)
    c_first = first // 4
    c_last = (first + count - 1) // 4
    calls = np.arange(c_first, c_last + 1, dtype=np.uint64)
    r = philox4x32_10(calls, np.uint64(step), np.uint64(rank), np.uint64(stream), k0, k1)
    flat = np.stack(r, axis=1).reshape(-1)  # word 4*call + lane
    off = first - 4 * c_first
    return flat[off:off + count].astype(np.uint32)


def uniform_open01(w):
    """u = (2*(w >> 9) + 1) * 2^-24: the 23 high bits of w, centred in its
    cell, giving u in (0, 1) with u never 0 or 1 (DESIGN.md R-UNIF).
    The value is exactly representable in fp32 and fp64."""
    w = np.asarray(w, dtype=np.uint64)
    return ((w >> np.uint64(9)).astype(np.float64) * 2.0 + 1.0) * 2.0 ** -24


def box_muller(ua, ub):
    """Standard normal pair (r cos(2 pi ub), r sin(2 pi ub)), r = sqrt(-2 ln ua)."""
    r = np.sqrt(-2.0 * np.log(ua))
    t = 2.0 * np.pi * ub
    return r * np.cos(t), r * np.sin(t)


def normals(seed, stream, step, rank, count):
    """count standard normals; normal f uses words (2*(f//2), 2*(f//2)+1):
    even f -> cos branch, odd f -> sin branch."""
    npairs = (count + 1) // 2
    w = words(seed, stream, step, rank, 0, 2 * npairs)
    ua = uniform_open01(w[0::2])
    ub = uniform_open01(w[1::2])
    zc, zs = box_muller(ua, ub)
    z = np.empty(2 * npairs, dtype=np.float64)
    z[0::2] = zc
    z[1::2] = zs
    return z[:count]
