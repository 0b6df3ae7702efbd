"""Pins for oracle/exchange.py: the paper's grouping example, counting
identities, and the ring = plain-sum invariant."""
import json
import os

import numpy as np

from oracle import exchange as xc

PAPER = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))


def test_grouping_paper_example():
    ex = PAPER["grouping_example"]
    groups, leaders = xc.group_layout(ex["world"], 4)
    assert groups == ex["inner"]
    assert leaders == [0, 4, 8] and len(leaders) == ex["outer_size"]


def test_grouping_other_layouts():
    assert xc.group_layout(8, 4) == ([[0, 1, 2, 3], [4, 5, 6, 7]], [0, 4])
    assert xc.group_layout(4, 4) == ([[0, 1, 2, 3]], [0])
    assert xc.group_layout(10, 4) == ([[0, 1, 2, 3], [4, 5, 6, 7], [8, 9]], [0, 4, 8])
    assert xc.group_layout(3, 1) == ([[0], [1], [2]], [0, 1, 2])


def test_outer_fire_counts():
    assert sum(xc.outer_fires(t, 10) for t in range(100)) == 10
    assert not xc.outer_fires(8, 10) and xc.outer_fires(9, 10)
    assert sum(xc.outer_fires(t, PAPER["outer_h"]["value"]) for t in range(PAPER["epochs"]["value"])) == 100
    assert all(xc.outer_fires(t, 1) for t in range(5))
    assert not any(xc.outer_fires(t, 0) for t in range(5))


def test_ring_delivers_every_packet_in_n_minus_1_hops():
    for n in range(1, 9):
        pk = [np.full(3, float(i)) for i in range(n)]
        held, hops = xc.ring_pass_along(pk)
        assert hops == n - 1
        for h in held:
            assert sorted(h) == list(range(n))
            for o, p in h.items():
                assert np.array_equal(p, pk[o])


def test_ring_small_example_and_identity():
    out = xc.ring_all_reduce([np.array([1.0]), np.array([2.0]), np.array([3.0])])
    assert all(o[0] == 6.0 for o in out)
    x = np.random.default_rng(0).normal(size=5)
    assert np.array_equal(xc.ring_all_reduce([x])[0], x)


def test_ring_equals_plain_sum_bitwise():
    rng = np.random.default_rng(1)
    for n in (2, 3, 5, 8, 16):
        pk = [rng.normal(size=1000) for _ in range(n)]
        plain = pk[0].copy()
        for p in pk[1:]:
            plain = plain + p
        for o in xc.ring_all_reduce(pk):
            assert np.array_equal(o, plain)
        assert np.allclose(plain, np.sum(pk, axis=0), rtol=1e-13, atol=1e-13)


def test_reduce_step_modes():
    rng = np.random.default_rng(2)
    world = 8
    hist = {t: [rng.normal(size=16) for _ in range(world)] for t in range(3)}
    t = 2
    tot = sum(hist[t][r] for r in range(world))
    # s = 0 ungrouped ring == sync allreduce (sum)
    a = xc.reduce_step(xc.MODE_ARAR, world, world, 0, 0, 0, t, hist)
    s = xc.reduce_step(xc.MODE_SYNC_ALLREDUCE, world, world, 0, 0, 0, t, hist)
    for r in range(world):
        assert np.array_equal(a[r], s[r]) and np.allclose(a[r], tot, rtol=1e-13, atol=1e-13)
    # g = world grouped == ungrouped
    g = xc.reduce_step(xc.MODE_ARAR_ARAR, world, world, 10, 0, 0, t, hist)
    assert all(np.array_equal(g[r], a[r]) for r in range(world))
    # NONE == own packet ; g = 1 == own packet
    n = xc.reduce_step(xc.MODE_NONE, world, world, 0, 0, 0, t, hist)
    g1 = xc.reduce_step(xc.MODE_ARAR_ARAR, world, 1, 0, 0, 0, t, hist)
    assert all(np.array_equal(n[r], hist[t][r]) and np.array_equal(g1[r], hist[t][r]) for r in range(world))
    # grouped without outer fire: equal within groups, sum of the group
    g4 = xc.reduce_step(xc.MODE_RMA_ARAR_ARAR, world, 4, 10, 0, 0, t, hist)
    for grp in ([0, 1, 2, 3], [4, 5, 6, 7]):
        ref = sum(hist[t][r] for r in grp)
        for r in grp:
            assert np.array_equal(g4[r], g4[grp[0]]) and np.allclose(g4[r], ref, rtol=1e-13, atol=1e-13)
    # outer fire at t = 2 with h = 3: leaders get the global sum, others keep the inner sum
    g4o = xc.reduce_step(xc.MODE_RMA_ARAR_ARAR, world, 4, 3, 0, 0, t, hist)
    assert np.allclose(g4o[0], tot, rtol=1e-13, atol=1e-13) and np.allclose(g4o[4], tot, rtol=1e-13, atol=1e-13)
    assert np.array_equal(g4o[1], g4[1])
    # mean
    m = xc.reduce_step(xc.MODE_ARAR, world, world, 0, 0, 1, t, hist)
    assert np.allclose(m[0], tot / world, rtol=1e-13, atol=1e-13)


def test_reduce_step_staleness():
    world = 3
    hist = {0: [np.full(2, 1.0 + r) for r in range(world)], 1: [np.full(2, 10.0 + r) for r in range(world)]}
    r0 = xc.reduce_step(xc.MODE_ARAR, world, world, 0, 1, 0, 0, hist)
    # step 0 with s = 1: own packet only (others are from step -1 = zero)
    assert [float(x[0]) for x in r0] == [1.0, 2.0, 3.0]
    r1 = xc.reduce_step(xc.MODE_ARAR, world, world, 0, 1, 0, 1, hist)
    # rank 1 at step 1: P_0^0 + P_1^1 + P_2^0 = 1 + 11 + 3
    assert float(r1[1][0]) == 15.0 and float(r1[0][0]) == 10.0 + 2.0 + 3.0
