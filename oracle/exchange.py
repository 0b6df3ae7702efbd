"""Generator-gradient exchange: grouping, Alg. 1 ring, outer ring, modes.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Paper:
* Alg. 1: N ranks, rank i sends g_i to rank i+1, receives
  g_{i-1} from rank i-1, and accumulates.  Read (R10) as a pass-along ring:
  in hop j = 1..N-1 every rank forwards to its successor the packet that
  originated j-1 ranks behind it, so after N-1 hops every rank holds every
  packet; each rank then sums them in ascending origin-rank order, which
  makes the result identical on every member and equal to the plain sum.
* Grouping (Tab. II): contiguous inner groups reduce every epoch;
  an outer group made of the first rank of each inner group ("fixed to be
  rank 0") reduces every h epochs (R13: fires iff (t+1) % h == 0; the
  outer result is used by the leader only, no rebroadcast).
* Modes (Tab. III): ARAR (ungrouped), ARAR-ARAR, RMA-ARAR-ARAR.
  Numerically the last two are the same reduction (they differ in the
  transport), and so is the one-hop all-gather variant of the inner group
  (mode 5: every member receives every packet directly); mode NONE is the ensemble of P:131; SYNC_ALLREDUCE is the
  synchronous baseline sum over all ranks.
* Only generator *weight* gradients travel.
* Staleness (R12): with s = 1 a rank combines its own packet of step t with
  the other members' packets of step t-1 (zero before step 0).
"""
import numpy as np

MODE_NONE = 0
MODE_ARAR = 1
MODE_ARAR_ARAR = 2
MODE_RMA_ARAR_ARAR = 3
MODE_SYNC_ALLREDUCE = 4
MODE_RMA_ALLGATHER = 5  # §8(f) row 3: the inner group by a one-hop all-gather -- same sums as 2 / 3
MODE_RMA_CHUNKED = 6    # §8(f) row 3: chunked reduce-scatter + all-gather (staleness 0) -- same sums as 2 / 3


def group_layout(world, group_size):
    """Inner groups of contiguous ranks (the last may be smaller, as in the
    SPEC's (10, 4) example) and the leaders = first rank of each group."""
    groups = [list(range(a, min(a + group_size, world))) for a in range(0, world, group_size)]
    leaders = [g[0] for g in groups]
    return groups, leaders


def outer_fires(step, h):
    """Outer-group exchange at the end of epoch t iff (t + 1) mod h == 0."""
    return h > 0 and (step + 1) % h == 0


def ring_pass_along(packets):
    """Simulate the N-1 hops of the pass-along ring over one group.

    packets: list of arrays, packets[i] = packet of the i-th member.
    Returns held[i] = dict origin -> packet, as held by member i after the
    last hop (every member must hold every origin).  The hop schedule is
    simulated explicitly so that a test can check delivery and hop counts.
    """
    n = len(packets)
    held = [{i: packets[i]} for i in range(n)]
    hops = 0
    for j in range(1, n):
        sends = []
        for i in range(n):
            origin = (i - j + 1) % n          # forwarded by member i at hop j
            sends.append(((i + 1) % n, origin, held[i][origin]))
        for dst, origin, pkt in sends:
            assert origin not in held[dst]
            held[dst][origin] = pkt
        hops += 1
    return held, hops


def fold_ascending(held_by_origin, origins):
    """((P_o0 + P_o1) + P_o2) + ... over the origins in ascending order."""
    acc = None
    for o in sorted(origins):
        acc = held_by_origin[o].copy() if acc is None else acc + held_by_origin[o]
    return acc


def ring_all_reduce(packets):
    """Every member's ring result (the ascending fold of all packets)."""
    held, _ = ring_pass_along(packets)
    return [fold_ascending(h, range(len(packets))) for h in held]


def reduce_step(mode, world, group_size, h, staleness, reduce_mean, t, history):
    """Reduced packet R_r^t of every rank at step t.

    history[t'][r] = packet P_r^{t'} for t' <= t (t' < 0 means zero).
    Returns list R[r].
    """
    def pkt(tt, r):
        if tt < 0:
            return np.zeros_like(history[t][r])
        return history[tt][r]

    if mode == MODE_NONE:
        return [pkt(t, r).copy() for r in range(world)]
    if mode == MODE_SYNC_ALLREDUCE:
        total = fold_ascending({r: pkt(t, r) for r in range(world)}, range(world))
        if reduce_mean:
            total = total / world
        return [total.copy() for _ in range(world)]
    if mode == MODE_ARAR:
        group_size, h = world, 0
    groups, leaders = group_layout(world, group_size)
    R = [None] * world
    for g in groups:
        for r in g:
            # what member r holds after the ring: own packet of step t, the
            # others' packets of step t - s
            held = {o: (pkt(t, o) if o == r else pkt(t - staleness, o)) for o in g}
            R[r] = fold_ascending(held, g)
            if reduce_mean:
                R[r] = R[r] / len(g)
    if outer_fires(t, h) and len(leaders) > 1:
        # the leaders' ring: every leader ends with the ascending fold of
        # the leaders' inner results of step t (Alg. 1 over the outer group)
        inner = {l: R[l] for l in leaders}
        outer = fold_ascending(inner, leaders)
        for l in leaders:
            R[l] = outer / len(leaders) if reduce_mean else outer.copy()
    return R
