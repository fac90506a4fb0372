"""Pins for oracle.dispatch (Alg. A2 line 7): hand-worked DRR orders, the DRR deficit
lemma and fairness bound, conservation, and the release-time rule of reading c22."""
import math
import random

import pytest

from conftest import read_golden
from oracle import dispatch as dp


def parse_example(r):
    q = [int(x) for x in r["quanta"].split()]
    sizes = [[int(x) for x in flow.split()] for flow in r["sizes"].split("|")]
    order = [tuple(int(v) for v in pair.split(":")) for pair in r["order"].split()]
    return q, sizes, order


@pytest.mark.parametrize("row", read_golden("wdrr_examples.csv"), ids=lambda r: r["example"])
def test_hand_worked_orders(row):
    q, sizes, order = parse_example(row)
    assert dp.drr_order(sizes, q) == order


def rounds_trace(sizes, q):
    """Deficit counters after every visit, from a literal transcription kept apart from
    drr_order: [(round, flow, sent bytes so far, deficit, still backlogged)] and the order."""
    n = len(sizes)
    D, head, sent = [0] * n, [0] * n, [0] * n
    out, order, k = [], [], 0
    backlog = {i for i in range(n) if sizes[i]}
    while backlog:
        k += 1
        for i in sorted(backlog):
            D[i] += q[i]
            while head[i] < len(sizes[i]) and sizes[i][head[i]] <= D[i]:
                D[i] -= sizes[i][head[i]]
                sent[i] += sizes[i][head[i]]
                order.append((i, head[i]))
                head[i] += 1
            done = head[i] == len(sizes[i])
            if done:
                D[i] = 0
                backlog.discard(i)
            out.append((k, i, sent[i], D[i], not done))
    return out, order


def random_case(rng, n_max=5, len_max=40, size_max=9):
    n = rng.randint(1, n_max)
    sizes = [[rng.randint(1, size_max) for _ in range(rng.randint(0, len_max))] for _ in range(n)]
    Q = rng.randint(size_max, 3 * size_max)
    w = [rng.choice([1, 1.5, 2, 3, 7.25]) for _ in range(n)]
    return sizes, dp.quanta(w, Q), w


def test_deficit_lemma_and_service_per_round():
    """Shreedhar-Varghese Lemma 1: with q_i >= Max a backlogged flow ends every visit with
    0 <= D_i < Max, so after k rounds it has sent k*q_i - D_i, in (k*q_i - Max, k*q_i]."""
    rng = random.Random(7)
    for _ in range(300):
        sizes, q, _ = random_case(rng)
        mx = max([s for f in sizes for s in f], default=1)
        tr, order = rounds_trace(sizes, q)
        assert order == dp.drr_order(sizes, q)   # the transcription sends what the oracle sends
        for k, i, sent, D, backlogged in tr:
            if backlogged:
                assert 0 <= D < mx
                assert sent == k * q[i] - D


def test_fairness_bound_on_every_prefix():
    """DRR fairness (Shreedhar-Varghese Thm. 1, normalised): while flows i and j are both
    backlogged, |sent_i/q_i - sent_j/q_j| < 2 + Max/min(q_i, q_j) on every prefix of the order.
    A scheduler that drops the deficit between rounds, or scales quanta the wrong way, fails."""
    rng = random.Random(11)
    for _ in range(200):
        sizes, q, _ = random_case(rng)
        mx = max([s for f in sizes for s in f], default=1)
        sent = [0] * len(sizes)
        left = [len(f) for f in sizes]
        for f, p in dp.drr_order(sizes, q):
            sent[f] += sizes[f][p]
            left[f] -= 1
            live = [i for i in range(len(sizes)) if left[i] > 0]
            for a in live:
                for b in live:
                    assert abs(sent[a] / q[a] - sent[b] / q[b]) < 2 + mx / min(q[a], q[b])


def test_long_run_shares_follow_weights():
    """All flows backlogged with equal packets: byte shares converge to the weights."""
    w = [1.0, 2.0, 5.0]
    sizes = [[32] * 4000 for _ in w]
    order = dp.drr_order(sizes, dp.quanta(w, 256))
    first = order[:2000]
    cnt = [sum(1 for f, _ in first if f == i) for i in range(3)]
    for i in range(3):
        assert abs(cnt[i] / sum(cnt) - w[i] / sum(w)) < 0.01


def test_conservation_and_per_flow_order():
    rng = random.Random(3)
    for _ in range(200):
        sizes, q, _ = random_case(rng)
        order = dp.drr_order(sizes, q)
        assert sorted(order) == [(i, p) for i in range(len(sizes)) for p in range(len(sizes[i]))]
        for i in range(len(sizes)):
            ps = [p for f, p in order if f == i]
            assert ps == sorted(ps)


def test_single_flow_and_quanta():
    assert dp.drr_order([[5, 1, 7]], [7]) == [(0, 0), (0, 1), (0, 2)]
    assert dp.quanta([2.0, 1.0, 4.0], 1000) == [2000, 1000, 4000]
    assert dp.quanta([3.0, 7.0], 10) == [10, math.floor(10 * 7.0 / 3.0)]
    assert dp.default_quantum(32768) == 262144 and dp.default_quantum(1 << 20) == 1 << 20
    with pytest.raises(ValueError):
        dp.quanta([1.0, 0.0], 8)


def test_runs_and_entries_tile_the_order():
    rng = random.Random(5)
    for _ in range(100):
        sizes, q, _ = random_case(rng)
        order = dp.drr_order(sizes, q)
        rs = dp.runs(order)
        flat = [(f, p) for f, first, c in rs for p in range(first, first + c)]
        assert flat == order
        for a, b in zip(rs, rs[1:]):  # maximal runs
            assert not (a[0] == b[0] and a[1] + a[2] == b[1])
        for E in (1, 3, 8):
            ents = dp.entries(rs, E)
            assert all(1 <= c <= E for _, _, c in ents)
            assert [(f, p) for f, first, c in ents for p in range(first, first + c)] == order


def test_release_times_single_flow_closed_form():
    """c22 with one request: entry k starts after k*E packets of b bytes -> floor(k*E*b*1e6/r) us."""
    sizes = [[32768] * 100]
    r = 3.3e9
    ents = dp.entries(dp.runs(dp.drr_order(sizes, [262144])), 8)
    rel = dp.release_us(ents, sizes, [r])
    assert rel == [math.floor(k * 8 * 32768 * 1e6 / r) for k in range(len(ents))]
    # the implied rate of the last release is the request's rate (up to the 1 us floor)
    assert abs((len(ents) - 1) * 8 * 32768 / (rel[-1] * 1e-6) / r - 1) < 1.0 / rel[-1]


def test_release_times_monotone_max_rule():
    """Hand example: flow 0 at 1 byte/us, flow 1 at 4 bytes/us, entries (0,0,1) (1,0,2) (0,1,1)
    (1,2,1) with 4-byte packets: own times 0, 0, 4e6/1e6=4, 8/4=2 -> released 0, 0, 4, 4."""
    sizes = [[4, 4], [4, 4, 4]]
    ents = [(0, 0, 1), (1, 0, 2), (0, 1, 1), (1, 2, 1)]
    assert dp.release_us(ents, sizes, [1e6, 4e6]) == [0, 0, 4, 4]
    rng = random.Random(9)
    for _ in range(50):
        sizes, q, w = random_case(rng)
        ents = dp.entries(dp.runs(dp.drr_order(sizes, q)), 4)
        rel = dp.release_us(ents, sizes, [x * 1e6 for x in w])
        assert rel == sorted(rel)
        # no free packets is the plain rule; every packet free releases everything at t0
        assert dp.release_us(ents, sizes, [x * 1e6 for x in w], [0] * len(sizes)) == rel
        assert dp.release_us(ents, sizes, [x * 1e6 for x in w], [len(s) for s in sizes]) == [0] * len(ents)


def test_plan_free_packets_first():
    """c25 by hand: flows of 4 equal 4-byte packets, Q = 4, flow 0's first 2 packets free.
    Front: (0, 0, 2).  DRR over the rest -- round 1: flow 0 packet 2, flow 1 packet 0; round 2:
    flow 0 packet 3, flow 1 packet 1; rounds 3-4: flow 1 alone, packets 2 and 3 (one run with 1)."""
    ents, rel = dp.plan([2, 2], L=2, tiles=1, tile_bytes=[4], weights=[1.0, 1.0], Q=4, E=8,
                        rates=[1e6, 1e6], free=[2, 0])
    assert ents == [(0, 0, 2), (0, 2, 1), (1, 0, 1), (0, 3, 1), (1, 1, 3)]
    assert rel == [0, 0, 0, 4, 4]
    # no free packets: the plain DRR plan
    assert dp.plan([2, 2], 2, 1, [4], [1.0, 1.0], Q=4, free=[0, 0])[0] == dp.plan([2, 2], 2, 1, [4], [1.0, 1.0], Q=4)[0]


def test_release_times_free_packets():
    """Reading c24 applied to c22: flow 0's first packet is mirrored (free), so its second entry
    has 0 paced bytes before it -> released 0 instead of 4; flow 1 unchanged (8 bytes at 4/us = 2).
    A free prefix that ends inside an entry counts only the paced bytes before that entry."""
    sizes = [[4, 4], [4, 4, 4]]
    ents = [(0, 0, 1), (1, 0, 2), (0, 1, 1), (1, 2, 1)]
    assert dp.release_us(ents, sizes, [1e6, 4e6], [1, 0]) == [0, 0, 0, 2]
    assert dp.release_us(ents, sizes, [1e6, 4e6], [0, 1]) == [0, 0, 4, 4]      # (1,2,1): 4 B / 4 = 1 -> max 4
    assert dp.release_us([(0, 0, 3), (0, 3, 3)], [[2] * 6], [1e6], [2]) == [0, 2]


def test_plan_layer_major_units():
    """plan(): unit u of a request is tile u % tiles; every request's units appear once, in
    layer-major order, and the light request's share per round is Q."""
    ents, rel = dp.plan([3, 2], L=2, tiles=2, tile_bytes=[32768, 32768], weights=[1.0, 3.0],
                        rates=[1e9, 3e9])
    got = {0: [], 1: []}
    for f, first, c in ents:
        got[f] += list(range(first, first + c))
    assert got == {0: list(range(12)), 1: list(range(8))}
    assert ents[0] == (0, 0, 8)            # Q = 256 KiB = 8 units for the light request
    assert ents[1] == (1, 0, 8)            # the heavy request (q = 24 units) sends all 8 of its units
    assert ents[2] == (0, 8, 4)
    assert rel == sorted(rel)
    with pytest.raises(ValueError):
        dp.plan([1], L=1, tiles=1, tile_bytes=[1 << 20], weights=[1.0], Q=4096)


# ---- Alg. A2 line 7 literally: packets are whole layer payloads ----------------------------
def _ints(s, conv=int):
    return [conv(x) for x in s.split()] if s.strip() else []


@pytest.mark.parametrize("row", read_golden("wdrr_layer_examples.csv"), ids=lambda r: r["example"])
def test_layer_payload_plan_hand_worked(row):
    n_chunks, tile_bytes = _ints(row["n_chunks"]), _ints(row["tile_bytes"])
    rates = _ints(row["rates"], float) or None
    free = _ints(row["free_layers"]) or None
    ents, rel = dp.layer_payload_plan(n_chunks, int(row["L"]), len(tile_bytes), tile_bytes,
                                      _ints(row["weights"], float), Q=int(row["Q"]), E=int(row["E"]),
                                      rates=rates, free_layers=free)
    want = [tuple(int(v) for v in e.split(":")) for e in row["entries"].split()]
    assert ents == want
    if rates:
        assert rel == _ints(row["release_us"])


def _random_batch(rng):
    n = rng.randint(1, 5)
    L = rng.randint(1, 6)
    tiles = rng.randint(1, 3)
    tile_bytes = [rng.choice([8, 12, 16, 32]) for _ in range(tiles)]
    n_chunks = [rng.randint(0, 7) for _ in range(n)]
    w = [rng.choice([1.0, 1.5, 2.0, 3.0, 7.25]) for _ in range(n)]
    return n_chunks, L, tiles, tile_bytes, w


def test_layer_payload_plan_covers_each_request_in_layer_order():
    """Conservation and order: every unit of every request exactly once, each request's units in
    layer-major order, and every dispatched layer whole (no entry run splits a layer between two
    visits) -- what makes the packet a 'layer payload'."""
    rng = random.Random(21)
    for _ in range(300):
        n_chunks, L, tiles, tile_bytes, w = _random_batch(rng)
        ents, _ = dp.layer_payload_plan(n_chunks, L, tiles, tile_bytes, w, E=rng.randint(1, 9))
        got = [[] for _ in n_chunks]
        for f, first, cnt in ents:
            got[f].extend(range(first, first + cnt))
        for f, n in enumerate(n_chunks):
            assert got[f] == list(range(n * tiles * L))
        # runs (before the cut into entries) start and end on layer boundaries
        upl = [n * tiles for n in n_chunks]
        for f, first, cnt in dp.runs([(f, u) for f, a, c in ents for u in range(a, a + c)]):
            assert first % upl[f] == 0 and cnt % upl[f] == 0


def test_unit_plan_tracks_layer_payload_plan():
    """Pin of reading c21 (the library's unit-granular DRR stands for Alg. A2's layer-payload DRR).
    Both are DRR with quanta proportional to the same weights, so while every request is backlogged
    each keeps request i's bytes within 2*q_i + Max of the fluid share B*q_i/sum(q) after B bytes
    (Shreedhar-Varghese: k*q_i - Max < sent_i <= k*q_i after k rounds, and sum q >= n*Max).  Hence
    on every prefix of the unit plan, request i's cumulative bytes differ from the layer-payload
    plan's (at the same total, up to the entry in progress) by at most (2*q_i + Max) of one plan
    plus that of the other.  Checked on random batches of 64-layer requests (many rounds before
    anyone finishes); a unit plan that ignores or inverts the weights fails it."""
    rng = random.Random(5)
    for _ in range(60):
        n = rng.randint(2, 4)
        L, tiles = 64, rng.randint(1, 2)
        tile_bytes = [rng.choice([8, 16]) for _ in range(tiles)]
        n_chunks = [rng.randint(4, 8) for _ in range(n)]
        w = [float(rng.randint(1, 4)) for _ in range(n)]
        usz = [dp.unit_sizes(k, L, tiles, tile_bytes) for k in n_chunks]
        maxU, maxP = max(tile_bytes), max(k * sum(tile_bytes) for k in n_chunks)
        # small quanta make the rounds fine enough for the bound to bite (default Q = 256 KiB
        # exceeds these toy requests): Q = the largest packet of each plan
        eu, _ = dp.plan(n_chunks, L, tiles, tile_bytes, w, Q=maxU, E=1)
        ep, _ = dp.layer_payload_plan(n_chunks, L, tiles, tile_bytes, w, Q=maxP, E=1)
        qU, qP = dp.quanta(w, maxU), dp.quanta(w, maxP)
        pu, pp = dp.bytes_by_flow_prefix(eu, usz), dp.bytes_by_flow_prefix(ep, usz)
        total = [sum(x) for x in usz]
        assert pu[-1][1] == pp[-1][1] == tuple(total)
        k = 0
        for B, per_u in pu:
            while pp[k + 1][0] < B:
                k += 1
            lo, hi = pp[k][1], pp[k + 1][1] if pp[k][0] < B else pp[k][1]
            if any(per_u[i] >= total[i] or hi[i] >= total[i] for i in range(n)):
                break   # only while every request is backlogged in both plans
            for i in range(n):
                bound = (2 * qU[i] + maxU) + (2 * qP[i] + maxP)
                assert lo[i] - bound <= per_u[i] <= hi[i] + bound


def test_layer_payload_plan_fairness_bound():
    """The layer-payload plan is a DRR like any other: Shreedhar-Varghese's normalised fairness
    bound holds between backlogged requests on every prefix, with Max = the largest layer payload."""
    rng = random.Random(9)
    for _ in range(200):
        n_chunks, L, tiles, tile_bytes, w = _random_batch(rng)
        sizes = [dp.layer_payload_sizes(n, L, tile_bytes) for n in n_chunks]
        mx = max([s for f in sizes for s in f], default=1)
        q = dp.quanta(w, dp.default_quantum(mx))
        sent = [0] * len(sizes)
        left = [len(f) if f and f[0] > 0 else 0 for f in sizes]
        for f, p in dp.drr_order(sizes, q):
            sent[f] += sizes[f][p]
            left[f] -= 1
            live = [i for i in range(len(sizes)) if left[i] > 0]
            for a in live:
                for b in live:
                    assert abs(sent[a] / q[a] - sent[b] / q[b]) < 2 + mx / min(q[a], q[b])
