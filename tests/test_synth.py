"""The seeded input recipe (synth/): determinism and the structure DESIGN.md states for it."""
import collections

import numpy as np

import synth


def test_serving_requests_mix():
    a = synth.serving_requests(11, 4000, 32, 4)
    assert a == synth.serving_requests(11, 4000, 32, 4)            # seeded
    longs = sum(1 for lg, _, _ in a if lg)
    assert abs(longs / 4000 - 0.5) < 0.03                         # 4K/64K 50/50
    assert {h for _, _, h in a} == {0.5, 0.875}
    short = collections.Counter(f for lg, f, _ in a if not lg)
    # Zipf(1.1): family 0 is the most popular, frequencies fall with rank
    assert short[0] > short[1] > short[4] > short[16]
    assert all(0 <= f < (4 if lg else 32) for lg, f, _ in a)


def test_serving_requests_affinity():
    ws = 4
    home_of = lambda lg, f: (f + 32 * int(lg)) % ws
    for rank in range(ws):
        a = synth.serving_requests(11 + rank, 4000, 32, 4, home_of=home_of, rank=rank, p_aff=0.875)
        local = np.mean([home_of(lg, f) == rank for lg, f, _ in a])
        assert abs(local - 0.875) < 0.03


def test_block_table_distinct_and_seeded():
    bt = synth.block_table(3, 100, 150)
    assert len(set(bt.tolist())) == 100 and bt.min() >= 0 and bt.max() < 150
    assert np.array_equal(bt, synth.block_table(3, 100, 150))


def test_chunk_payload_range_is_a_slice_of_the_chunk():
    full = synth.chunk_payload(5, (1, 7), 4096)
    for off, n in ((0, 64), (8, 100), (2048, 2048), (4000, 96)):
        assert np.array_equal(synth.chunk_payload_range(5, (1, 7), off, n), full[off:off + n])


def test_config5_routing_strong_scaling():
    """Config 5's placement (benchlib/config5.py): the same 128 requests at every N; each served by its
    family's home rank with probability ~p_aff, otherwise by a seeded uniform draw; N = 1 all local."""
    from benchlib import config5
    reqs = synth.serving_requests(5, 2000, config5.N_SHORT, config5.N_LONG)
    assert reqs == synth.serving_requests(5, 2000, config5.N_SHORT, config5.N_LONG)
    for ws in (1, 2, 4, 8):
        home_of = lambda long, f: (f + config5.N_SHORT * int(long)) % ws
        served = config5.route(reqs, ws, home_of)
        assert served == config5.route(reqs, ws, home_of)
        local = np.mean([s == home_of(lg, f) for s, (lg, f, _) in zip(served, reqs)])
        if ws == 1:
            assert local == 1.0
        else:   # off-home draws land on the home rank 1/ws of the time
            want = config5.P_AFF + (1 - config5.P_AFF) / ws
            assert abs(local - want) < 0.03
        assert set(served) <= set(range(ws))
