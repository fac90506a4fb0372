"""The library's WDRR claim order (oc_wdrr_plan, host code; Alg. A2 lines 6-7) against the oracle:
identical entries and release times on random batches, ragged units included."""
import random
import time

import numpy as np
import pytest

import paper_2605_22850_b200 as oc
from oracle import dispatch as dp


def lib_plan(n_chunks, L, tiles, tile_bytes, weights, Q=0, E=0, hold=False, free=None):
    req, first, cnt, rel = oc.wdrr_plan([n * L * tiles for n in n_chunks], tile_bytes, weights,
                                        quantum_bytes=Q, entry_units=E, hold_rates=hold, free_units=free)
    return list(zip(req.tolist(), first.tolist(), cnt.tolist())), rel.tolist()


def test_random_batches_match_oracle():
    rng = random.Random(2605)
    for case in range(120):
        n = rng.randint(1, 6)
        L = rng.randint(1, 4)
        tiles = rng.randint(1, 3)
        tile_bytes = [rng.choice([2048, 16384, 32768]) for _ in range(tiles)]
        n_chunks = [rng.randint(0, 12) for _ in range(n)]
        if sum(n_chunks) == 0:
            n_chunks[0] = 1
        weights = [rng.choice([1.0, 2.0, 3.7, 0.5, 12.25]) * 1e9 for _ in range(n)]
        Q = rng.choice([0, max(tile_bytes), 3 * max(tile_bytes) + 5])
        E = rng.choice([0, 1, 3, 8])
        hold = rng.random() < 0.5
        # mirrored leading layers (reading c24): whole layers of units, sometimes none
        free = [rng.randint(0, L) * n * tiles for n in n_chunks] if rng.random() < 0.5 else None
        got, rel = lib_plan(n_chunks, L, tiles, tile_bytes, weights, Q, E, hold, free)
        want, wrel = dp.plan(n_chunks, L, tiles, tile_bytes, weights, Q=Q, E=E or 8,
                             rates=weights if hold else None, free=free)
        assert got == want, case
        assert rel == (wrel if hold else [0] * len(want)), case


def test_errors():
    with pytest.raises(oc.ObjcacheError) as e:
        oc.wdrr_plan([4, 4], [32768], [1.0, 0.0])
    assert e.value.code == oc.OC_EINVAL
    with pytest.raises(oc.ObjcacheError) as e:
        oc.wdrr_plan([4], [32768], [1.0], quantum_bytes=4096)       # Q below the largest unit
    assert e.value.code == oc.OC_EINVAL
    with pytest.raises(oc.ObjcacheError) as e:                     # 2^32 us of release time
        oc.wdrr_plan([1 << 20], [32768], [1.0], hold_rates=True)
    assert e.value.code == oc.OC_ERANGE
    with pytest.raises(ValueError):
        oc.wdrr_plan([4, 4], [32768], [1.0])


def test_config4_scale():
    """BASELINE config 4 (70B layout, 16 x 32K at 50% / 87.5% hit, 32 KiB units): the plan of the
    whole epoch is host work before layer 0, so it must be cheap; every unit appears once, in
    per-request order, and the first round gives each request its quantum."""
    n_chunks = [1024 if i % 2 == 0 else 1792 for i in range(16)]
    n_units = [n * 80 * 2 for n in n_chunks]
    rates = [(n * 65536) / 0.03 for n in n_chunks]
    t = time.perf_counter()
    req, first, cnt, rel = oc.wdrr_plan(n_units, [32768, 32768], rates, hold_rates=True)
    dt = time.perf_counter() - t
    assert dt < 0.5, dt
    for i in range(16):
        m = req == i
        f, c = first[m].astype(np.int64), cnt[m].astype(np.int64)
        assert f[0] == 0 and np.all(f[1:] == f[:-1] + c[:-1]) and f[-1] + c[-1] == n_units[i]
    assert np.all(np.diff(rel.astype(np.int64)) >= 0)
    # round 1: the light requests send Q = 256 KiB (8 units), the heavy ones 1792/1024 x that
    assert cnt[0] == 8 and req[0] == 0


def test_free_units_edge_cases():
    """free_units beyond a request's units (clamped: all of it is free), zero for some members, and
    for an empty member: planner = oracle (reading c25)."""
    n_chunks, L, tiles, tb = [3, 0, 2], 2, 2, [32768, 16384]
    w = [1e9, 2e9, 3e9]
    for free in ([100, 0, 1], [0, 5, 0], [12, 0, 8], [3, 0, 0]):
        got, rel = lib_plan(n_chunks, L, tiles, tb, w, E=3, hold=True, free=free)
        want, wrel = dp.plan(n_chunks, L, tiles, tb, w, E=3, rates=w, free=free)
        assert got == want and rel == wrel, free
    got, rel = lib_plan(n_chunks, L, tiles, tb, w, hold=True, free=[100, 0, 100])
    assert all(r == 0 for r in rel) and [e[0] for e in got] == [0] * 2 + [2] * 1   # every unit free


def test_layer_packet_batches_match_oracle():
    """layer_packets = L (Alg. A2 line 7 as written: a DRR packet is a request's whole layer payload):
    the library's planner equals oracle.dispatch.layer_payload_plan entry for entry and in release
    times, with and without mirrored leading layers."""
    rng = random.Random(2597)
    for case in range(120):
        n = rng.randint(1, 6)
        L = rng.randint(1, 5)
        tiles = rng.randint(1, 3)
        tile_bytes = [rng.choice([2048, 16384, 32768]) for _ in range(tiles)]
        n_chunks = [rng.randint(0, 12) for _ in range(n)]
        if sum(n_chunks) == 0:
            n_chunks[0] = 1
        weights = [rng.choice([1.0, 2.0, 3.7, 0.5, 12.25]) * 1e9 for _ in range(n)]
        maxp = max(k * sum(tile_bytes) for k in n_chunks)
        Q = rng.choice([0, maxp, 2 * maxp + 7])
        E = rng.choice([0, 1, 3, 8])
        hold = rng.random() < 0.5
        free_layers = [rng.randint(0, L) for _ in range(n)] if rng.random() < 0.5 else None
        free_units = [f * k * tiles for f, k in zip(free_layers, n_chunks)] if free_layers else None
        req, first, cnt, rel = oc.wdrr_plan([k * L * tiles for k in n_chunks], tile_bytes, weights,
                                            quantum_bytes=Q, entry_units=E, hold_rates=hold,
                                            free_units=free_units, layer_packets=L)
        got = list(zip(req.tolist(), first.tolist(), cnt.tolist()))
        want, wrel = dp.layer_payload_plan(n_chunks, L, tiles, tile_bytes, weights, Q=Q, E=E or 8,
                                           rates=weights if hold else None, free_layers=free_layers)
        assert got == want, case
        assert rel.tolist() == (wrel if hold else [0] * len(want)), case


def test_layer_packet_errors():
    with pytest.raises(oc.ObjcacheError) as e:     # 7 units are not 2 whole layers
        oc.wdrr_plan([7], [32768], [1.0], layer_packets=2)
    assert e.value.code == oc.OC_EINVAL
    with pytest.raises(oc.ObjcacheError) as e:     # Q below a 4-unit layer payload
        oc.wdrr_plan([8], [32768], [1.0], quantum_bytes=65536, layer_packets=2)
    assert e.value.code == oc.OC_EINVAL
    with pytest.raises(oc.ObjcacheError) as e:     # free units must be whole layers
        oc.wdrr_plan([8], [32768], [1.0], free_units=[3], layer_packets=2)
    assert e.value.code == oc.OC_EINVAL
