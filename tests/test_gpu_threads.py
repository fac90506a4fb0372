"""Host threads against one store (SURVEY 8(b) ownership: puts of distinct keys and racing
identical puts are safe; the index is single-writer / multi-reader).

Python threads call the library through ctypes, which drops the GIL for the call, so the C code
really runs concurrently.  Checked: racing identical puts store one copy and count it once,
conflicting puts of one key leave exactly one winner (the rest get EIMMUTABLE), readers
see only valid prefixes while writers run, and descriptors built and fetched from several threads
on their own streams all deliver the oracle's bytes."""
import threading

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_2605_22850_b200 as oc  # noqa: E402
from oracle.geometry import Layout as OLayout  # noqa: E402
from scenario import (lib_target, make_dest, oracle_result, payload_stack,  # noqa: E402
                      requests_family, sentinel_buffer)

pytestmark = pytest.mark.gpu

T = 8  # threads


def run_threads(fn):
    errs = []

    def wrap(i):
        try:
            fn(i)
        except BaseException as e:  # noqa: BLE001 -- re-raised in the main thread
            errs.append(e)

    th = [threading.Thread(target=wrap, args=(i,)) for i in range(T)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if errs:
        raise errs[0]


@pytest.mark.parametrize("tier", [oc.TIER_HBM, oc.TIER_PINNED_HOST])
def test_racing_puts_readers_and_fetches(tier):
    lay = OLayout(3, 2, 64, 2, 16)
    n_shared, seed = 24, 91
    reqs = requests_family(lay, seed, n_shared, [3 + i for i in range(T)])
    fam_keys = [oc.chunk_keys(r.tokens, 16) for r in reqs]
    shared_keys = fam_keys[0][:n_shared]
    shared_payload = payload_stack(lay, seed, reqs[0].payload_ids[:n_shared])
    total = n_shared + sum(3 + i for i in range(T))
    st = oc.Store(lay, capacity=total, tier=tier)
    n_new = [0] * T
    seen = [[] for _ in range(T)]

    def writer(i):
        r = reqs[i]
        for rnd in range(4):                    # the shared prefix, raced by every thread, twice
            if rnd % 2 == 0:
                n_new[i] += st.put_chunks(shared_keys, shared_payload)
            else:
                own = slice(n_shared, r.n_chunks)
                n_new[i] += st.put_chunks(fam_keys[i][own], payload_stack(lay, seed, r.payload_ids[own]))
            m = st.match_prefix(r.tokens)       # a reader between writes: a valid prefix of the chain
            assert np.array_equal(m, fam_keys[i][:len(m)])
            seen[i].append(len(m))

    run_threads(writer)
    assert st.count == total
    assert sum(n_new) == total                   # every chunk counted once, by one of the racers
    for i, r in enumerate(reqs):
        assert seen[i] == sorted(seen[i])        # the store is append-only: matches only grow
        assert seen[i][-1] == r.n_chunks
        assert len(set(st.lookup(fam_keys[i]).tolist())) == r.n_chunks

    # descriptors built and fetched concurrently, one stream per thread
    dests = [make_dest(lay, r.n_chunks, "nhd" if i % 2 else "hnd", Bs=8, first_token=i, seed=i)
             for i, r in enumerate(reqs)]
    bufs = [sentinel_buffer(d.size) for d in dests]

    def fetcher(i):
        s = torch.cuda.Stream()
        for rnd in range(3):
            d = oc.build_descriptor(st, st.match_prefix(reqs[i].tokens), lay, lib_target(oc, dests[i], bufs[i].data_ptr()))
            d.fetch_layerwise(s, engine=(oc.COPY_AUTO, oc.COPY_BULK, oc.COPY_LDST)[rnd])
            d.sync_layer(lay.num_layers - 1)
            s.synchronize()
            d.close()

    run_threads(fetcher)
    torch.cuda.synchronize()
    for i, r in enumerate(reqs):
        assert np.array_equal(bufs[i].cpu().numpy(), oracle_result(lay, seed, r, dests[i])), i
    st.close()


def test_conflicting_puts_one_winner():
    """Every thread puts the same key with its own bytes: one put stores it, the others are
    refused with EIMMUTABLE, and the stored object is the winner's bytes."""
    lay = OLayout(2, 2, 64, 2, 16)
    req = requests_family(lay, 5, 0, [1])[0]
    key = oc.chunk_keys(req.tokens, 16)[:1]
    payloads = [payload_stack(lay, 100 + i, req.payload_ids[:1]) for i in range(T)]
    outcome = [None] * T
    st = oc.Store(lay, capacity=4)

    def put(i):
        try:
            outcome[i] = st.put_chunks(key, payloads[i])
        except oc.ObjcacheError as e:
            outcome[i] = e.code

    run_threads(put)
    assert sorted(outcome) == sorted([oc.OC_EIMMUTABLE] * (T - 1) + [1])
    winner = outcome.index(1)
    dest = make_dest(lay, 1, "flat")
    buf = sentinel_buffer(dest.size)
    d = oc.build_descriptor(st, key, lay, lib_target(oc, dest, buf.data_ptr()))
    d.fetch_layerwise(None)
    d.sync_layer(lay.num_layers - 1)
    torch.cuda.synchronize()
    got = buf.cpu().numpy()
    want = oracle_result(lay, 100 + winner, req, dest)
    assert np.array_equal(got, want)
    d.close()
    st.close()
