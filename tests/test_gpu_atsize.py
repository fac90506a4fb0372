"""At-size parity for BASELINE configs 3 and 4: every byte of the destination the bench fetches into,
against the oracle, layer by layer (VERDICT r1 "Next round" 1b/1c).

Config 3: Llama-3-8B layout, one 64K-token hit (N = 4096 chunks, 8 GiB), from an HBM store and from
a pinned-host store through both host-tier engines (copy engine + scatter, SM zero-copy), into a
fragmented paged NHD cache (Bs = 16, pool 1.25x): all 32 layers, every byte of each layer's K and V
caches (unused blocks keep their 0xA5 sentinels) and the buffer's pads.
Config 4: Llama-3-70B layout, one 32K request at 87.5% hit (N = 1792, 8.75 GiB), HBM store and
pinned-host store (copy engine): 17 layers in full, and the unused blocks of all 80 layers.

The expected bytes come from the oracle (Alg. A1 gather, oracle.assemble, then the paged scatter)
over a store that regenerates each chunk's layer slice from synth (RangeGet); the library side puts
the same synth payloads in batches.  Nothing is shared but the seeded inputs.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_2605_22850_b200 as oc  # noqa: E402
import synth  # noqa: E402
from oracle import keys as okeys  # noqa: E402
from oracle.geometry import Layout as OLayout  # noqa: E402
from scenario import (SynthStore, lib_target, make_dest, oracle_layer, requests_family,  # noqa: E402
                      sentinel_buffer)

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def _fetch(store, keys, lay, dest, engine):
    buf = sentinel_buffer(dest.size)
    d = oc.build_descriptor(store, keys, lay, lib_target(oc, dest, buf.data_ptr()))
    s, cons = torch.cuda.Stream(), torch.cuda.Stream()
    d.fetch_layerwise(s, engine=engine)
    for layer in range(lay.num_layers):          # the consumer's per-layer waits, in order
        d.wait_layer(layer, cons)
    cons.synchronize()
    s.synchronize()
    t = d.layer_times().astype(np.int64)
    assert np.all(np.diff(t) >= 0)               # announced in layer order
    d.close()
    return buf


def _check_layer(lay, ostore, okl, dest, bufs, layer):
    lo, want = oracle_layer(lay, ostore, okl, dest, layer)
    w = torch.from_numpy(want).cuda()
    for name, buf in bufs.items():
        got = buf[lo:lo + want.size]
        if not torch.equal(got, w):
            first = int((got != w).nonzero()[0].item())
            raise AssertionError(f"{name}: layer {layer} differs from the oracle at byte {first} of its region")


def _check_pads(dest, bufs):
    end = dest.v_off[-1] + (dest.v_off[-1] - dest.k_off[-1])
    for name, buf in bufs.items():
        assert bool((buf[:dest.k_off[0]] == 0xA5).all()) and bool((buf[end:] == 0xA5).all()), name


def _check_unused_blocks(lay, dest, bufs):
    """Every block the prefix does not use keeps its sentinel, in every layer's K and V cache."""
    L = lay.num_layers
    per_kv = dest.v_off[0] - dest.k_off[0]
    pool = per_kv // dest.block_stride
    unused = sorted(set(range(pool)) - set(dest.block_table))
    idx = torch.tensor(unused, dtype=torch.long, device="cuda")
    for name, buf in bufs.items():
        caches = buf[dest.k_off[0]:dest.k_off[0] + L * 2 * per_kv].view(L * 2, pool, dest.block_stride)
        for c in range(0, L * 2, 16):
            assert bool((caches[c:c + 16].index_select(1, idx) == 0xA5).all()), (name, c)


def _setup(lay, seed, n_chunks, tiers):
    req = requests_family(lay, seed, 0, [n_chunks])[0]
    keys = oc.chunk_keys(req.tokens, lay.chunk_tokens)
    okl = okeys.chunk_keys(req.tokens, lay.chunk_tokens)
    assert [bytes(k) for k in keys] == [bytes(k) for k in okl]
    stores = {t: oc.Store(lay, capacity=n_chunks, tier=t) for t in tiers}
    for i in range(0, n_chunks, 256):
        pl = synth.payloads(seed, req.payload_ids[i:i + 256], oc.geometry(lay)[2])
        for st in stores.values():
            assert st.put_chunks(keys[i:i + 256], pl) == min(256, n_chunks - i)
    for st in stores.values():
        assert st.match_prefix(req.tokens).shape[0] == n_chunks
    return req, keys, okl, stores, SynthStore(seed, okl, req.payload_ids)


def test_config3_64k_all_layers_every_byte():
    lay = OLayout(*synth.LLAMA3_8B.as_tuple())
    N = 65536 // lay.chunk_tokens
    req, keys, okl, stores, ostore = _setup(lay, 64, N, (oc.TIER_HBM, oc.TIER_PINNED_HOST))
    dest = make_dest(lay, N, "nhd", Bs=16, first_token=0, pool_factor=1.25, seed=65)
    bufs = {"hbm": _fetch(stores[oc.TIER_HBM], keys, lay, dest, oc.COPY_AUTO),
            "pinned_ce": _fetch(stores[oc.TIER_PINNED_HOST], keys, lay, dest, oc.COPY_CE),
            "pinned_sm": _fetch(stores[oc.TIER_PINNED_HOST], keys, lay, dest, oc.COPY_BULK)}
    for st in stores.values():
        st.close()
    for layer in range(lay.num_layers):
        _check_layer(lay, ostore, okl, dest, bufs, layer)
    _check_pads(dest, bufs)
    del bufs
    torch.cuda.empty_cache()


def test_config4_70b_32k_request():
    lay = OLayout(*synth.LLAMA3_70B.as_tuple())
    N = (32768 * 7 // 8) // lay.chunk_tokens          # 87.5% of a 32K request: 1792 chunks
    assert N == 1792
    req, keys, okl, stores, ostore = _setup(lay, 70, N, (oc.TIER_HBM, oc.TIER_PINNED_HOST))
    dest = make_dest(lay, N, "nhd", Bs=16, first_token=0, pool_factor=1.25, seed=71)
    bufs = {"hbm": _fetch(stores[oc.TIER_HBM], keys, lay, dest, oc.COPY_AUTO),
            "pinned_ce": _fetch(stores[oc.TIER_PINNED_HOST], keys, lay, dest, oc.COPY_CE)}
    for st in stores.values():
        st.close()
    for layer in list(range(0, lay.num_layers, 5)) + [lay.num_layers - 1]:
        _check_layer(lay, ostore, okl, dest, bufs, layer)
    _check_unused_blocks(lay, dest, bufs)
    _check_pads(dest, bufs)
    del bufs
    torch.cuda.empty_cache()


def test_bench_headline_launch_configuration():
    """The headline exactly as bench.py times it (benchlib.headline.build_sets: the rotating requests'
    chunks at random slab positions, fragmented paged caches; fetches back to back with
    OC_FETCH_OVERLAP on one copy stream, the consumer waiting on each request's last layer): every
    rotating request's 32 layers read back through its block table equal the oracle's Alg. A1
    payloads byte for byte, and the rest of each cache keeps its sentinel."""
    from benchlib import headline, verify
    from benchlib.common import ROTATE
    lay_t = synth.LLAMA3_8B.as_tuple()
    lay = OLayout(*lay_t)
    L, G = lay_t[0], lay_t[4]
    dev = torch.device("cuda", 0)
    store, sets = headline.build_sets(oc, torch, dev, lay_t, 256, rank=0)
    for st in sets:
        st["cache"].fill_(0xA5)
    descs = [oc.build_descriptor(store, st["keys"], lay_t, st["target"]) for st in sets]
    copy_s, cons_s = torch.cuda.Stream(), torch.cuda.Stream()
    copy_s.wait_stream(torch.cuda.current_stream())
    for i in range(3 * ROTATE):                     # back to back, overlapped, rotating
        descs[i % ROTATE].fetch_layerwise(copy_s, overlap=True)
        descs[i % ROTATE].wait_layer(L - 1, cons_s)
    torch.cuda.synchronize()
    for st in sets:
        idx = verify.slot_index(torch, dev, st["bt"], 256 * G, 16)
        ok, nbytes, _, _ = verify.full_check(torch, lay, st["seed"], st["keys"], st["ids"], st["cache"], idx,
                                             range(L))
        assert ok and nbytes == 256 * L * oc.geometry(lay_t)[1], st["seed"]
        rows = st["cache"].view(L, 2, -1, oc.geometry(lay_t)[0])
        mask = torch.ones(rows.shape[2], dtype=torch.bool, device=dev)
        mask[idx] = False
        assert bool((rows[:, :, mask] == 0xA5).all()), st["seed"]
    for d in descs:
        d.close()
    store.close()
    del sets
    torch.cuda.empty_cache()
