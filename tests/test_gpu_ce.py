"""CE engine (pinned-host chunks: strided copy-engine transfers into an HBM stage, then the bulk
scatter kernel) vs the oracle, byte for byte, including chains whose slots form several runs."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_2605_22850_b200 as oc  # noqa: E402
from oracle.geometry import Layout as OLayout  # noqa: E402
from scenario import (lib_target, make_dest, oracle_result, payload_stack,  # noqa: E402
                      requests_family, sentinel_buffer)

pytestmark = pytest.mark.gpu


def fetch_and_check(st, lay, seed, req, dest, keys=None, delivery=oc.DELIVER_LAYER_MAJOR, **opts):
    keys = st.match_prefix(req.tokens)[:req.n_chunks] if keys is None else keys
    buf = sentinel_buffer(dest.size)
    d = oc.build_descriptor(st, keys, lay, lib_target(oc, dest, buf.data_ptr()), delivery)
    s, cons = torch.cuda.Stream(), torch.cuda.Stream()
    d.fetch_layerwise(s, engine=oc.COPY_CE, **opts)
    d.wait_layer(lay.num_layers - 1, cons)
    cons.synchronize()
    assert np.array_equal(buf.cpu().numpy(), oracle_result(lay, seed, req, dest))
    t = d.layer_times().astype(np.int64)
    assert np.all(np.diff(t[1:]) >= 0)
    return d, buf


@pytest.mark.parametrize("lay", [OLayout(3, 2, 64, 2, 16), OLayout(2, 4, 32, 2, 20), OLayout(5, 1, 16, 2, 16)])
@pytest.mark.parametrize("kind,Bs,first", [("nhd", 16, 0), ("nhd", 8, 5), ("hnd", 16, 3), ("flat", 16, 0),
                                           ("nhd", 1, 2)])
@pytest.mark.parametrize("unit_bytes", [0, 1024])
def test_ce_parity_one_run(lay, kind, Bs, first, unit_bytes):
    req = requests_family(lay, 7, 0, [9])[0]
    with oc.Store(lay, capacity=16, tier=oc.TIER_PINNED_HOST) as st:
        st.put_chunks(oc.chunk_keys(req.tokens, lay.chunk_tokens), payload_stack(lay, 7, req.payload_ids))
        dest = make_dest(lay, req.n_chunks, kind, Bs=Bs, first_token=first, seed=3)
        d, _ = fetch_and_check(st, lay, 7, req, dest, unit_bytes=unit_bytes)
        d.close()


def test_ce_several_runs_and_refetch():
    """Request B's chain: the family's 8 shared chunks (put with A), then its own 3 chunks put after
    an unrelated request's -- three runs of slots; refetched with every engine in turn."""
    lay = OLayout(3, 2, 64, 2, 16)
    a, b = requests_family(lay, 11, 8, [2, 3])
    other = requests_family(lay, 12, 0, [4])[0]
    with oc.Store(lay, capacity=32, tier=oc.TIER_PINNED_HOST) as st:
        ka, kb, ko = (oc.chunk_keys(r.tokens, 16) for r in (a, b, other))
        st.put_chunks(ka, payload_stack(lay, 11, a.payload_ids))
        st.put_chunks(ko, payload_stack(lay, 12, other.payload_ids))
        st.put_chunks(kb[8:10], payload_stack(lay, 11, b.payload_ids[8:10]))
        st.put_chunks(ko[:1], payload_stack(lay, 12, other.payload_ids[:1]))      # dedup, no slot
        st.put_chunks(kb[10:], payload_stack(lay, 11, b.payload_ids[10:]))
        slots = st.lookup(kb)
        runs = 1 + int(np.count_nonzero(np.diff(slots.astype(np.int64)) != 2 * 16 * 256 * 3))
        assert runs == 2
        dest = make_dest(lay, b.n_chunks, "nhd", Bs=8, first_token=1, seed=5)
        d, buf = fetch_and_check(st, lay, 11, b, dest)
        s = torch.cuda.Stream()
        for engine in (oc.COPY_BULK, oc.COPY_CE, oc.COPY_LDST, oc.COPY_CE, oc.COPY_CE):
            with torch.cuda.stream(s):
                buf.fill_(0xA5)
            d.fetch_layerwise(s, engine=engine, max_ctas=3 if engine == oc.COPY_CE else 0)
            d.sync_layer(lay.num_layers - 1)
            s.synchronize()
            assert np.array_equal(buf.cpu().numpy(), oracle_result(lay, 11, b, dest)), engine
        d.close()


def test_ce_chunk_major_delivery():
    lay = OLayout(4, 2, 64, 2, 16)
    req = requests_family(lay, 21, 0, [6])[0]
    with oc.Store(lay, capacity=8, tier=oc.TIER_PINNED_HOST) as st:
        st.put_chunks(oc.chunk_keys(req.tokens, 16), payload_stack(lay, 21, req.payload_ids))
        dest = make_dest(lay, req.n_chunks, "hnd", Bs=16, seed=2)
        d, _ = fetch_and_check(st, lay, 21, req, dest, delivery=oc.DELIVER_CHUNK_MAJOR)
        d.close()


def test_ce_errors():
    lay = OLayout(2, 2, 64, 2, 16)
    req = requests_family(lay, 31, 0, [3])[0]
    keys = oc.chunk_keys(req.tokens, 16)
    dest = make_dest(lay, 3, "nhd", Bs=16)
    buf = sentinel_buffer(dest.size)
    with oc.Store(lay, capacity=4) as hbm:                       # HBM store: no CE path
        hbm.put_chunks(keys, payload_stack(lay, 31, req.payload_ids))
        d = oc.build_descriptor(hbm, keys, lay, lib_target(oc, dest, buf.data_ptr()))
        with pytest.raises(oc.ObjcacheError) as e:
            d.fetch_layerwise(None, engine=oc.COPY_CE)
        assert e.value.code == oc.OC_ENOTSUP
        d.close()
    with oc.Store(lay, capacity=4, tier=oc.TIER_PINNED_HOST) as st:
        st.put_chunks(keys, payload_stack(lay, 31, req.payload_ids))
        d = oc.build_descriptor(st, keys, lay, lib_target(oc, dest, buf.data_ptr()))
        for kw in ({"pace_Bps": 1e9}, {"mode": oc.FETCH_PER_LAYER}):
            with pytest.raises(oc.ObjcacheError) as e:
                d.fetch_layerwise(None, engine=oc.COPY_CE, **kw)
            assert e.value.code == oc.OC_ENOTSUP
        d.fetch_layerwise(None, engine=oc.COPY_CE)               # still usable after the refusals
        d.sync_layer(1)
        torch.cuda.synchronize()
        assert np.array_equal(buf.cpu().numpy(), oracle_result(lay, 31, req, dest))
        d.close()


def test_ce_flat_target_direct_and_refetch():
    """FLAT target: the copy engine writes the client buffer B_l directly (no stage); refetches
    alternate with the kernel engines on the same descriptor (epochs stay consistent)."""
    lay = OLayout(3, 2, 64, 2, 16)
    a, b = requests_family(lay, 31, 5, [3, 2])
    with oc.Store(lay, capacity=16, tier=oc.TIER_PINNED_HOST) as st:
        st.put_chunks(oc.chunk_keys(a.tokens, 16), payload_stack(lay, 31, a.payload_ids))
        st.put_chunks(oc.chunk_keys(b.tokens, 16), payload_stack(lay, 31, b.payload_ids))   # 2 runs for b
        dest = make_dest(lay, b.n_chunks, "flat")
        buf = sentinel_buffer(dest.size)
        d = oc.build_descriptor(st, st.match_prefix(b.tokens), lay, lib_target(oc, dest, buf.data_ptr()))
        s, cons = torch.cuda.Stream(), torch.cuda.Stream()
        want = oracle_result(lay, 31, b, dest)
        for engine in (oc.COPY_CE, oc.COPY_BULK, oc.COPY_CE, oc.COPY_LDST, oc.COPY_CE):
            with torch.cuda.stream(s):
                buf.fill_(0xA5)
            d.fetch_layerwise(s, engine=engine)
            for l in range(lay.num_layers):
                d.wait_layer(l, cons)
            cons.synchronize()
            s.synchronize()
            assert np.array_equal(buf.cpu().numpy(), want), engine
            t = d.layer_times().astype(np.int64)
            assert np.all(np.diff(t) >= 0)
        d.close()


@pytest.mark.parametrize("hot", [1, 2, 3])
def test_hot_layer_mirror(hot):
    """A pinned-host store mirroring its chunks' first `hot` layers in HBM: every engine (split
    launches for the kernel engines; mirror copies for the CE engine) delivers the oracle's bytes,
    for a chain of two slot runs, into paged and flat targets."""
    lay = OLayout(3, 2, 64, 2, 16)
    a, b = requests_family(lay, 41, 4, [2, 3])
    with oc.Store(lay, capacity=16, tier=oc.TIER_PINNED_HOST) as st:
        st.set_hot_layers(hot)
        st.put_chunks(oc.chunk_keys(a.tokens, 16), payload_stack(lay, 41, a.payload_ids))
        st.put_chunks(oc.chunk_keys(b.tokens, 16), payload_stack(lay, 41, b.payload_ids))
        for kind in ("nhd", "hnd", "flat"):
            dest = make_dest(lay, b.n_chunks, kind, Bs=8, first_token=2 if kind != "flat" else 0, seed=9)
            buf = sentinel_buffer(dest.size)
            d = oc.build_descriptor(st, st.match_prefix(b.tokens), lay, lib_target(oc, dest, buf.data_ptr()))
            s, cons = torch.cuda.Stream(), torch.cuda.Stream()
            want = oracle_result(lay, 41, b, dest)
            for engine in (oc.COPY_AUTO, oc.COPY_BULK, oc.COPY_LDST, oc.COPY_CE):
                with torch.cuda.stream(s):
                    buf.fill_(0xA5)
                d.fetch_layerwise(s, engine=engine)
                for l in range(lay.num_layers):
                    d.wait_layer(l, cons)
                cons.synchronize()
                s.synchronize()
                assert np.array_equal(buf.cpu().numpy(), want), (kind, engine)
                t = d.layer_times().astype(np.int64)
                assert np.all(np.diff(t) >= 0)
            d.close()


def test_hot_layer_errors():
    lay = OLayout(2, 2, 64, 2, 16)
    req = requests_family(lay, 42, 0, [2])[0]
    keys = oc.chunk_keys(req.tokens, 16)
    with oc.Store(lay, capacity=4) as hbm:
        with pytest.raises(oc.ObjcacheError) as e:
            hbm.set_hot_layers(1)
        assert e.value.code == oc.OC_EINVAL
    with oc.Store(lay, capacity=4, tier=oc.TIER_PINNED_HOST) as st:
        with pytest.raises(oc.ObjcacheError) as e:
            st.set_hot_layers(3)
        assert e.value.code == oc.OC_ERANGE
        st.set_hot_layers(1)
        st.put_chunks(keys, payload_stack(lay, 42, req.payload_ids))
        with pytest.raises(oc.ObjcacheError) as e:
            st.set_hot_layers(2)
        assert e.value.code == oc.OC_EINVAL
        src = make_dest(lay, 2, "nhd")
        cache = sentinel_buffer(src.size)
        with pytest.raises(oc.ObjcacheError) as e:
            oc.put_from_paged(st, keys, lay, lib_target(oc, src, cache.data_ptr()))
        assert e.value.code == oc.OC_ENOTSUP


def test_hot_layer_mirror_pitch_per_store():
    """Stores with different mirror depths in one chain (own store: 2 mirrored layers, attached
    pinned-host peer: 1).  The descriptor mirrors min = 1 layer, but each slot run must read its
    own store's mirror with that store's pitch (hot_layers * S) -- every engine, byte for byte."""
    lay = OLayout(3, 2, 64, 2, 16)
    req = requests_family(lay, 43, 0, [9])[0]
    keys = oc.chunk_keys(req.tokens, 16)
    pl = payload_stack(lay, 43, req.payload_ids)
    with oc.Store(lay, capacity=16, tier=oc.TIER_PINNED_HOST) as own, \
            oc.Store(lay, capacity=16, tier=oc.TIER_PINNED_HOST) as peer:
        own.set_hot_layers(2)
        peer.set_hot_layers(1)
        own.put_chunks(keys[:6], pl[:6])
        peer.put_chunks(keys[6:], pl[6:])
        own.attach_peer(peer)
        for kind in ("nhd", "flat"):
            dest = make_dest(lay, req.n_chunks, kind, Bs=8, first_token=0, seed=13)
            buf = sentinel_buffer(dest.size)
            d = oc.build_descriptor(own, own.match_prefix(req.tokens), lay, lib_target(oc, dest, buf.data_ptr()))
            want = oracle_result(lay, 43, req, dest)
            s, cons = torch.cuda.Stream(), torch.cuda.Stream()
            for engine in (oc.COPY_CE, oc.COPY_BULK, oc.COPY_LDST):
                with torch.cuda.stream(s):
                    buf.fill_(0xA5)
                d.fetch_layerwise(s, engine=engine)
                d.wait_layer(lay.num_layers - 1, cons)
                cons.synchronize()
                s.synchronize()
                assert np.array_equal(buf.cpu().numpy(), want), (kind, engine)
            d.close()


def test_attach_peer_rejects_cycles():
    lay = OLayout(2, 2, 64, 2, 16)
    with oc.Store(lay, capacity=4) as a, oc.Store(lay, capacity=4) as b, oc.Store(lay, capacity=4) as c:
        a.attach_peer(b)
        b.attach_peer(c)
        for x, y in ((b, a), (c, a), (c, b)):
            with pytest.raises(oc.ObjcacheError) as e:
                x.attach_peer(y)
            assert e.value.code == oc.OC_EINVAL
        req = requests_family(lay, 44, 0, [2])[0]
        assert a.match_prefix(req.tokens).shape[0] == 0   # a miss walks a -> b -> c and stops


@pytest.mark.parametrize("kind", ["nhd", "hnd"])
def test_auto_engine_large_layers_from_pinned_host(kind):
    """AUTO with a pinned-host store and >= 32 MiB layers (here 64 chunks x 512 KiB) into a paged
    target takes the copy engine + scatter path; with smaller layers zero-copy -- both byte-exact."""
    lay = OLayout(2, 64, 128, 2, 16)                  # row 16 KiB, S = 512 KiB
    for n in (64, 8):                                  # 32 MiB layers (CE) and 4 MiB layers (zero-copy)
        req = requests_family(lay, 13, 0, [n])[0]
        with oc.Store(lay, capacity=n, tier=oc.TIER_PINNED_HOST) as st:
            keys = oc.chunk_keys(req.tokens, 16)
            st.put_chunks(keys, payload_stack(lay, 13, req.payload_ids))
            dest = make_dest(lay, n, kind, Bs=16, first_token=0, seed=4)
            buf = sentinel_buffer(dest.size)
            d = oc.build_descriptor(st, keys, lay, lib_target(oc, dest, buf.data_ptr()))
            s, cons = torch.cuda.Stream(), torch.cuda.Stream()
            d.fetch_layerwise(s)                       # engine = COPY_AUTO
            d.wait_layer(lay.num_layers - 1, cons)
            cons.synchronize()
            assert np.array_equal(buf.cpu().numpy(), oracle_result(lay, 13, req, dest)), n
            d.close()
