"""Offload path: paged KV cache -> new chunk slots (oc_put_from_paged) vs the oracle."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_2605_22850_b200 as oc  # noqa: E402
from oracle import keys as okeys  # noqa: E402
from oracle.assemble import fetch_layerwise, offload_paged  # noqa: E402
from oracle.descriptor import FlatTarget as OFlat, build_descriptor as obuild  # noqa: E402
from oracle.geometry import Layout as OLayout, chunk_layer_bytes  # noqa: E402
from oracle.store import ChunkStore  # noqa: E402
from scenario import lib_target, make_dest, oracle_target, requests_family, sentinel_buffer  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("engine", ["bulk", "ldst"])
@pytest.mark.parametrize("kind,Bs,first", [("nhd", 16, 0), ("nhd", 8, 5), ("hnd", 8, 3), ("nhd", 32, 17)])
def test_offload_then_fetch_flat_matches_oracle(monkeypatch, engine, kind, Bs, first):
    monkeypatch.setenv("OC_OFFLOAD_ENGINE", engine)
    lay = OLayout(3, 2, 64, 2, 16)
    N = 7
    req = requests_family(lay, 40, 0, [N])[0]
    src = make_dest(lay, N, kind, Bs=Bs, first_token=first, seed=40)
    gen = torch.Generator(device="cuda").manual_seed(7)
    cache = torch.randint(0, 256, (src.size,), dtype=torch.uint8, device="cuda", generator=gen)
    keys = oc.chunk_keys(req.tokens, 16)
    with oc.Store(lay, capacity=N + 1) as st:
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())  # the cache bytes were written on the current stream
        assert oc.put_from_paged(st, keys, lay, lib_target(oc, src, cache.data_ptr()), s) == N
        s.synchronize()
        assert st.count == N
        assert oc.put_from_paged(st, keys, lay, lib_target(oc, src, cache.data_ptr()), s) == 0   # dedup
        # read the new chunks back through a flat (Alg. A1 client buffer) fetch
        W = N * lay.num_layers * chunk_layer_bytes(lay)
        flat = sentinel_buffer(W)
        d = oc.build_descriptor(st, keys, lay, oc.FlatTarget(flat.data_ptr(), W))
        d.fetch_layerwise(s)
        d.sync_layer(lay.num_layers - 1)
        got = flat.cpu().numpy()
        d.close()
    # oracle: offload from the same cache bytes, then the flat fetch
    mem = cache.cpu().numpy()
    ost = ChunkStore(lay)
    okeys_ = okeys.chunk_keys(req.tokens, 16)
    assert offload_paged(ost, okeys_, lay, oracle_target(src), mem) == N
    want = np.full(W, 0xA5, np.uint8)
    fetch_layerwise(ost, obuild(ost, okeys_, lay, OFlat(0, W)), want)
    assert np.array_equal(got, want)


@pytest.mark.parametrize("engine", ["bulk", "ldst"])
def test_offload_round_trip_into_another_cache(monkeypatch, engine):
    monkeypatch.setenv("OC_OFFLOAD_ENGINE", engine)
    lay = OLayout(2, 4, 32, 2, 16)
    N = 9
    req = requests_family(lay, 41, 0, [N])[0]
    a = make_dest(lay, N, "nhd", Bs=16, first_token=0, seed=1)
    b = make_dest(lay, N, "hnd", Bs=8, first_token=3, seed=2)
    gen = torch.Generator(device="cuda").manual_seed(9)
    cache_a = torch.randint(0, 256, (a.size,), dtype=torch.uint8, device="cuda", generator=gen)
    cache_b = sentinel_buffer(b.size)
    keys = oc.chunk_keys(req.tokens, 16)
    with oc.Store(lay, capacity=N) as st:
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        oc.put_from_paged(st, keys, lay, lib_target(oc, a, cache_a.data_ptr()), s)
        d = oc.build_descriptor(st, keys, lay, lib_target(oc, b, cache_b.data_ptr()))
        d.fetch_layerwise(s)                         # ordered after the offload on the same stream
        d.sync_layer(1)
        got = cache_b.cpu().numpy()
        d.close()
    ost = ChunkStore(lay)
    ok = okeys.chunk_keys(req.tokens, 16)
    offload_paged(ost, ok, lay, oracle_target(a), cache_a.cpu().numpy())
    want = np.full(b.size, 0xA5, np.uint8)
    fetch_layerwise(ost, obuild(ost, ok, lay, oracle_target(b)), want)
    assert np.array_equal(got, want)


def test_offload_errors():
    lay = OLayout(2, 2, 32, 2, 16)
    req = requests_family(lay, 42, 0, [4])[0]
    src = make_dest(lay, 4, "nhd", Bs=16)
    cache = torch.zeros(src.size, dtype=torch.uint8, device="cuda")
    keys = oc.chunk_keys(req.tokens, 16)
    with oc.Store(lay, capacity=2) as st:
        with pytest.raises(oc.ObjcacheError) as e:
            oc.put_from_paged(st, keys, lay, lib_target(oc, src, cache.data_ptr()))
        assert e.value.code == oc.OC_EFULL and e.value.bad_index == 2
        torch.cuda.synchronize()
        assert st.count == 2
        with pytest.raises(oc.ObjcacheError) as e:
            oc.put_from_paged(st, keys, lay, oc.FlatTarget(cache.data_ptr(), src.size))
        assert e.value.code == oc.OC_EINVAL


@pytest.mark.parametrize("engine", ["bulk", "ldst"])
def test_offload_into_pinned_host_store(monkeypatch, engine):
    """Offload whose slots live in the pinned host tier (writes cross PCIe), read back through a
    fetch from that tier, against the oracle."""
    monkeypatch.setenv("OC_OFFLOAD_ENGINE", engine)
    lay = OLayout(3, 2, 64, 2, 16)
    N = 10
    req = requests_family(lay, 42, 0, [N])[0]
    src = make_dest(lay, N, "nhd", Bs=16, first_token=4, seed=42)
    gen = torch.Generator(device="cuda").manual_seed(42)
    cache = torch.randint(0, 256, (src.size,), dtype=torch.uint8, device="cuda", generator=gen)
    keys = oc.chunk_keys(req.tokens, 16)
    W = N * lay.num_layers * chunk_layer_bytes(lay)
    with oc.Store(lay, capacity=N, tier=oc.TIER_PINNED_HOST) as st:
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        assert oc.put_from_paged(st, keys, lay, lib_target(oc, src, cache.data_ptr()), s) == N
        flat = sentinel_buffer(W)
        d = oc.build_descriptor(st, keys, lay, oc.FlatTarget(flat.data_ptr(), W))
        d.fetch_layerwise(s)
        d.sync_layer(lay.num_layers - 1)
        got = flat.cpu().numpy()
        d.close()
    ost = ChunkStore(lay)
    ok = okeys.chunk_keys(req.tokens, 16)
    assert offload_paged(ost, ok, lay, oracle_target(src), cache.cpu().numpy()) == N
    want = np.full(W, 0xA5, np.uint8)
    fetch_layerwise(ost, obuild(ost, ok, lay, OFlat(0, W)), want)
    assert np.array_equal(got, want)


def test_offload_into_padded_slots_then_fetch():
    """A layout whose HBM slots are padded (oc_slot_pitch: 1.25 MiB chunks -> 41 granules of 32 KiB):
    offload (put_from_paged) and put_chunks write at slot * pitch, lookups return those addresses,
    and fetches of both read them back -- byte-exact against the oracle's offload + Alg. A1."""
    from scenario import payload_stack
    lay = OLayout(20, 8, 128, 2, 16)
    lay_t = (20, 8, 128, 2, 16)
    chunk = oc.geometry(lay_t)[2]
    pitch = oc.slot_pitch(lay_t, oc.TIER_HBM)
    assert pitch == 41 * 32768 and chunk == 40 * 32768
    N = 5
    r1, r2 = requests_family(lay, 42, 0, [N, N])
    src = make_dest(lay, N, "nhd", Bs=16, first_token=0, seed=42)
    gen = torch.Generator(device="cuda").manual_seed(11)
    cache = torch.randint(0, 256, (src.size,), dtype=torch.uint8, device="cuda", generator=gen)
    k1, k2 = oc.chunk_keys(r1.tokens, 16), oc.chunk_keys(r2.tokens, 16)
    W = N * lay.num_layers * chunk_layer_bytes(lay)
    with oc.Store(lay, capacity=2 * N) as st:
        assert st.slot_pitch == pitch and st.slab[1] == 2 * N * pitch
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        assert oc.put_from_paged(st, k1, lay, lib_target(oc, src, cache.data_ptr()), s) == N
        s.synchronize()
        assert st.put_chunks(k2, payload_stack(lay, 42, r2.payload_ids)) == N
        base = st.slab[0]
        addrs = sorted(int(a) - base for a in st.lookup(list(k1) + list(k2)))
        assert addrs == [i * pitch for i in range(2 * N)]
        got = []
        for keys in (k1, k2):
            flat = sentinel_buffer(W)
            d = oc.build_descriptor(st, keys, lay, oc.FlatTarget(flat.data_ptr(), W))
            d.fetch_layerwise(s)
            d.sync_layer(lay.num_layers - 1)
            got.append(flat.cpu().numpy())
            d.close()
    ost = ChunkStore(lay)
    ok1, ok2 = okeys.chunk_keys(r1.tokens, 16), okeys.chunk_keys(r2.tokens, 16)
    assert offload_paged(ost, ok1, lay, oracle_target(src), cache.cpu().numpy()) == N
    want1 = np.full(W, 0xA5, np.uint8)
    fetch_layerwise(ost, obuild(ost, ok1, lay, OFlat(0, W)), want1)
    assert np.array_equal(got[0], want1)
    from scenario import Dest, oracle_result
    assert np.array_equal(got[1], oracle_result(lay, 42, r2, Dest(kind="flat", size=W, flat_off=0, flat_cap=W)))
