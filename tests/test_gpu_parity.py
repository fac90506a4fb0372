"""GPU parity: libobjcache's fetch (C ABI -> sm_100a kernels) against the oracle, byte for byte.

Every comparison covers the whole destination buffer, including the 0xA5 sentinel bytes the
fetch must not touch (reading c5).  Sizes span several work units with ragged tails; the
Llama-3-8B 4K case is the bench configuration; 64K is checked on sampled layers.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_2605_22850_b200 as oc  # noqa: E402
import synth  # noqa: E402
from oracle.geometry import Layout as OLayout, chunk_layer_bytes, row_bytes  # noqa: E402
from scenario import (lib_target, make_dest, oracle_result, payload_stack,  # noqa: E402
                      requests_family, sentinel_buffer)

pytestmark = pytest.mark.gpu

MODES = [oc.FETCH_PERSISTENT, oc.FETCH_PER_LAYER]
ENGINES = [oc.COPY_LDST, oc.COPY_BULK]


def lay_of(named):
    return OLayout(*named.as_tuple())


def run_lib(lay, seed, req, dest, tier=oc.TIER_HBM, mode=oc.FETCH_PERSISTENT, unit_bytes=0, max_ctas=0,
            delivery=oc.DELIVER_LAYER_MAJOR, store=None, engine=oc.COPY_BULK):
    own = store is None
    if own:
        store = oc.Store(lay, capacity=req.n_chunks + 2, tier=tier)
        keys = oc.chunk_keys(req.tokens, lay.chunk_tokens)[:req.n_chunks]
        store.put_chunks(keys, payload_stack(lay, seed, req.payload_ids[:req.n_chunks]))
    keys = store.match_prefix(req.tokens)[:req.n_chunks]
    assert keys.shape[0] == req.n_chunks
    buf = sentinel_buffer(dest.size)
    desc = oc.build_descriptor(store, keys, lay, lib_target(oc, dest, buf.data_ptr()), delivery)
    s = torch.cuda.Stream()
    desc.fetch_layerwise(s, mode=mode, unit_bytes=unit_bytes, max_ctas=max_ctas, engine=engine)
    desc.sync_layer(lay.num_layers - 1)
    torch.cuda.synchronize()
    out = buf.cpu().numpy()
    desc.close()
    if own:
        store.close()
    return out


def assert_same(got, want):
    if not np.array_equal(got, want):
        bad = np.flatnonzero(got != want)
        raise AssertionError(f"{bad.size} bytes differ; first at {bad[:8].tolist()}: "
                             f"got {got[bad[:8]].tolist()} want {want[bad[:8]].tolist()}")


# ---- tiny config (BASELINE.json configs[0]) -------------------------------------------------------
def test_tiny_store_match_and_dedup():
    lay = lay_of(synth.TINY)
    a, b = requests_family(lay, 0, 8, [2, 3], [5, 0])
    with oc.Store(lay, capacity=16) as st:
        pa = payload_stack(lay, 0, a.payload_ids)
        pb = payload_stack(lay, 0, b.payload_ids)
        assert st.put_chunks(oc.chunk_keys(a.tokens, 16), pa) == 10
        assert st.put_chunks(oc.chunk_keys(b.tokens, 16), pb) == 3         # 8 shared chunks deduplicated
        assert st.count == 13
        assert st.match_prefix(a.tokens).shape[0] == 10
        assert st.match_prefix(b.tokens).shape[0] == 11
        q = a.tokens.copy()
        q[8 * 16 + 3] ^= 1
        assert st.match_prefix(q).shape[0] == 8
        assert st.match_prefix(q[:7]).shape[0] == 0
        # lookup returns slot addresses inside the slab, and the slots hold the put bytes
        addrs = st.lookup(oc.chunk_keys(b.tokens, 16))
        base, nbytes = st.slab
        n, pitch = pb.shape[1], st.slot_pitch
        assert pitch >= n and nbytes == 16 * pitch
        assert len(set(addrs.tolist())) == 11
        for ad in addrs:
            assert (int(ad) - base) % pitch == 0 and int(ad) - base + n <= nbytes


@pytest.mark.parametrize("kind", ["nhd", "hnd", "flat"])
@pytest.mark.parametrize("Bs,first", [(8, 0), (16, 5), (32, 16), (1, 3)])
@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("engine", ENGINES)
def test_tiny_parity(kind, Bs, first, mode, engine):
    lay = lay_of(synth.TINY)
    for req in requests_family(lay, 0, 8, [2, 3], [5, 0]):
        dest = make_dest(lay, req.n_chunks, kind, Bs=Bs, first_token=first, seed=Bs + first)
        assert_same(run_lib(lay, 0, req, dest, mode=mode, engine=engine), oracle_result(lay, 0, req, dest))


# ---- several units per chunk, ragged tiles, odd sizes -----------------------------------------------
@pytest.mark.parametrize("kind", ["nhd", "hnd"])
@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("unit_bytes", [4096, 0, 1000])
@pytest.mark.parametrize("engine", ENGINES)
def test_ragged_units(kind, mode, unit_bytes, engine):
    lay = OLayout(3, 4, 64, 2, 20)             # row = 512 B; unit 4096 B -> tiles of 8, 8, 4 rows
    req = requests_family(lay, 3, 0, [7])[0]
    dest = make_dest(lay, req.n_chunks, kind, Bs=16, first_token=3, seed=5)
    assert_same(run_lib(lay, 3, req, dest, mode=mode, unit_bytes=unit_bytes, engine=engine),
                oracle_result(lay, 3, req, dest))


@pytest.mark.parametrize("max_ctas", [1, 3, 37])
@pytest.mark.parametrize("engine", ENGINES)
def test_grid_caps(max_ctas, engine):
    lay = OLayout(4, 2, 128, 2, 16)
    req = requests_family(lay, 4, 0, [9])[0]
    dest = make_dest(lay, req.n_chunks, "nhd", Bs=8, first_token=1, seed=6)
    for mode in MODES:
        assert_same(run_lib(lay, 4, req, dest, mode=mode, max_ctas=max_ctas, engine=engine),
                    oracle_result(lay, 4, req, dest))


@pytest.mark.parametrize("engine", ENGINES)
def test_single_chunk_single_layer(engine):
    lay = OLayout(1, 1, 8, 2, 1)               # row = 16 B: the smallest legal row
    req = requests_family(lay, 8, 0, [1])[0]
    for kind in ("nhd", "hnd", "flat"):
        dest = make_dest(lay, 1, kind, Bs=1, seed=1)
        assert_same(run_lib(lay, 8, req, dest, engine=engine), oracle_result(lay, 8, req, dest))


@pytest.mark.parametrize("engine", ENGINES)
def test_pinned_host_tier(engine):
    lay = OLayout(3, 4, 64, 2, 20)
    req = requests_family(lay, 9, 0, [6])[0]
    for kind in ("nhd", "hnd", "flat"):
        dest = make_dest(lay, req.n_chunks, kind, Bs=16, first_token=2, seed=2)
        assert_same(run_lib(lay, 9, req, dest, tier=oc.TIER_PINNED_HOST, engine=engine),
                    oracle_result(lay, 9, req, dest))


def test_chunk_major_delivery():
    lay = lay_of(synth.TINY)
    req = requests_family(lay, 1, 0, [5])[0]
    dest = make_dest(lay, req.n_chunks, "nhd", Bs=16, seed=3)
    assert_same(run_lib(lay, 1, req, dest, delivery=oc.DELIVER_CHUNK_MAJOR), oracle_result(lay, 1, req, dest))


def test_peer_store_resolution():
    # "fake remote": half the chain lives in a second store, attached as a peer (same GPU).
    lay = OLayout(2, 2, 64, 2, 16)
    req = requests_family(lay, 11, 0, [10])[0]
    keys = oc.chunk_keys(req.tokens, 16)
    pl = payload_stack(lay, 11, req.payload_ids)
    local, remote = oc.Store(lay, capacity=16), oc.Store(lay, capacity=16)
    local.put_chunks(keys[:4], pl[:4])
    remote.put_chunks(keys[4:], pl[4:])
    assert local.match_prefix(req.tokens).shape[0] == 4
    local.attach_peer(remote)
    assert local.match_prefix(req.tokens).shape[0] == 10
    dest = make_dest(lay, 10, "nhd", Bs=16, first_token=7, seed=4)
    assert_same(run_lib(lay, 11, req, dest, store=local), oracle_result(lay, 11, req, dest))


@pytest.mark.parametrize("engine", [oc.COPY_BULK, oc.COPY_LDST, oc.COPY_AUTO])
@pytest.mark.parametrize("host_first", [False, True])
def test_mixed_tier_chain(engine, host_first):
    """One request whose chain is split between an HBM store and a pinned-host store attached as
    its peer: one launch reads HBM and host memory (PCIe) and delivers every byte."""
    lay = OLayout(3, 2, 64, 2, 16)
    req = requests_family(lay, 12, 0, [11])[0]
    keys = oc.chunk_keys(req.tokens, 16)
    pl = payload_stack(lay, 12, req.payload_ids)
    first_tier, second_tier = (oc.TIER_PINNED_HOST, oc.TIER_HBM) if host_first else (oc.TIER_HBM, oc.TIER_PINNED_HOST)
    local, peer = oc.Store(lay, capacity=16, tier=first_tier), oc.Store(lay, capacity=16, tier=second_tier)
    local.put_chunks(keys[:6], pl[:6])
    peer.put_chunks(keys[6:], pl[6:])
    local.attach_peer(peer)
    for kind in ("nhd", "hnd"):
        dest = make_dest(lay, 11, kind, Bs=8, first_token=3, seed=6)
        assert_same(run_lib(lay, 12, req, dest, store=local, engine=engine), oracle_result(lay, 12, req, dest))
    local.close()
    peer.close()


# ---- the bench configuration: Llama-3-8B, 4K-token prefix hit -----------------------------------
@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("engine", ENGINES)
def test_llama8b_4k_full(mode, engine):
    lay = lay_of(synth.LLAMA3_8B)
    req = requests_family(lay, 2024, 0, [256])[0]
    dest = make_dest(lay, 256, "nhd", Bs=16, seed=7)
    got = run_lib(lay, 2024, req, dest, mode=mode, engine=engine)
    assert_same(got, oracle_result(lay, 2024, req, dest, layers=range(lay.num_layers)))


@pytest.mark.parametrize("G", [64, 256])
@pytest.mark.parametrize("engine", ENGINES)
def test_llama8b_4k_other_granularities(G, engine):
    lay = lay_of(synth.with_chunk_tokens(synth.LLAMA3_8B, G))
    req = requests_family(lay, 77, 0, [4096 // G])[0]
    dest = make_dest(lay, req.n_chunks, "nhd", Bs=16, first_token=16, seed=8)
    assert_same(run_lib(lay, 77, req, dest, engine=engine),
                oracle_result(lay, 77, req, dest, layers=range(lay.num_layers)))


@pytest.mark.slow
def test_llama8b_64k_sampled_layers():
    lay = lay_of(synth.LLAMA3_8B)
    N = 4096
    req = requests_family(lay, 64, 0, [N])[0]
    row, S, G = row_bytes(lay), chunk_layer_bytes(lay), 16
    pl = payload_stack(lay, 64, req.payload_ids)                      # 8 GiB, host
    dest = make_dest(lay, N, "nhd", Bs=16, pool_factor=1.0, seed=9)
    with oc.Store(lay, capacity=N) as st:
        keys = oc.chunk_keys(req.tokens, 16)
        assert st.put_chunks(keys, pl) == N
        buf = sentinel_buffer(dest.size)
        desc = oc.build_descriptor(st, keys, lay, lib_target(oc, dest, buf.data_ptr()))
        desc.fetch_layerwise(torch.cuda.current_stream())
        desc.sync_layer(31)
        torch.cuda.synchronize()
        bt = np.asarray(dest.block_table, np.int64)
        u = np.arange(N * G)
        slots = bt[u // 16] * 16 + u % 16
        pool_rows = len(bt) * 16
        for l in (0, 1, 17, 31):
            want = pl[:, l * S:(l + 1) * S].reshape(N, 2, G, row)        # Alg. A1 slice of every chunk
            for kv, off in ((0, dest.k_off[l]), (1, dest.v_off[l])):
                cache = buf[off:off + pool_rows * row].view(pool_rows, row).cpu().numpy()
                assert np.array_equal(cache[slots], want[:, kv].reshape(N * G, row)), (l, kv)
        desc.close()
        del buf


def test_llama70b_layout_sampled_layers():
    """BASELINE config 4's layout (L = 80): a 2K-token prefix (N = 128) into a fragmented paged
    cache, first_token offset 8, checked against the oracle on sampled layers."""
    lay = lay_of(synth.LLAMA3_70B)
    N = 128
    req = requests_family(lay, 70, 0, [N])[0]
    dest = make_dest(lay, N, "nhd", Bs=16, first_token=8, seed=70)
    layers = (0, 1, 39, 78, 79)
    want = oracle_result(lay, 70, req, dest, layers=layers)
    with oc.Store(lay, capacity=N) as st:
        keys = oc.chunk_keys(req.tokens, 16)
        assert st.put_chunks(keys, payload_stack(lay, 70, req.payload_ids)) == N
        buf = sentinel_buffer(dest.size)
        desc = oc.build_descriptor(st, keys, lay, lib_target(oc, dest, buf.data_ptr()))
        desc.fetch_layerwise(torch.cuda.current_stream())
        desc.sync_layer(79)
        got = buf.cpu().numpy()
        per_kv = dest.v_off[0] - dest.k_off[0]                 # one layer's K (or V) cache
        for l in layers:
            for off in (dest.k_off[l], dest.v_off[l]):
                assert np.array_equal(got[off:off + per_kv], want[off:off + per_kv]), l
        desc.close()


# ---- layer-ready semantics ----------------------------------------------------------------------------
@pytest.mark.parametrize("wait_kind", ["value", "kernel", "relay"])
@pytest.mark.parametrize("engine", ENGINES)
def test_wait_layer_orders_consumer(monkeypatch, wait_kind, engine):
    """A consumer stream that waits on layer l and then snapshots layer l must see final bytes even
    though the (paced) fetch is still running -- for each way a wait is enqueued (the default spin
    kernel, the opt-in stream value wait on the consumer stream, the opt-in relay stream + event)."""
    if wait_kind == "value":
        monkeypatch.setenv("OC_WAIT_VALUE", "1")
    if wait_kind == "relay":
        monkeypatch.setenv("OC_WAIT_RELAY", "1")
    lay = OLayout(6, 2, 64, 2, 16)
    req = requests_family(lay, 21, 0, [8])[0]
    dest = make_dest(lay, 8, "flat")
    want = oracle_result(lay, 21, req, dest)
    with oc.Store(lay, capacity=8) as st:
        keys = oc.chunk_keys(req.tokens, 16)
        st.put_chunks(keys, payload_stack(lay, 21, req.payload_ids))
        buf = sentinel_buffer(dest.size)
        desc = oc.build_descriptor(st, keys, lay, lib_target(oc, dest, buf.data_ptr()))
        copy_s, cons = torch.cuda.Stream(), torch.cuda.Stream()
        layer_bytes = 8 * chunk_layer_bytes(lay)
        pace = layer_bytes / 3e-3                                            # one layer every 3 ms
        snaps = []
        desc.fetch_layerwise(copy_s, pace_Bps=pace, engine=engine)
        for l in range(lay.num_layers):
            desc.wait_layer(l, cons)
            with torch.cuda.stream(cons):
                o = dest.flat_off + l * layer_bytes
                snaps.append(buf[o:o + layer_bytes].clone())
        torch.cuda.synchronize()
        for l, sn in enumerate(snaps):
            o = dest.flat_off + l * layer_bytes
            assert np.array_equal(sn.cpu().numpy(), want[o:o + layer_bytes]), l
        t = desc.layer_times().astype(np.int64)
        assert np.all(np.diff(t[1:]) > 0)                                   # announced in increasing l
        # layer l cannot be ready before its release time t0 + l * 3 ms
        assert np.all(t[1:] - t[0] >= np.arange(lay.num_layers) * 3_000_000 - 50_000)
        desc.close()


@pytest.mark.parametrize("engine", ENGINES)
def test_refetch_epochs_and_sync(engine):
    lay = OLayout(4, 2, 64, 2, 16)
    req = requests_family(lay, 5, 0, [6])[0]
    dest = make_dest(lay, 6, "nhd", Bs=8, seed=2)
    want = oracle_result(lay, 5, req, dest)
    with oc.Store(lay, capacity=8) as st:
        keys = oc.chunk_keys(req.tokens, 16)
        st.put_chunks(keys, payload_stack(lay, 5, req.payload_ids))
        buf = sentinel_buffer(dest.size)
        desc = oc.build_descriptor(st, keys, lay, lib_target(oc, dest, buf.data_ptr()))
        s = torch.cuda.Stream()
        for it in range(5):
            with torch.cuda.stream(s):
                buf.fill_(0xA5)
            desc.fetch_layerwise(s, mode=MODES[it % 2], engine=engine)
            for l in range(lay.num_layers):
                desc.sync_layer(l)
            torch.cuda.synchronize()
            assert_same(buf.cpu().numpy(), want)
        desc.close()


# ---- error conventions -----------------------------------------------------------------------------
def test_errors():
    lay = lay_of(synth.TINY)
    req = requests_family(lay, 0, 0, [4])[0]
    keys = oc.chunk_keys(req.tokens, 16)
    pl = payload_stack(lay, 0, req.payload_ids)
    dest = make_dest(lay, 4, "nhd", Bs=16)
    with oc.Store(lay, capacity=5) as st:
        assert st.put_chunks(keys, pl) == 4
        bad = pl.copy()
        bad[2, 0] ^= 1
        with pytest.raises(oc.ObjcacheError) as e:
            st.put_chunks(keys, bad)
        assert e.value.code == oc.OC_EIMMUTABLE and e.value.bad_index == 2
        other = oc.chunk_keys(synth.tokens(99, 32), 16)
        with pytest.raises(oc.ObjcacheError) as e:
            st.put_chunks(other, payload_stack(lay, 99, [(9, 0), (9, 1)]))
        assert e.value.code == oc.OC_EFULL and e.value.bad_index == 1
        buf = sentinel_buffer(dest.size)
        tgt = lib_target(oc, dest, buf.data_ptr())
        missing = np.concatenate([keys[:2], oc.chunk_keys(synth.tokens(7, 16), 16), keys[2:]])
        with pytest.raises(oc.ObjcacheError) as e:
            oc.build_descriptor(st, missing, lay, tgt)
        assert e.value.code == oc.OC_ENOTFOUND and e.value.bad_index == 2
        with pytest.raises(oc.ObjcacheError) as e:
            oc.build_descriptor(st, keys[:0], lay, tgt)
        assert e.value.code == oc.OC_EINVAL
        short = lib_target(oc, dest, buf.data_ptr())
        short.block_table = short.block_table[:3]
        with pytest.raises(oc.ObjcacheError) as e:
            oc.build_descriptor(st, keys, lay, short)
        assert e.value.code == oc.OC_ERANGE
        dup = lib_target(oc, dest, buf.data_ptr())
        dup.block_table = list(dup.block_table)
        dup.block_table[1] = dup.block_table[0]
        with pytest.raises(oc.ObjcacheError) as e:
            oc.build_descriptor(st, keys, lay, dup)
        assert e.value.code == oc.OC_EINVAL
        mis = lib_target(oc, dest, buf.data_ptr() + 8)
        with pytest.raises(oc.ObjcacheError) as e:
            oc.build_descriptor(st, keys, lay, mis)
        assert e.value.code == oc.OC_EALIGN
        with pytest.raises(oc.ObjcacheError) as e:
            oc.build_descriptor(st, keys, (2, 2, 16, 2, 32), tgt)              # layout != store's
        assert e.value.code == oc.OC_EINVAL
        flat_small = oc.FlatTarget(buf.data_ptr(), 4 * 2 * chunk_layer_bytes(lay) - 16)
        with pytest.raises(oc.ObjcacheError) as e:
            oc.build_descriptor(st, keys, lay, flat_small)
        assert e.value.code == oc.OC_ERANGE
        desc = oc.build_descriptor(st, keys, lay, tgt)
        with pytest.raises(oc.ObjcacheError) as e:
            desc.wait_layer(0)
        assert e.value.code == oc.OC_EINVAL                                  # nothing fetched yet
        desc.fetch_layerwise()
        with pytest.raises(oc.ObjcacheError) as e:
            desc.wait_layer(2)
        assert e.value.code == oc.OC_ERANGE
        with pytest.raises(oc.ObjcacheError) as e:
            desc.fetch_layerwise(mode=oc.FETCH_PER_LAYER, pace_Bps=1e9)
        assert e.value.code == oc.OC_ENOTSUP
        desc.sync_layer(1)
        torch.cuda.synchronize()
        desc.close()


def test_alternating_engines_and_unit_sizes_on_one_descriptor():
    """The per-layer unit counters are monotone across fetches while the unit size (and so the
    units per layer) may change from one fetch to the next."""
    lay = OLayout(3, 2, 64, 2, 16)
    req = requests_family(lay, 12, 0, [9])[0]
    dest = make_dest(lay, 9, "nhd", Bs=16, first_token=5, seed=12)
    want = oracle_result(lay, 12, req, dest)
    with oc.Store(lay, capacity=9) as st:
        keys = oc.chunk_keys(req.tokens, 16)
        st.put_chunks(keys, payload_stack(lay, 12, req.payload_ids))
        buf = sentinel_buffer(dest.size)
        desc = oc.build_descriptor(st, keys, lay, lib_target(oc, dest, buf.data_ptr()))
        s, cons = torch.cuda.Stream(), torch.cuda.Stream()
        plan = [(oc.COPY_BULK, 0, oc.FETCH_PERSISTENT), (oc.COPY_LDST, 1024, oc.FETCH_PERSISTENT),
                (oc.COPY_BULK, 512, oc.FETCH_PER_LAYER), (oc.COPY_LDST, 0, oc.FETCH_PER_LAYER),
                (oc.COPY_BULK, 2048, oc.FETCH_PERSISTENT), (oc.COPY_LDST, 4096, oc.FETCH_PERSISTENT)]
        for engine, ub, mode in plan:
            with torch.cuda.stream(s):
                buf.fill_(0xA5)
            desc.fetch_layerwise(s, mode=mode, engine=engine, unit_bytes=ub)
            desc.wait_layer(lay.num_layers - 1, cons)
            cons.synchronize()
            assert_same(buf.cpu().numpy(), want)
            torch.cuda.synchronize()
        desc.close()


# ---- the paper's unfused flow: gather into the flat client buffer, then scatter it ---------------
@pytest.mark.parametrize("kind,Bs,first", [("nhd", 16, 0), ("hnd", 8, 3), ("nhd", 32, 17)])
@pytest.mark.parametrize("unit_bytes", [0, 1024])
def test_gather_to_flat_then_scatter_flat(kind, Bs, first, unit_bytes):
    """Alg. A1 into the flat client buffer B_0..B_{L-1}, then oc_scatter_flat into a paged cache:
    both the flat payload and the paged result equal the oracle's."""
    lay = OLayout(3, 2, 64, 2, 16)
    req = requests_family(lay, 77, 0, [9])[0]
    with oc.Store(lay, capacity=12) as st:
        keys = oc.chunk_keys(req.tokens, 16)
        st.put_chunks(keys, payload_stack(lay, 77, req.payload_ids))
        fdest = make_dest(lay, 9, "flat")
        fbuf = sentinel_buffer(fdest.size)
        df = oc.build_descriptor(st, keys, lay, lib_target(oc, fdest, fbuf.data_ptr()))
        pdest = make_dest(lay, 9, kind, Bs=Bs, first_token=first, seed=5)
        pbuf = sentinel_buffer(pdest.size)
        dp = oc.build_descriptor(st, keys, lay, lib_target(oc, pdest, pbuf.data_ptr()))
        s = torch.cuda.Stream()
        df.fetch_layerwise(s, unit_bytes=unit_bytes)
        dp.scatter_flat(fbuf.data_ptr() + fdest.flat_off, fdest.flat_cap, s, unit_bytes=unit_bytes)
        dp.sync_layer(lay.num_layers - 1)
        s.synchronize()
        assert_same(fbuf.cpu().numpy(), oracle_result(lay, 77, req, fdest))
        assert_same(pbuf.cpu().numpy(), oracle_result(lay, 77, req, pdest))
        t = dp.layer_times().astype(np.int64)
        assert t[0] > 0 and np.all(np.diff(t[1:]) >= 0)
        dp.fetch_layerwise(s)                                    # a normal fetch afterwards still works
        dp.sync_layer(lay.num_layers - 1)
        s.synchronize()
        assert_same(pbuf.cpu().numpy(), oracle_result(lay, 77, req, pdest))
        with pytest.raises(oc.ObjcacheError) as e:
            dp.scatter_flat(fbuf.data_ptr() + fdest.flat_off, fdest.flat_cap - 16, s)
        assert e.value.code == oc.OC_ERANGE
        with pytest.raises(oc.ObjcacheError) as e:
            dp.scatter_flat(fbuf.data_ptr() + fdest.flat_off + 8, fdest.flat_cap, s)
        assert e.value.code == oc.OC_EALIGN
        df.close()
        dp.close()


# ---- OC_FETCH_OVERLAP: back-to-back launches overlapping each other's tails ----------------------
@pytest.mark.parametrize("kind,engine", [("nhd", "bulk"), ("nhd", "ldst"), ("hnd", "ldst")])
@pytest.mark.parametrize("lay,n_chunks", [(OLayout(2, 2, 16, 2, 16), 10), (OLayout(3, 2, 64, 2, 16), 40),
                                          (OLayout(32, 8, 128, 2, 16), 64)])
def test_overlap_back_to_back(lay, n_chunks, kind, engine):
    """Several requests fetched back to back with OC_FETCH_OVERLAP (each launch may start during the
    previous one's tail), the same descriptor twice in a row included, with the TMA engine and the
    LD/ST engine (NHD and head-split HND targets): every destination equals the oracle, consumer
    waits on each request's last layer complete, layer times are monotone."""
    eng = oc.COPY_BULK if engine == "bulk" else oc.COPY_LDST
    reqs = [requests_family(lay, 60 + i, 0, [n_chunks])[0] for i in range(3)]
    store = oc.Store(lay, capacity=3 * n_chunks)
    for i, r in enumerate(reqs):
        store.put_chunks(oc.chunk_keys(r.tokens, lay.chunk_tokens), payload_stack(lay, 60 + i, r.payload_ids))
    dests = [make_dest(lay, n_chunks, kind, Bs=16, first_token=3 * i, seed=70 + i) for i in range(3)]
    bufs = [sentinel_buffer(d.size) for d in dests]
    descs = [oc.build_descriptor(store, store.match_prefix(r.tokens), lay, lib_target(oc, d, b.data_ptr()))
             for r, d, b in zip(reqs, dests, bufs)]
    s, cons = torch.cuda.Stream(), torch.cuda.Stream()
    order = [0, 1, 2, 2, 0, 1, 1, 2, 0] * 3
    for i in order:
        descs[i].fetch_layerwise(s, overlap=True, engine=eng)
        descs[i].wait_layer(lay.num_layers - 1, cons)
    cons.synchronize()
    s.synchronize()
    for r, d, b, desc, seed in zip(reqs, dests, bufs, descs, (60, 61, 62)):
        assert_same(b.cpu().numpy(), oracle_result(lay, seed, r, d))
        t = desc.layer_times().astype(np.int64)
        assert np.all(np.diff(t[1:]) >= 0)
    # a plain fetch after overlapped ones still sees consistent counters
    for desc in descs:
        desc.fetch_layerwise(s)
        desc.sync_layer(lay.num_layers - 1)
    for desc in descs:
        desc.close()
    store.close()


@pytest.mark.parametrize("lay,n_chunks", [(OLayout(3, 2, 64, 2, 16), 40), (OLayout(32, 8, 128, 2, 16), 64)])
def test_first_layer_full_and_yield(lay, n_chunks):
    """The co-running launch shapes: OC_FETCH_FIRST_LAYER_FULL (layer 0 with the whole GPU, the rest
    under a copy-CTA budget, both engines) and OC_FETCH_YIELD (layer 0 persistent, the rest one unit
    per CTA on a low-priority stream): same bytes as the oracle, layers announced in order."""
    req = requests_family(lay, 81, 0, [n_chunks])[0]
    dest = make_dest(lay, n_chunks, "nhd", Bs=16, first_token=5, seed=82)
    want = oracle_result(lay, 81, req, dest)
    store = oc.Store(lay, capacity=n_chunks)
    store.put_chunks(oc.chunk_keys(req.tokens, lay.chunk_tokens), payload_stack(lay, 81, req.payload_ids))
    buf = sentinel_buffer(dest.size)
    d = oc.build_descriptor(store, store.match_prefix(req.tokens), lay, lib_target(oc, dest, buf.data_ptr()))
    s, cons = torch.cuda.Stream(priority=0), torch.cuda.Stream(priority=-1)
    for opts in (dict(engine=oc.COPY_BULK, max_ctas=4, first_layer_full=True),
                 dict(engine=oc.COPY_LDST, max_ctas=7, first_layer_full=True),
                 dict(engine=oc.COPY_BULK, yield_sms=True), dict(engine=oc.COPY_BULK)):
        with torch.cuda.stream(s):
            buf.fill_(0xA5)
        d.fetch_layerwise(s, **opts)
        for l in range(lay.num_layers):
            d.wait_layer(l, cons)
        cons.synchronize()
        s.synchronize()
        assert_same(buf.cpu().numpy(), want)
        t = d.layer_times().astype(np.int64)
        assert np.all(np.diff(t) >= 0), opts
    d.close()
    store.close()
