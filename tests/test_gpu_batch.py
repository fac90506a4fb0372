"""Batched fetch (several requests, one launch, layer-major across the batch) vs the oracle."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_2605_22850_b200 as oc  # noqa: E402
from oracle.geometry import Layout as OLayout  # noqa: E402
from scenario import lib_target, make_dest, oracle_result, payload_stack, requests_family, sentinel_buffer  # noqa: E402

pytestmark = pytest.mark.gpu


def setup_batch(lay, specs, tier=oc.TIER_HBM):
    """specs: list of (seed, n_chunks, kind, Bs, first_token).  Each request has its own chain."""
    cap = sum(n for _, n, *_ in specs) + 2
    st = oc.Store(lay, capacity=cap, tier=tier)
    items = []
    for seed, n, kind, Bs, first in specs:
        req = requests_family(lay, seed, 0, [n])[0]
        keys = oc.chunk_keys(req.tokens, lay.chunk_tokens)
        st.put_chunks(keys, payload_stack(lay, seed, req.payload_ids))
        dest = make_dest(lay, n, kind, Bs=Bs, first_token=first, seed=seed)
        buf = sentinel_buffer(dest.size)
        desc = oc.build_descriptor(st, st.match_prefix(req.tokens), lay, lib_target(oc, dest, buf.data_ptr()))
        items.append({"seed": seed, "req": req, "dest": dest, "buf": buf, "desc": desc})
    torch.cuda.synchronize()  # the sentinel fills (current stream) land before fetches on other streams
    return st, items


def check(lay, items):
    for it in items:
        want = oracle_result(lay, it["seed"], it["req"], it["dest"])
        got = it["buf"].cpu().numpy()
        assert np.array_equal(got, want), f"request seed {it['seed']} differs"


SPECS = [(1, 3, "nhd", 16, 0), (2, 7, "hnd", 8, 5), (3, 1, "flat", 16, 0), (4, 12, "nhd", 32, 17),
         (5, 5, "nhd", 1, 2)]


@pytest.mark.parametrize("lay", [OLayout(3, 2, 64, 2, 16), OLayout(2, 4, 32, 2, 20)])
@pytest.mark.parametrize("unit_bytes", [0, 1024, 3072])
@pytest.mark.parametrize("order,blk_kib,claim", [(oc.BATCH_BY_REQUEST, 0, 0), (oc.BATCH_BY_POSITION, 16, 3),
                                                 (oc.BATCH_BY_POSITION, 4096, 8), (oc.BATCH_BY_POSITION, 16, 1)])
@pytest.mark.parametrize("engine", [oc.COPY_BULK, oc.COPY_LDST])
def test_batch_parity(lay, unit_bytes, order, blk_kib, claim, engine, monkeypatch):
    if blk_kib:   # 16 KiB: blocks of 1-2 positions, partial last blocks in every run
        monkeypatch.setenv("OC_BYPOS_BLOCK_KIB", str(blk_kib))
    if claim:     # units per claim; 3 leaves a ragged last claim
        monkeypatch.setenv("OC_BYPOS_CLAIM", str(claim))
    st, items = setup_batch(lay, SPECS)
    b = oc.Batch([it["desc"] for it in items], order=order)
    s = torch.cuda.Stream()
    b.fetch(s, unit_bytes=unit_bytes, engine=engine)
    for it in items:
        it["desc"].sync_layer(lay.num_layers - 1)
    torch.cuda.synchronize()
    check(lay, items)
    for it in items:                                     # each request announced its layers in order
        t = it["desc"].layer_times().astype(np.int64)
        assert np.all(np.diff(t[1:]) >= 0) and t[1] >= t[0]
    b.close()
    st.close()


def test_batch_refetch_and_mix_with_single_fetches():
    lay = OLayout(3, 2, 64, 2, 16)
    st, items = setup_batch(lay, SPECS[:3])
    b = oc.Batch([it["desc"] for it in items])
    s, cons = torch.cuda.Stream(), torch.cuda.Stream()
    for rnd in range(4):
        with torch.cuda.stream(s):
            for it in items:
                it["buf"].fill_(0xA5)
        if rnd % 2 == 0:
            b.fetch(s, max_ctas=3 if rnd == 2 else 0)
        else:
            for it in items:
                it["desc"].fetch_layerwise(s, engine=oc.COPY_LDST if rnd == 3 else oc.COPY_BULK)
        for it in items:
            it["desc"].wait_layer(lay.num_layers - 1, cons)
        cons.synchronize()
        torch.cuda.synchronize()
        check(lay, items)
    b.close()
    st.close()


@pytest.mark.parametrize("order", [oc.BATCH_BY_REQUEST, oc.BATCH_BY_POSITION])
@pytest.mark.parametrize("engine", [oc.COPY_BULK, oc.COPY_LDST, oc.COPY_AUTO])
def test_batch_pinned_host_tier(order, engine):
    lay = OLayout(2, 4, 32, 2, 16)
    st, items = setup_batch(lay, SPECS, tier=oc.TIER_PINNED_HOST)
    b = oc.Batch([it["desc"] for it in items], order=order)
    b.fetch(torch.cuda.current_stream(), engine=engine)
    torch.cuda.synchronize()
    for it in items:
        it["desc"].sync_layer(1)
    check(lay, items)
    b.close()
    st.close()


def test_batch_errors():
    lay = OLayout(2, 2, 64, 2, 16)
    st, items = setup_batch(lay, SPECS[:2])
    d = [it["desc"] for it in items]
    with pytest.raises(oc.ObjcacheError) as e:
        oc.Batch([d[0], d[0]])
    assert e.value.code == oc.OC_EINVAL
    with pytest.raises(oc.ObjcacheError) as e:
        oc.Batch([])
    assert e.value.code == oc.OC_EINVAL
    other = OLayout(2, 2, 64, 2, 8)
    st2, items2 = setup_batch(other, SPECS[:1])
    with pytest.raises(oc.ObjcacheError) as e:
        oc.Batch([d[0], items2[0]["desc"]])
    assert e.value.code == oc.OC_EINVAL
    b = oc.Batch(d)
    o = oc.CFetchOpts(oc.FETCH_PERSISTENT, oc.COPY_BULK, 0, 0, 1e9)
    assert oc._lib.oc_fetch_batch(b._h, o, None) == oc.OC_ENOTSUP
    o = oc.CFetchOpts(oc.FETCH_PER_LAYER, oc.COPY_BULK, 0, 0, 0.0)
    assert oc._lib.oc_fetch_batch(b._h, o, None) == oc.OC_ENOTSUP
    b.close()
    st.close()
    st2.close()


# ---- WDRR claim order (Alg. A2 lines 6-7) ------------------------------------------------------
@pytest.mark.parametrize("lay,unit_bytes", [(OLayout(3, 2, 64, 2, 16), 0), (OLayout(2, 4, 32, 2, 20), 3072),
                                            (OLayout(2, 4, 32, 2, 20), 1024), (OLayout(1, 1, 16, 2, 8), 0)])
@pytest.mark.parametrize("hold", [False, True])
@pytest.mark.parametrize("E", [0, 1, 3])
@pytest.mark.parametrize("engine", [oc.COPY_BULK, oc.COPY_AUTO])
def test_wdrr_parity(lay, unit_bytes, hold, E, engine):
    """Every byte lands as in the oracle whatever the interleaving (ragged units included: 3072 B
    units of 12 rows cut a 40-row slice into 12+12+12+4), and each request's layers are announced
    in order."""
    st, items = setup_batch(lay, SPECS)
    b = oc.Batch([it["desc"] for it in items])
    s = torch.cuda.Stream()
    weights = [2e9, 0.5e9, 7e9, 1e9, 3.3e9]
    b.fetch(s, unit_bytes=unit_bytes, wdrr_weights=weights, quantum_bytes=unit_bytes or 0, entry_units=E,
            hold_rates=hold, engine=engine)
    for it in items:
        it["desc"].sync_layer(lay.num_layers - 1)
    torch.cuda.synchronize()
    check(lay, items)
    for it in items:
        t = it["desc"].layer_times().astype(np.int64)
        assert np.all(np.diff(t[1:]) >= 0) and t[1] >= t[0]
    b.close()
    st.close()


@pytest.mark.parametrize("hold", [False, True])
@pytest.mark.parametrize("engine", [oc.COPY_BULK, oc.COPY_LDST])
def test_wdrr_layer_packets_parity(hold, engine):
    """Alg. A2 line 7 as written: DRR packets are whole layer payloads (layer_packets = L) -- the
    same bytes as the oracle, layers announced in order, through both copy engines."""
    lay = OLayout(3, 2, 64, 2, 16)
    st, items = setup_batch(lay, SPECS)
    b = oc.Batch([it["desc"] for it in items])
    s = torch.cuda.Stream()
    b.fetch(s, wdrr_weights=[2e9, 0.5e9, 7e9, 1e9, 3.3e9], hold_rates=hold, engine=engine,
            layer_packets=lay.num_layers)
    for it in items:
        it["desc"].sync_layer(lay.num_layers - 1)
    torch.cuda.synchronize()
    check(lay, items)
    for it in items:
        t = it["desc"].layer_times().astype(np.int64)
        assert np.all(np.diff(t[1:]) >= 0) and t[1] >= t[0]
    b.close()
    st.close()


def test_wdrr_refetch_mixed_with_other_orders():
    """Epoch bookkeeping across WDRR, layer-major batch and single fetches of the same descriptors
    (the WDRR observer reads each request's next layer back from its ready word)."""
    lay = OLayout(3, 2, 64, 2, 16)
    st, items = setup_batch(lay, SPECS)
    b = oc.Batch([it["desc"] for it in items])
    s, cons = torch.cuda.Stream(), torch.cuda.Stream()
    for rnd in range(6):
        with torch.cuda.stream(s):
            for it in items:
                it["buf"].fill_(0xA5)
        if rnd in (0, 3, 5):
            b.fetch(s, wdrr_weights=[1e9 * (k + 1) for k in range(len(items))], hold_rates=rnd == 3,
                    max_ctas=2 if rnd == 5 else 0)
        elif rnd == 1:
            b.fetch(s)
        else:
            for it in items:
                it["desc"].fetch_layerwise(s)
        for it in items:
            it["desc"].wait_layer(lay.num_layers - 1, cons)
        cons.synchronize()
        torch.cuda.synchronize()
        check(lay, items)
    b.close()
    st.close()


def test_wdrr_pinned_host_and_errors():
    lay = OLayout(2, 4, 32, 2, 16)
    st, items = setup_batch(lay, SPECS, tier=oc.TIER_PINNED_HOST)
    b = oc.Batch([it["desc"] for it in items])
    b.fetch(torch.cuda.current_stream(), wdrr_weights=[1.0, 2.0, 3.0, 4.0, 5.0])
    torch.cuda.synchronize()
    check(lay, items)
    with pytest.raises(ValueError):
        b.fetch(None, wdrr_weights=[1.0])
    with pytest.raises(oc.ObjcacheError) as e:
        b.fetch(None, wdrr_weights=[1.0, 1.0, 0.0, 1.0, 1.0])
    assert e.value.code == oc.OC_EINVAL
    b.close()
    st.close()


def big_pair(n_chunks):
    """Two Llama-3-8B-layout requests of n_chunks chunks each, HBM store, NHD paged targets."""
    import synth
    lay = synth.LLAMA3_8B.as_tuple()
    L, G, Bs = lay[0], lay[4], 16
    row, S, chunk = oc.geometry(lay)
    st = oc.Store(lay, capacity=2 * n_chunks)
    descs, caches = [], []
    for r in range(2):
        (tok,), _ = synth.family_streams(100 + r, G, 0, [n_chunks])
        keys = oc.chunk_keys(tok, G)
        for b0 in range(0, n_chunks, 64):
            b1 = min(n_chunks, b0 + 64)
            st.put_chunks(keys[b0:b1], torch.randint(0, 256, (b1 - b0, chunk), dtype=torch.uint8, device="cuda"))
        need = n_chunks * G // Bs
        cache = torch.empty((L, 2, need, Bs, row), dtype=torch.uint8, device="cuda")
        per_kv = need * Bs * row
        kb = [cache.data_ptr() + l * 2 * per_kv for l in range(L)]
        tgt = oc.PagedTarget(kb, [x + per_kv for x in kb], Bs * row, row, lay[2] * lay[3], Bs,
                             synth.block_table(r, need, need), 0)
        descs.append(oc.build_descriptor(st, keys, lay, tgt))
        caches.append(cache)
    torch.cuda.synchronize()
    return st, descs, caches, n_chunks * S * L


def finish_ms(d):
    t = d.layer_times().astype(np.int64)
    return (t[-1] - t[0]) / 1e6


def test_wdrr_work_conserving_shares():
    """Unpaced WDRR over a saturated link (HBM here) with weights 1:3 and equal payloads: the
    heavy request gets 3/4 of the bandwidth until it finishes, so its finish time is (4/3)/2 = 2/3
    of the light request's."""
    st, descs, caches, W = big_pair(1024)                        # 2 x 2 GiB
    b = oc.Batch(descs)
    s = torch.cuda.Stream()
    for _ in range(2):
        b.fetch(s, wdrr_weights=[1.0, 3.0])
        s.synchronize()
    ratio = finish_ms(descs[1]) / finish_ms(descs[0])
    assert 0.6 < ratio < 0.74, ratio
    b.close()
    st.close()


def test_wdrr_hold_rates():
    """hold_rates: request i is delivered at weights[i] bytes/s (Alg. A2 line 6): the last layer
    of a request lands at about W / r_i (the last entry's release plus one entry's copy)."""
    st, descs, caches, W = big_pair(256)                          # 2 x 512 MiB
    rates = [50e9, 150e9]
    b = oc.Batch(descs)
    s = torch.cuda.Stream()
    b.fetch(s, wdrr_weights=rates, hold_rates=True)
    s.synchronize()
    for d, r in zip(descs, rates):
        want = W / r * 1e3
        assert abs(finish_ms(d) - want) < 0.05 * want + 0.2, (finish_ms(d), want)
    b.close()
    st.close()


@pytest.mark.parametrize("order,blk_kib", [(oc.BATCH_BY_REQUEST, 0), (oc.BATCH_BY_POSITION, 24),
                                           (oc.BATCH_BY_POSITION, 4096)])
def test_batch_shared_prefix_family(order, blk_kib, monkeypatch):
    if blk_kib:
        monkeypatch.setenv("OC_BYPOS_BLOCK_KIB", str(blk_kib))
    """Requests of one prefix family (8 shared chunks, then own chunks; one request is the bare
    shared prefix) through one store: every member's bytes as the oracle, both orders, refetched."""
    lay = OLayout(3, 2, 64, 2, 16)
    reqs = requests_family(lay, 21, 8, [2, 0, 5, 3])
    with oc.Store(lay, capacity=64) as st:
        items = []
        for i, req in enumerate(reqs):
            keys = oc.chunk_keys(req.tokens, lay.chunk_tokens)
            st.put_chunks(keys, payload_stack(lay, 21, req.payload_ids))
            dest = make_dest(lay, req.n_chunks, "nhd" if i % 2 else "hnd", Bs=8, first_token=i, seed=40 + i)
            buf = sentinel_buffer(dest.size)
            desc = oc.build_descriptor(st, keys, lay, lib_target(oc, dest, buf.data_ptr()))
            items.append({"seed": 21, "req": req, "dest": dest, "buf": buf, "desc": desc})
        torch.cuda.synchronize()
        b = oc.Batch([it["desc"] for it in items], order=order)
        s = torch.cuda.Stream()
        for rnd in range(3):
            with torch.cuda.stream(s):
                for it in items:
                    it["buf"].fill_(0xA5)
            b.fetch(s, max_ctas=2 if rnd == 1 else 0, unit_bytes=1024 if rnd == 2 else 0)
            s.synchronize()
            check(lay, items)
        b.close()
        assert oc._lib.oc_batch_set_order(None, 1) == oc.OC_EINVAL


def test_wdrr_single_member_batch():
    """n = 1: WDRR degenerates to the member's own layer-major order (held rate or not)."""
    lay = OLayout(2, 2, 64, 2, 16)
    st, items = setup_batch(lay, SPECS[1:2])
    b = oc.Batch([items[0]["desc"]])
    s = torch.cuda.Stream()
    for hold in (False, True):
        with torch.cuda.stream(s):
            items[0]["buf"].fill_(0xA5)
        b.fetch(s, wdrr_weights=[2e9], hold_rates=hold, entry_units=1)
        s.synchronize()
        check(lay, items)
    b.close()
    st.close()


def test_wdrr_hold_rates_skip_mirrored_layers():
    """hold_rates on a pinned-host store that mirrors its chunks' first K layers in HBM (reading
    c24): the mirrored layers never cross the paced link, so they land at once and the request's
    pace covers only the other L-K layers -- the last layer lands at about (L-K)/L * W / r_i, not
    W / r_i.  Bytes equal the oracle's."""
    lay, K, n = OLayout(8, 2, 64, 2, 16), 2, 64
    rates = [200e6, 400e6]
    st = oc.Store(lay, capacity=2 * n + 2, tier=oc.TIER_PINNED_HOST)
    st.set_hot_layers(K)
    items = []
    for i, seed in enumerate((71, 72)):
        req = requests_family(lay, seed, 0, [n])[0]
        st.put_chunks(oc.chunk_keys(req.tokens, 16), payload_stack(lay, seed, req.payload_ids))
        dest = make_dest(lay, n, "nhd", Bs=16, first_token=3 * i, seed=seed)
        buf = sentinel_buffer(dest.size)
        desc = oc.build_descriptor(st, st.match_prefix(req.tokens), lay, lib_target(oc, dest, buf.data_ptr()))
        items.append({"seed": seed, "req": req, "dest": dest, "buf": buf, "desc": desc})
    W = n * lay.num_layers * 2 * 16 * 256                       # one request's bytes
    b = oc.Batch([it["desc"] for it in items])
    s = torch.cuda.Stream()
    # the default Q (256 KiB) is a quarter of one request's mirrored bytes: the mirrored units
    # still all go first (reading c25), so no mirrored unit waits behind a paced one
    b.fetch(s, wdrr_weights=rates, hold_rates=True, free_units=[0, 0])   # mirrors not declared
    s.synchronize()
    check(lay, items)
    t = items[0]["desc"].layer_times().astype(np.int64)
    want0 = (K - 1) / lay.num_layers * W / rates[0] * 1e3                # layer K-1 paced like the rest
    assert (t[K - 1] - t[0]) / 1e6 > 0.6 * want0, ((t[K - 1] - t[0]) / 1e6, want0)
    for it in items:
        it["buf"].fill_(0xA5)
    torch.cuda.synchronize()
    b.fetch(s, wdrr_weights=rates, hold_rates=True)                    # default: the members' mirrors
    s.synchronize()
    check(lay, items)
    for it, r in zip(items, rates):
        t = it["desc"].layer_times().astype(np.int64)
        assert (t[K - 1] - t[0]) / 1e6 < 0.5                     # mirrored layers: no pacing
        want = (lay.num_layers - K) / lay.num_layers * W / r * 1e3
        got = (t[-1] - t[0]) / 1e6
        assert abs(got - want) < 0.08 * want + 0.3, (got, want)
    b.close()
    st.close()
