"""Randomised parity: 400 seeded configurations drawn over the whole option space -- layout (L,
n_kv, d, p, G), chunk count, target (paged NHD / head-split HND / flat), block size and first-token
offset, store tier (HBM, pinned host), engine (AUTO, TMA, LD/ST, copy engine), mode (persistent,
per-layer events), unit size, copy-CTA cap,
and delivery as one fetch or as layer ranges (oc_fetch_layers) -- each delivery compared byte for
byte, sentinels included, with the oracle's Alg. A1 gather + paged scatter.  The
draws are deterministic (seeded), so a failure names a reproducible case."""
import random

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_2605_22850_b200 as oc  # noqa: E402
from oracle.geometry import Layout as OLayout  # noqa: E402
from scenario import lib_target, make_dest, oracle_result, payload_stack, requests_family, sentinel_buffer  # noqa: E402

pytestmark = pytest.mark.gpu


def _case(i):
    r = random.Random(9000 + i)
    lay = OLayout(r.choice([1, 2, 3, 5, 8]), r.choice([1, 2, 4, 8]), r.choice([8, 16, 64, 128]),
                  r.choice([1, 2, 4]), r.choice([4, 8, 16, 32]))
    if (lay.head_dim * lay.elem_bytes) % 16:        # d*p must be a 16-byte multiple (OC_EALIGN otherwise)
        lay = OLayout(lay.num_layers, lay.kv_heads, lay.head_dim, 16 // lay.head_dim * 2, lay.chunk_tokens)
    row = lay.kv_heads * lay.head_dim * lay.elem_bytes
    kind = r.choice(["nhd", "nhd", "hnd", "flat"])
    opts = {}
    engine = r.choice(["auto", "bulk", "ldst"])
    if engine != "auto":
        opts["engine"] = oc.COPY_BULK if engine == "bulk" else oc.COPY_LDST
    if r.random() < 0.3:
        opts["max_ctas"] = r.choice([1, 3, 17, 150])
    if r.random() < 0.4:
        opts["unit_bytes"] = r.choice([row, 2 * row, 4096, 16384, 65536])
    ranged = r.random() < 0.25 and lay.num_layers > 1
    if not ranged and r.random() < 0.25:
        opts["mode"] = oc.FETCH_PER_LAYER
    host = r.random() < 0.2                         # pinned-host chunk store (PCIe reads)
    if host and not ranged and "mode" not in opts and r.random() < 0.5:
        opts["engine"] = oc.COPY_CE                 # copy engine into an HBM stage + the scatter kernel
        opts.pop("max_ctas", None)
    return dict(lay=lay, n=r.randint(1, 40), kind=kind, Bs=r.choice([1, 4, 8, 16, 32]),
                first=r.randint(0, 20) if kind != "flat" else 0, opts=opts, ranged=ranged, seed=9100 + i,
                split=r.randint(1, lay.num_layers - 1) if ranged else 0,
                tier=oc.TIER_PINNED_HOST if host else oc.TIER_HBM)


@pytest.mark.parametrize("i", range(400))
def test_random_configuration(i):
    c = _case(i)
    lay, n = c["lay"], c["n"]
    req = requests_family(lay, c["seed"], 0, [n])[0]
    st = oc.Store(lay, capacity=n, tier=c["tier"], device=0)
    keys = oc.chunk_keys(req.tokens, lay.chunk_tokens)
    st.put_chunks(keys, payload_stack(lay, c["seed"], req.payload_ids))
    dest = make_dest(lay, n, c["kind"], Bs=c["Bs"], first_token=c["first"], seed=c["seed"])
    buf = sentinel_buffer(dest.size)
    d = oc.build_descriptor(st, keys, lay, lib_target(oc, dest, buf.data_ptr()))
    s, cons = torch.cuda.Stream(), torch.cuda.Stream()
    if c["ranged"]:
        ro = {k: v for k, v in c["opts"].items() if k in ("engine", "max_ctas", "unit_bytes")}
        if ro.get("engine") is None and c["kind"] == "flat":
            ro["engine"] = oc.COPY_BULK
        d.fetch_layers(0, c["split"], s, **ro)
        d.fetch_layers(c["split"], lay.num_layers, s, **{k: v for k, v in ro.items() if k != "unit_bytes"})
    else:
        d.fetch_layerwise(s, **c["opts"])
    for l in range(lay.num_layers):
        d.wait_layer(l, cons)
    cons.synchronize()
    s.synchronize()
    assert d.layers_ready() == lay.num_layers
    got = buf.cpu().numpy()
    want = oracle_result(lay, c["seed"], req, dest)
    bad = np.flatnonzero(got != want)
    assert bad.size == 0, f"case {i} {c}: {bad.size} bytes differ, first at {bad[:4]}"
    t = d.layer_times().astype(np.int64)
    assert np.all(np.diff(t[1:]) >= 0), f"case {i}: layers announced out of order"
    d.close()
    st.close()


def _batch_case(i):
    r = random.Random(7000 + i)
    lay = OLayout(r.choice([1, 2, 4, 6]), r.choice([1, 2, 8]), r.choice([16, 64, 128]), 2, r.choice([8, 16, 32]))
    n_members = r.randint(1, 6)
    shared = r.randint(0, 6)                        # members of one prefix family share `shared` chunks
    own = [r.randint(0 if shared else 1, 12) for _ in range(n_members)]
    kinds = [r.choice(["nhd", "nhd", "hnd"]) for _ in range(n_members)]
    order = r.choice(["request", "position", "wdrr", "wdrr_held", "wdrr_layer"])
    engine = r.choice(["auto", "bulk", "ldst"]) if order in ("request", "position") else "bulk"
    return dict(lay=lay, shared=shared, own=own, kinds=kinds, order=order, engine=engine,
                Bs=r.choice([4, 8, 16]), seed=7100 + i, unit=r.choice([0, 0, 4096, 16384]),
                max_ctas=r.choice([0, 0, 2, 9]))


@pytest.mark.parametrize("i", range(120))
def test_random_batch(i):
    """One launch for several requests of one prefix family (shared chunks read through one store
    slot), in a random claim order -- by request, position-major, or weighted deficit round robin
    (unit or layer-payload packets, rates held or not; Alg. A2 line 7) -- every member's delivery
    byte-exact against the oracle."""
    c = _batch_case(i)
    lay = c["lay"]
    reqs = requests_family(lay, c["seed"], c["shared"], c["own"])
    st = oc.Store(lay, capacity=c["shared"] + sum(c["own"]), device=0)
    for rq in reqs:
        st.put_chunks(oc.chunk_keys(rq.tokens, lay.chunk_tokens), payload_stack(lay, c["seed"], rq.payload_ids))
    dests = [make_dest(lay, rq.n_chunks, k, Bs=c["Bs"], first_token=j % 5, seed=c["seed"] + j)
             for j, (rq, k) in enumerate(zip(reqs, c["kinds"]))]
    bufs = [sentinel_buffer(dd.size) for dd in dests]
    descs = [oc.build_descriptor(st, st.match_prefix(rq.tokens), lay, lib_target(oc, dd, b.data_ptr()))
             for rq, dd, b in zip(reqs, dests, bufs)]
    order = oc.BATCH_BY_POSITION if c["order"] == "position" else oc.BATCH_BY_REQUEST
    b = oc.Batch(descs, order=order)
    s, cons = torch.cuda.Stream(), torch.cuda.Stream()
    eng = {"auto": oc.COPY_AUTO, "bulk": oc.COPY_BULK, "ldst": oc.COPY_LDST}[c["engine"]]
    kw = dict(engine=eng, unit_bytes=c["unit"], max_ctas=c["max_ctas"])
    if c["order"].startswith("wdrr"):
        rates = [float(random.Random(c["seed"] + j).choice([2e9, 5e9, 2e10])) for j in range(len(descs))]
        kw.update(wdrr_weights=rates, hold_rates=c["order"] == "wdrr_held",
                  layer_packets=lay.num_layers if c["order"] == "wdrr_layer" else 0)
    b.fetch(s, **kw)
    for dsc in descs:
        dsc.wait_layer(lay.num_layers - 1, cons)
    cons.synchronize()
    s.synchronize()
    for j, (rq, dd, buf) in enumerate(zip(reqs, dests, bufs)):
        got = buf.cpu().numpy()
        want = oracle_result(lay, c["seed"], rq, dd)
        bad = np.flatnonzero(got != want)
        assert bad.size == 0, f"batch case {i} member {j} {c}: {bad.size} bytes differ"
    b.close()
    for dsc in descs:
        dsc.close()
    st.close()


@pytest.mark.parametrize("i", range(80))
def test_random_offload(i, monkeypatch):
    """The offload path (paged KV -> new chunk objects, oc_put_from_paged) on random layouts,
    targets, block sizes and offsets, both kernels, HBM or pinned-host store: the stored chunks,
    read back through a flat fetch (the Alg. A1 client buffer), equal the oracle's offload of the
    same cache bytes followed by its gather."""
    from oracle import keys as okeys
    from oracle.assemble import fetch_layerwise as ofetch, offload_paged
    from oracle.descriptor import FlatTarget as OFlat, build_descriptor as obuild
    from oracle.geometry import chunk_layer_bytes
    from oracle.store import ChunkStore
    from scenario import oracle_target
    r = random.Random(6000 + i)
    lay = OLayout(r.choice([1, 2, 3, 5]), r.choice([1, 2, 8]), r.choice([16, 32, 128]), 2, r.choice([8, 16, 32]))
    n = r.randint(1, 24)
    kind = r.choice(["nhd", "nhd", "hnd"])
    monkeypatch.setenv("OC_OFFLOAD_ENGINE", r.choice(["bulk", "ldst"]))
    tier = oc.TIER_PINNED_HOST if r.random() < 0.25 else oc.TIER_HBM
    req = requests_family(lay, 6100 + i, 0, [n])[0]
    src = make_dest(lay, n, kind, Bs=r.choice([4, 8, 16, 32]), first_token=r.randint(0, 19), seed=6100 + i)
    gen = torch.Generator(device="cuda").manual_seed(6100 + i)
    cache = torch.randint(0, 256, (src.size,), dtype=torch.uint8, device="cuda", generator=gen)
    keys = oc.chunk_keys(req.tokens, lay.chunk_tokens)
    W = n * lay.num_layers * chunk_layer_bytes(lay)
    with oc.Store(lay, capacity=n, tier=tier) as st:
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        assert oc.put_from_paged(st, keys, lay, lib_target(oc, src, cache.data_ptr()), s) == n
        s.synchronize()
        flat = sentinel_buffer(W)
        d = oc.build_descriptor(st, keys, lay, oc.FlatTarget(flat.data_ptr(), W))
        d.fetch_layerwise(s)
        d.sync_layer(lay.num_layers - 1)
        got = flat.cpu().numpy()
        d.close()
    ost = ChunkStore(lay)
    ok_ = okeys.chunk_keys(req.tokens, lay.chunk_tokens)
    assert offload_paged(ost, ok_, lay, oracle_target(src), cache.cpu().numpy()) == n
    want = np.full(W, 0xA5, np.uint8)
    ofetch(ost, obuild(ost, ok_, lay, OFlat(0, W)), want)
    bad = np.flatnonzero(got != want)
    assert bad.size == 0, f"offload case {i}: {bad.size} bytes differ"
