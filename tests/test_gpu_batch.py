"""Batched fetch (several requests, one launch, layer-major across the batch) vs the oracle."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_2605_22850_b200 as oc  # noqa: E402
from oracle.geometry import Layout as OLayout  # noqa: E402
from scenario import lib_target, make_dest, oracle_result, payload_stack, requests_family  # noqa: E402

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
        buf = torch.full((dest.size,), 0xA5, dtype=torch.uint8, device="cuda")
        desc = oc.build_descriptor(st, st.match_prefix(req.tokens), lay, lib_target(oc, dest, buf.data_ptr()))
        items.append({"seed": seed, "req": req, "dest": dest, "buf": buf, "desc": desc})
    return st, items


def check(lay, items):
    for it in items:
        want = oracle_result(lay, it["seed"], it["req"], it["dest"])
        got = it["buf"].cpu().numpy()
        assert np.array_equal(got, want), f"request seed {it['seed']} differs"


SPECS = [(1, 3, "nhd", 16, 0), (2, 7, "hnd", 8, 5), (3, 1, "flat", 16, 0), (4, 12, "nhd", 32, 17),
         (5, 5, "nhd", 1, 2)]


@pytest.mark.parametrize("lay", [OLayout(3, 2, 64, 2, 16), OLayout(2, 4, 32, 2, 20)])
@pytest.mark.parametrize("unit_bytes", [0, 1024])
def test_batch_parity(lay, unit_bytes):
    st, items = setup_batch(lay, SPECS)
    b = oc.Batch([it["desc"] for it in items])
    s = torch.cuda.Stream()
    b.fetch(s, unit_bytes=unit_bytes)
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


def test_batch_pinned_host_tier():
    lay = OLayout(2, 4, 32, 2, 16)
    st, items = setup_batch(lay, SPECS, tier=oc.TIER_PINNED_HOST)
    b = oc.Batch([it["desc"] for it in items])
    b.fetch(torch.cuda.current_stream())
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
