"""Parity at the BASELINE layouts for the paths added on top of the single fetch: the CE engine on
the e2e configuration (Llama-3-8B, 4K hit, pinned-host store) and config-5-style batches of
prefix-sharing requests in every claim order, against the oracle (sampled layers for batches)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_2605_22850_b200 as oc  # noqa: E402
import synth  # noqa: E402
from oracle.geometry import Layout as OLayout  # noqa: E402
from scenario import (lib_target, make_dest, oracle_result, payload_stack,  # noqa: E402
                      requests_family, sentinel_buffer)

pytestmark = pytest.mark.gpu


def lay_of(named):
    return OLayout(*named.as_tuple())


def test_llama8b_4k_ce_engine_full():
    """The e2e leg's configuration: 256 chunks in the pinned-host store, CE engine, every layer."""
    lay = lay_of(synth.LLAMA3_8B)
    req = requests_family(lay, 4040, 0, [256])[0]
    dest = make_dest(lay, 256, "nhd", Bs=16, seed=41)
    with oc.Store(lay, capacity=256, tier=oc.TIER_PINNED_HOST) as st:
        keys = oc.chunk_keys(req.tokens, 16)
        assert st.put_chunks(keys, payload_stack(lay, 4040, req.payload_ids)) == 256
        buf = sentinel_buffer(dest.size)
        d = oc.build_descriptor(st, st.match_prefix(req.tokens), lay, lib_target(oc, dest, buf.data_ptr()))
        s = torch.cuda.Stream()
        d.fetch_layerwise(s, engine=oc.COPY_CE)
        d.sync_layer(lay.num_layers - 1)
        s.synchronize()
        assert np.array_equal(buf.cpu().numpy(), oracle_result(lay, 4040, req, dest))
        d.close()


@pytest.mark.parametrize("order", ["by_request", "by_position", "wdrr", "wdrr_held"])
def test_llama8b_prefix_family_batch(order):
    """Config 5 in miniature at the real layout: one family's 128-chunk shared prefix read by three
    requests (own tails 0 / 32 / 64 chunks) plus an unrelated 96-chunk request, one launch; every
    request's bytes on sampled layers equal the oracle's and the sentinels elsewhere survive."""
    lay = lay_of(synth.LLAMA3_8B)
    fam = requests_family(lay, 500, 128, [0, 32, 64])
    other = requests_family(lay, 501, 0, [96])[0]
    reqs = [(500, r) for r in fam] + [(501, other)]
    layers = (0, 13, 31)
    with oc.Store(lay, capacity=128 + 32 + 64 + 96) as st:
        items = []
        for i, (seed, r) in enumerate(reqs):
            keys = oc.chunk_keys(r.tokens, 16)
            st.put_chunks(keys, payload_stack(lay, seed, r.payload_ids))
            dest = make_dest(lay, r.n_chunks, "nhd", Bs=16, first_token=16 * i, seed=60 + i)
            buf = sentinel_buffer(dest.size)
            d = oc.build_descriptor(st, keys, lay, lib_target(oc, dest, buf.data_ptr()))
            items.append((seed, r, dest, buf, d))
        b = oc.Batch([it[4] for it in items],
                     order=oc.BATCH_BY_POSITION if order == "by_position" else oc.BATCH_BY_REQUEST)
        s = torch.cuda.Stream()
        if order.startswith("wdrr"):
            sizes = [float(it[1].n_chunks) * 65536 * 32 for it in items]
            rates = [x / 2e-3 for x in sizes]                     # every request done in ~2 ms
            b.fetch(s, wdrr_weights=rates, hold_rates=order == "wdrr_held")
        else:
            b.fetch(s)
        s.synchronize()
        for seed, r, dest, buf, d in items:
            d.sync_layer(lay.num_layers - 1)
            got = buf.cpu().numpy()
            want = oracle_result(lay, seed, r, dest, layers=layers)
            per_kv = dest.v_off[0] - dest.k_off[0]
            for l in layers:
                for off in (dest.k_off[l], dest.v_off[l]):
                    assert np.array_equal(got[off:off + per_kv], want[off:off + per_kv]), (order, l)
            assert np.all(got[:dest.k_off[0]] == 0xA5)
            t = d.layer_times().astype(np.int64)
            assert np.all(np.diff(t[1:]) >= 0)
        b.close()
        for it in items:
            it[4].close()
