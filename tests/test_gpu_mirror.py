"""The host copy of the ready word (oc_layers_ready, wait_layer's fast path): a layer the host sees
as announced is in place in device memory -- read back without any stream ordering, it equals the
oracle's Alg. A1 gather + paged scatter of that layer -- and the count is monotone
within a fetch, restarts with the next fetch (epochs) and is all-or-nothing for chunk-major
delivery (Eq. 2 chunkwise)."""
import time

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_2605_22850_b200 as oc  # noqa: E402
from oracle.geometry import Layout as OLayout, chunk_layer_bytes  # noqa: E402
from oracle.store import ChunkStore  # noqa: E402
from oracle import keys as okeys  # noqa: E402
from scenario import lib_target, make_dest, oracle_layer, payload_stack, requests_family, sentinel_buffer  # noqa: E402

pytestmark = pytest.mark.gpu

LAY = OLayout(8, 8, 128, 2, 16)   # Llama-3 head geometry, 8 layers: 64 KiB per chunk-layer


def _setup(n, seed, delivery=None):
    st = oc.Store(LAY, capacity=n, device=0)
    req = requests_family(LAY, seed, 0, [n])[0]
    keys = oc.chunk_keys(req.tokens, LAY.chunk_tokens)
    payload = payload_stack(LAY, seed, req.payload_ids)
    st.put_chunks(keys, payload)
    dest = make_dest(LAY, n, "nhd", Bs=16, seed=seed)
    buf = sentinel_buffer(dest.size)
    args = () if delivery is None else (delivery,)
    d = oc.build_descriptor(st, keys, LAY, lib_target(oc, dest, buf.data_ptr()), *args)
    ost = ChunkStore(LAY)
    oks = okeys.chunk_keys(req.tokens, LAY.chunk_tokens)[:n]
    ost.put(oks, payload)
    return st, d, dest, buf, ost, oks


@pytest.mark.parametrize("mode", ["persistent", "per_layer"])
def test_layers_ready_never_ahead_of_the_bytes(mode):
    n = 64
    st, d, dest, buf, ost, oks = _setup(n, 71)
    layer_bytes = n * chunk_layer_bytes(LAY)
    s = torch.cuda.Stream()
    if mode == "persistent":   # paced: layer l released at t0 + l * 2 ms (minimal pacer, reading c20)
        d.fetch_layerwise(s, pace_Bps=layer_bytes / 2e-3)
    else:
        d.fetch_layerwise(s, mode=oc.FETCH_PER_LAYER)
    seen, checked, t_end = 0, set(), time.time() + 20
    while seen < LAY.num_layers and time.time() < t_end:
        k = d.layers_ready()
        assert k >= seen, "layers_ready went backwards within a fetch"
        for l in range(seen, k):
            lo, want = oracle_layer(LAY, ost, oks, dest, l)
            got = buf[lo:lo + want.size].cpu().numpy()   # torch's current stream: no order with `s`
            assert np.array_equal(got, want), f"layer {l} reported ready before its bytes landed"
            checked.add(l)
        seen = k
    assert seen == LAY.num_layers and checked == set(range(LAY.num_layers))
    s.synchronize()
    # the next fetch starts from zero: nothing of epoch 2 is announced before its launch runs
    hold = torch.cuda.Stream()
    oc.emulate_compute(50_000_000, hold)                 # 50 ms in front of the second fetch
    d.fetch_layerwise(hold)
    assert d.layers_ready() == 0
    for l in range(LAY.num_layers):
        d.wait_layer(l, torch.cuda.current_stream())
    hold.synchronize()
    assert d.layers_ready() == LAY.num_layers
    d.close()
    st.close()


def test_wait_layer_fast_path_keeps_consumer_order():
    """Every wait after the layer is announced returns without enqueuing; the consumer still sees
    the bytes (a copy on the consumer stream after the waits equals the oracle)."""
    n = 32
    st, d, dest, buf, ost, oks = _setup(n, 72)
    s, cons = torch.cuda.Stream(), torch.cuda.Stream()
    d.fetch_layerwise(s)
    d.sync_layer(LAY.num_layers - 1)
    assert d.layers_ready() == LAY.num_layers
    out = torch.empty_like(buf)
    for l in range(LAY.num_layers):
        d.wait_layer(l, cons)
    with torch.cuda.stream(cons):
        out.copy_(buf)
    cons.synchronize()
    for l in range(LAY.num_layers):
        lo, want = oracle_layer(LAY, ost, oks, dest, l)
        assert np.array_equal(out[lo:lo + want.size].cpu().numpy(), want)
    d.close()
    st.close()


def test_layers_ready_chunk_major_all_or_nothing():
    n = 16
    st, d, dest, buf, ost, oks = _setup(n, 73, oc.DELIVER_CHUNK_MAJOR)
    hold = torch.cuda.Stream()
    oc.emulate_compute(30_000_000, hold)
    d.fetch_layerwise(hold)
    assert d.layers_ready() == 0
    hold.synchronize()
    assert d.layers_ready() == LAY.num_layers
    d.close()
    st.close()


def test_layers_ready_before_fetch_is_einval():
    st, d, dest, buf, ost, oks = _setup(4, 74)
    with pytest.raises(oc.ObjcacheError) as e:
        d.layers_ready()
    assert e.value.code == oc.OC_EINVAL
    d.close()
    st.close()
