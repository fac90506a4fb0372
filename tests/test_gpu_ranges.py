"""oc_fetch_layers: a fetch requested in layer ranges, each range launched when the consumer wants
it (the co-run schedule of the stall leg), delivers exactly what one fetch_layerwise does -- Alg. A1's
gather + paged scatter of every layer, whole buffer including sentinel bytes -- and
announces each range's layers in order (wait_layer / layers_ready)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_2605_22850_b200 as oc  # noqa: E402
import synth  # noqa: E402
from oracle.geometry import Layout as OLayout  # noqa: E402
from scenario import lib_target, make_dest, oracle_result, payload_stack, requests_family, sentinel_buffer  # noqa: E402

pytestmark = pytest.mark.gpu


def _setup(lay, n, seed, kind="nhd", Bs=16, first_token=0):
    st = oc.Store(lay, capacity=n, device=0)
    req = requests_family(lay, seed, 0, [n])[0]
    keys = oc.chunk_keys(req.tokens, lay.chunk_tokens)
    st.put_chunks(keys, payload_stack(lay, seed, req.payload_ids))
    dest = make_dest(lay, n, kind, Bs=Bs, first_token=first_token, seed=seed)
    buf = sentinel_buffer(dest.size)
    d = oc.build_descriptor(st, keys, lay, lib_target(oc, dest, buf.data_ptr()))
    return st, req, dest, buf, d


@pytest.mark.parametrize("ranges,opts", [
    ([(0, 1), (1, 2), (2, 5), (5, 8)], {}),
    ([(0, 2), (2, 8)], {"engine": oc.COPY_BULK, "max_ctas": 7, "unit_bytes": 8192, "lean": True}),
    ([(0, 1)] + [(l, l + 1) for l in range(1, 8)], {"engine": oc.COPY_LDST, "max_ctas": 5}),
    ([(0, 8)], {"lean": True}),
    # later ranges with one copy CTA per unit (OC_FETCH_YIELD on a continuation)
    ([(0, 2)] + [(l, l + 1) for l in range(2, 8)], {"engine": oc.COPY_BULK, "yield_later": True}),
])
def test_ranges_equal_oracle(ranges, opts):
    lay = OLayout(8, 8, 128, 2, 16)
    st, req, dest, buf, d = _setup(lay, 37, 81, Bs=16, first_token=5)
    streams = [torch.cuda.Stream(), torch.cuda.Stream(priority=-1)]
    cons = torch.cuda.Stream()
    prev = None
    opts = dict(opts)
    yield_later = opts.pop("yield_later", False)
    for i, (l0, l1) in enumerate(ranges):
        s = streams[i % 2]
        if prev is not None:          # ranges of one fetch in sequence (the caller's guarantee)
            s.wait_event(prev)
        d.fetch_layers(l0, l1, s, **opts, **({"yield_sms": True} if yield_later and l0 > 0 else {}))
        prev = torch.cuda.Event()
        prev.record(s)
        for l in range(l0, l1):
            d.wait_layer(l, cons)
    cons.synchronize()
    assert d.layers_ready() == lay.num_layers
    t = d.layer_times().astype(np.int64)
    assert np.all(np.diff(t[1:]) >= 0)
    assert np.array_equal(buf.cpu().numpy(), oracle_result(lay, 81, req, dest))
    # a second, whole fetch after the ranged one: same bytes again, next epoch
    buf.fill_(0xA5)
    torch.cuda.synchronize()
    d.fetch_layerwise(streams[0])
    d.sync_layer(lay.num_layers - 1)
    assert np.array_equal(buf.cpu().numpy(), oracle_result(lay, 81, req, dest))
    d.close()
    st.close()


def test_ranges_consumer_gated_hnd():
    """Each range waits for the consumer stream (the co-run schedule): layer l+1 is requested after
    the consumer has passed layer l; head-split target (LD/ST engine under AUTO)."""
    lay = OLayout(6, 4, 64, 2, 16)
    st, req, dest, buf, d = _setup(lay, 19, 82, kind="hnd", Bs=8)
    copy_s, cons = torch.cuda.Stream(), torch.cuda.Stream()
    d.fetch_layers(0, 1, copy_s)
    for l in range(lay.num_layers):
        d.wait_layer(l, cons)
        oc.emulate_compute(200_000, cons)
        if l + 1 < lay.num_layers:
            ev = torch.cuda.Event()
            ev.record(cons)
            copy_s.wait_event(ev)
            d.fetch_layers(l + 1, l + 2, copy_s)
    cons.synchronize()
    copy_s.synchronize()
    assert np.array_equal(buf.cpu().numpy(), oracle_result(lay, 82, req, dest))
    d.close()
    st.close()


def test_range_errors():
    lay = OLayout(4, 2, 16, 2, 16)
    st, req, dest, buf, d = _setup(lay, 6, 83)
    s = torch.cuda.Stream()
    for l0, l1 in ((0, 0), (2, 1), (0, 5)):
        with pytest.raises(oc.ObjcacheError) as e:
            d.fetch_layers(l0, l1, s)
        assert e.value.code == oc.OC_ERANGE
    with pytest.raises(oc.ObjcacheError) as e:      # no open fetch to continue
        d.fetch_layers(1, 2, s)
    assert e.value.code == oc.OC_EINVAL
    d.fetch_layers(0, 2, s, unit_bytes=4096)
    with pytest.raises(oc.ObjcacheError) as e:      # gap
        d.fetch_layers(3, 4, s)
    assert e.value.code == oc.OC_EINVAL
    with pytest.raises(oc.ObjcacheError) as e:      # the unit size belongs to the opening call
        d.fetch_layers(2, 3, s, unit_bytes=8192)
    assert e.value.code == oc.OC_EINVAL
    with pytest.raises(oc.ObjcacheError) as e:      # a new fetch while this one is open
        d.fetch_layerwise(s)
    assert e.value.code == oc.OC_EINVAL
    with pytest.raises(oc.ObjcacheError) as e:
        d.fetch_layers(0, 1, s)
    assert e.value.code == oc.OC_EINVAL
    with pytest.raises(oc.ObjcacheError) as e:
        d.fetch_layers(2, 3, s, engine=oc.COPY_CE)
    assert e.value.code == oc.OC_ENOTSUP
    d.fetch_layers(2, 4, s, unit_bytes=4096)
    s.synchronize()
    assert d.layers_ready() == lay.num_layers
    assert np.array_equal(buf.cpu().numpy(), oracle_result(lay, 83, req, dest))
    d.fetch_layerwise(s)                            # closed: a new fetch is accepted again
    s.synchronize()
    d.close()
    st.close()


def test_later_range_running_first_is_announced_in_order():
    """Range [0, 2) waits 30 ms behind a spin on its stream while range [2, 8) runs at once on
    another: layers 2.. complete first but are announced only after layers 0-1 (the observer of a
    later range waits for the earlier layers' announcement)."""
    import time
    lay = OLayout(8, 8, 128, 2, 16)
    st, req, dest, buf, d = _setup(lay, 29, 84)
    a, b = torch.cuda.Stream(), torch.cuda.Stream()
    oc.emulate_compute(30_000_000, a)
    d.fetch_layers(0, 2, a)
    d.fetch_layers(2, 8, b)
    time.sleep(0.01)
    assert d.layers_ready() == 0           # range [2, 8) is done or running, layers 0-1 are not
    b.synchronize()                        # the later range's kernel ends only after announcing
    assert d.layers_ready() == lay.num_layers
    a.synchronize()
    t = d.layer_times().astype(np.int64)
    assert np.all(np.diff(t[1:]) >= 0)
    assert np.array_equal(buf.cpu().numpy(), oracle_result(lay, 84, req, dest))
    d.close()
    st.close()
