"""Stall accounting on the device (Eq. 3): the compute-window spin
(oc.emulate_compute) stamps the same %globaltimer clock as the fetch's layer-ready stamps, so a
consumer chain's measured timeline can be checked against wait_layer's contract (no window of
layer l starts before layer l is ready) and against the oracle's free-running recurrence."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_2605_22850_b200 as oc  # noqa: E402
from oracle import stall as ostall  # noqa: E402
from oracle.geometry import Layout as OLayout, chunk_layer_bytes  # noqa: E402
from scenario import lib_target, make_dest, oracle_result, payload_stack, requests_family, sentinel_buffer  # noqa: E402

pytestmark = pytest.mark.gpu


def test_emulate_compute_duration_and_errors():
    stamps = torch.zeros(2, dtype=torch.int64, device="cuda")
    for ns in (0, 20_000, 1_000_000):
        oc.emulate_compute(ns, None, stamps)
        torch.cuda.synchronize()
        t0, t1 = stamps.tolist()
        assert t1 - t0 >= ns
        assert t1 - t0 < ns + 100_000
    oc.emulate_compute(1000)                                   # no stamps, default stream
    torch.cuda.synchronize()
    with pytest.raises(oc.ObjcacheError) as e:
        oc.emulate_compute(61 * 10**9)
    assert e.value.code == oc.OC_ERANGE
    with pytest.raises(oc.ObjcacheError) as e:
        oc.emulate_compute(10, None, stamps.data_ptr() + 4)
    assert e.value.code == oc.OC_EALIGN


def _setup(st, lay, seed, n, delivery=oc.DELIVER_LAYER_MAJOR):
    req = requests_family(lay, seed, 0, [n])[0]
    dest = make_dest(lay, n, "nhd", Bs=16, seed=seed)
    keys = oc.chunk_keys(req.tokens, lay.chunk_tokens)
    st.put_chunks(keys, payload_stack(lay, seed, req.payload_ids))
    buf = sentinel_buffer(dest.size)
    d = oc.build_descriptor(st, keys, lay, lib_target(oc, dest, buf.data_ptr()), delivery)
    return req, dest, buf, d


def _chain(d, L, C_ns, copy_s, cons, **fetch):
    stamps = torch.zeros((L, 2), dtype=torch.int64, device="cuda")
    torch.cuda.synchronize()
    d.fetch_layerwise(copy_s, **fetch)
    for l in range(L):
        d.wait_layer(l, cons)
        oc.emulate_compute(C_ns, cons, stamps[l])
    torch.cuda.synchronize()
    return d.layer_times().astype(np.int64), stamps.cpu().numpy()


@pytest.mark.parametrize("engine", [oc.COPY_BULK, oc.COPY_LDST])
@pytest.mark.parametrize("C_ms,X_ms", [(0.3, 1.0), (1.5, 0.5)])
def test_consumer_timeline_matches_free_running_model(engine, C_ms, X_ms):
    """Paced fetch (layer l released at t0 + l*X) under windows C: transfer-bound (X > C) and
    compute-bound (X < C) cases.  Every window starts after its layer is ready and after the
    previous window; the oracle's free-running recurrence on the measured ready times and window
    lengths predicts the measured end within a small per-layer dispatch overhead."""
    lay = OLayout(8, 2, 64, 2, 16)
    L = lay.num_layers
    with oc.Store(lay, capacity=8) as st:
        req, dest, buf, d = _setup(st, lay, 31, 8)
        copy_s, cons = torch.cuda.Stream(), torch.cuda.Stream()
        pace = 8 * chunk_layer_bytes(lay) / (X_ms * 1e-3)
        t, stamps = _chain(d, L, int(C_ms * 1e6), copy_s, cons, pace_Bps=pace, engine=engine)
        ready = t[1:] - t[0]
        start, end = stamps[:, 0] - t[0], stamps[:, 1] - t[0]
        assert np.all(start >= ready)                          # wait_layer holds the window back
        assert np.all(start[1:] >= end[:-1])                   # one consumer stream, in order
        assert np.all(end - start >= int(C_ms * 1e6))
        C = (end - start).astype(np.float64)
        model_end, m_start, _, _ = ostall.free_running(ready.astype(np.float64), C)
        assert end[-1] >= model_end - 1_000                    # never faster than the recurrence
        assert end[-1] - model_end < L * 60_000                # ≤ 60 µs dispatch overhead per layer
        # pacing: layer l is not ready before t0 + l * X
        assert np.all(ready >= np.arange(L) * X_ms * 1e6 - 50_000)
        assert np.array_equal(buf.cpu().numpy(), oracle_result(lay, 31, req, dest))
        d.close()


def test_chunkwise_delivery_holds_every_window():
    """Eq. 2 chunkwise side: with CHUNK_MAJOR delivery even layer 0's window waits for the whole
    prefix (all layers' bytes in place)."""
    lay = OLayout(6, 2, 64, 2, 16)
    L = lay.num_layers
    with oc.Store(lay, capacity=8) as st:
        req, dest, buf, d = _setup(st, lay, 33, 8, oc.DELIVER_CHUNK_MAJOR)
        copy_s, cons = torch.cuda.Stream(), torch.cuda.Stream()
        pace = 8 * chunk_layer_bytes(lay) / 1e-3                # one layer per ms -> prefix ~ L ms
        t, stamps = _chain(d, L, 10_000, copy_s, cons, pace_Bps=pace)
        start = stamps[:, 0] - t[0]
        assert start[0] >= (L - 1) * 1_000_000 - 50_000
        assert start[0] >= t[L] - t[0]
        assert np.array_equal(buf.cpu().numpy(), oracle_result(lay, 33, req, dest))
        d.close()


@pytest.mark.parametrize("strict", [False, True])
def test_pacer_release_schedule(strict):
    """Minimal pacer (c20): layer l starts at t0 + l*X and is copied at full speed, so it is ready
    just after l*X.  Strict pacing: byte b is released at t0 + b/r, so layer l (8 units) is ready
    only after its last unit's release at l*X + 7X/8."""
    lay = OLayout(8, 2, 64, 2, 16)
    L = lay.num_layers
    X = 0.5e-3
    with oc.Store(lay, capacity=8) as st:
        req, dest, buf, d = _setup(st, lay, 41, 8)
        s = torch.cuda.Stream()
        d.fetch_layerwise(s, pace_Bps=8 * chunk_layer_bytes(lay) / X, pace_strict=strict)
        d.sync_layer(L - 1)
        t = d.layer_times().astype(np.int64)
        ready = (t[1:] - t[0]) / 1e9
        for l in range(L):
            lo = l * X + (7 * X / 8 if strict else 0.0)
            assert lo - 20e-6 <= ready[l] <= lo + 150e-6, (l, ready[l], lo)
        if strict:   # over windows of >= 10 pacing quanta, delivered / elapsed <= 1.05 r
            s_layer = 8 * chunk_layer_bytes(lay)
            for i in range(L):
                for j in range(i + 2, L):
                    assert (j - i) * s_layer / (ready[j] - ready[i]) <= 1.05 * s_layer / X, (i, j)
        torch.cuda.synchronize()
        assert np.array_equal(buf.cpu().numpy(), oracle_result(lay, 41, req, dest))
        with pytest.raises(oc.ObjcacheError) as e:
            d.fetch_layerwise(s, pace_Bps=1e9, pace_strict=True, engine=oc.COPY_LDST)
        assert e.value.code == oc.OC_ENOTSUP
        d.close()


@pytest.mark.parametrize("strict", [False, True])
def test_pacer_skips_mirrored_layers(strict):
    """A pinned-host store mirroring layers 0-1 in HBM: the mirrored layers do not cross the paced
    link, so they are ready at once and the link's schedule starts with layer 2."""
    lay = OLayout(8, 2, 64, 2, 16)
    L, K, X = lay.num_layers, 2, 0.5e-3
    with oc.Store(lay, capacity=8, tier=oc.TIER_PINNED_HOST) as st:
        st.set_hot_layers(K)
        req, dest, buf, d = _setup(st, lay, 43, 8)
        s = torch.cuda.Stream()
        d.fetch_layerwise(s, pace_Bps=8 * chunk_layer_bytes(lay) / X, pace_strict=strict)
        d.sync_layer(L - 1)
        t = d.layer_times().astype(np.int64)
        ready = (t[1:] - t[0]) / 1e9
        for l in range(L):
            lo = 0.0 if l < K else (l - K) * X + (7 * X / 8 if strict else 0.0)
            assert lo - 20e-6 <= ready[l] <= lo + 200e-6, (l, ready[l], lo)
        torch.cuda.synchronize()
        assert np.array_equal(buf.cpu().numpy(), oracle_result(lay, 43, req, dest))
        d.close()
