"""Many descriptors built and fetched back to back on several non-blocking streams, with pooled
descriptor memory recycled as earlier requests retire (the serving pattern of config 5).  Every
fetch must see its own freshly uploaded descriptor block: launches are ordered after the
block's host -> device upload, never after a plain cudaMemcpy that may still be in flight."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_2605_22850_b200 as oc  # noqa: E402
from oracle.geometry import Layout as OLayout  # noqa: E402
from scenario import Request, lib_target, make_dest, oracle_result, payload_stack, requests_family, sentinel_buffer  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("engine", [oc.COPY_BULK, oc.COPY_LDST])
def test_streams_of_requests_with_recycled_descriptors(engine):
    lay = OLayout(4, 2, 64, 2, 16)
    fams = [requests_family(lay, 900 + f, 0, [24])[0] for f in range(4)]
    rng = np.random.default_rng(7)
    streams = [torch.cuda.Stream() for _ in range(8)]
    with oc.Store(lay, capacity=4 * 24) as st:
        keys = []
        for f, req in enumerate(fams):
            k = oc.chunk_keys(req.tokens, 16)
            st.put_chunks(k, payload_stack(lay, 900 + f, req.payload_ids))
            keys.append(k)
        inflight, checked = [], 0

        def retire(item):
            ev, d, buf, want = item
            ev.synchronize()
            assert np.array_equal(buf.cpu().numpy(), want)
            d.close()

        for i in range(160):
            f = int(rng.integers(0, 4))
            n = int(rng.integers(1, 25))
            req = Request(fams[f].tokens, fams[f].payload_ids, n)
            dest = make_dest(lay, n, "nhd", Bs=int(rng.choice([8, 16, 32])), seed=i)
            want = oracle_result(lay, 900 + f, req, dest)
            buf = sentinel_buffer(dest.size)
            d = oc.build_descriptor(st, keys[f][:n], lay, lib_target(oc, dest, buf.data_ptr()))
            s = streams[i % len(streams)]
            s.wait_stream(torch.cuda.current_stream())          # buf's fill happened on the current stream
            d.fetch_layerwise(s, engine=engine)
            ev = torch.cuda.Event()
            ev.record(s)
            inflight.append((ev, d, buf, want))
            if len(inflight) > 12:
                retire(inflight.pop(0))
                checked += 1
        for item in inflight:
            retire(item)
            checked += 1
        assert checked == 160


def test_consumer_wait_on_fresh_descriptor():
    """A consumer waits on a brand-new descriptor right after its fetch is enqueued: the ready word
    it waits on was just uploaded, possibly into a recycled block whose old word was large."""
    lay = OLayout(4, 2, 64, 2, 16)
    req = requests_family(lay, 950, 0, [8])[0]
    with oc.Store(lay, capacity=8) as st:
        k = oc.chunk_keys(req.tokens, 16)
        st.put_chunks(k, payload_stack(lay, 950, req.payload_ids))
        dest = make_dest(lay, 8, "flat")
        want = oracle_result(lay, 950, req, dest)
        for it in range(40):
            # age a block: many epochs push its ready word far up, then recycle it
            scratch = torch.empty(dest.size, dtype=torch.uint8, device="cuda")
            old = oc.build_descriptor(st, k, lay, lib_target(oc, dest, scratch.data_ptr()))
            for _ in range(3):
                old.fetch_layerwise(pace_Bps=0.0)
            torch.cuda.synchronize()
            old.close()
            del scratch
            buf = sentinel_buffer(dest.size)
            copy_s, cons = torch.cuda.Stream(), torch.cuda.Stream()
            copy_s.wait_stream(torch.cuda.current_stream())
            d = oc.build_descriptor(st, k, lay, lib_target(oc, dest, buf.data_ptr()))
            d.fetch_layerwise(copy_s, pace_Bps=8 * 2048 * 4 / 2e-3)    # one layer per 2 ms
            d.wait_layer(lay.num_layers - 1, cons)
            with torch.cuda.stream(cons):
                snap = buf.clone()
            torch.cuda.synchronize()
            assert np.array_equal(snap.cpu().numpy(), want), it
            d.close()


def test_every_path_at_once():
    """Single fetches (TMA, LD/ST, strict-paced), CE fetches from a pinned-host store, and batches
    in every claim order, all in flight together on their own streams and recycled as they retire:
    no path may disturb another's pooled descriptor blocks, claim counters or stages."""
    lay = OLayout(3, 2, 64, 2, 16)
    rng = np.random.default_rng(11)
    fams = [requests_family(lay, 970 + f, 0, [20])[0] for f in range(3)]
    streams = [torch.cuda.Stream() for _ in range(6)]
    with oc.Store(lay, capacity=64) as hbm, oc.Store(lay, capacity=64, tier=oc.TIER_PINNED_HOST) as host:
        keys = []
        for f, req in enumerate(fams):
            k = oc.chunk_keys(req.tokens, 16)
            pl = payload_stack(lay, 970 + f, req.payload_ids)
            hbm.put_chunks(k, pl)
            host.put_chunks(k, pl)
            keys.append(k)

        def new_item(i, store):
            f = int(rng.integers(0, 3))
            n = int(rng.integers(1, 21))
            req = Request(fams[f].tokens, fams[f].payload_ids, n)
            dest = make_dest(lay, n, str(rng.choice(["nhd", "hnd", "flat"])), Bs=int(rng.choice([8, 16])),
                             seed=1000 + i)
            buf = sentinel_buffer(dest.size)
            d = oc.build_descriptor(store, keys[f][:n], lay, lib_target(oc, dest, buf.data_ptr()))
            return d, buf, oracle_result(lay, 970 + f, req, dest)

        inflight = []

        def retire(item):
            ev, ds, bufs, wants, batch = item
            ev.synchronize()
            for buf, want in zip(bufs, wants):
                assert np.array_equal(buf.cpu().numpy(), want)
            if batch is not None:
                batch.close()
            for d in ds:
                d.close()

        for i in range(60):
            s = streams[i % len(streams)]
            kind = i % 6
            if kind < 4:
                d, buf, want = new_item(i, host if kind == 3 else hbm)
                s.wait_stream(torch.cuda.current_stream())
                opts = [{"engine": oc.COPY_BULK}, {"engine": oc.COPY_LDST},
                        {"engine": oc.COPY_BULK, "pace_Bps": 4e9, "pace_strict": True},
                        {"engine": oc.COPY_CE}][kind]
                d.fetch_layerwise(s, **opts)
                ds, bufs, wants, batch = [d], [buf], [want], None
            else:
                items = [new_item(i * 10 + m, hbm) for m in range(3)]
                ds, bufs, wants = [x[0] for x in items], [x[1] for x in items], [x[2] for x in items]
                s.wait_stream(torch.cuda.current_stream())
                if kind == 4:
                    batch = oc.Batch(ds, order=oc.BATCH_BY_POSITION)
                    batch.fetch(s)
                else:
                    batch = oc.Batch(ds)
                    batch.fetch(s, wdrr_weights=[1e9, 2e9, 5e9], hold_rates=bool(i % 2))
            ev = torch.cuda.Event()
            ev.record(s)
            inflight.append((ev, ds, bufs, wants, batch))
            if len(inflight) > 8:
                retire(inflight.pop(0))
        for item in inflight:
            retire(item)
