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
