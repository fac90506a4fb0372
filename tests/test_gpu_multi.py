"""Chunks homed on another GPU: the same fetch kernels read a peer
GPU's HBM store over NVLink.  Needs >= 2 GPUs (skipped otherwise; the one-GPU versions of these
paths -- a peer store and an IPC-imported store on the same device -- are in test_gpu_parity.py
and test_gpu_ipc.py).

1. One process: a store on GPU 1 attached as a peer of a store on GPU 0 (peer access enabled by
   attach_peer); half of a request's chunks live on each; fetched into a GPU 0 paged cache with
   the TMA, LD/ST and CE-free engines, in a WDRR batch, and with OC_FETCH_OVERLAP -- bit-exact.
2. Two processes on distinct devices: the owner on GPU 1 exports its store (CUDA IPC handle + key
   table); the consumer on GPU 0 imports it, attaches it and fetches -- bit-exact, every engine."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.multiprocessing as mp  # noqa: E402

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2,
                                 reason="needs two GPUs")]


def test_peer_store_on_another_gpu():
    import paper_2605_22850_b200 as oc
    from oracle.geometry import Layout
    from scenario import lib_target, make_dest, oracle_result, payload_stack, requests_family, sentinel_buffer
    for lay, n in ((Layout(3, 2, 64, 2, 16), 12), (Layout(32, 8, 128, 2, 16), 64)):
        req = requests_family(lay, 41, 0, [n])[0]
        keys = oc.chunk_keys(req.tokens, lay.chunk_tokens)
        pl = payload_stack(lay, 41, req.payload_ids)
        torch.cuda.set_device(0)
        local = oc.Store(lay, capacity=n, device=0)
        remote = oc.Store(lay, capacity=n, device=1)
        local.put_chunks(keys[:n // 2], pl[:n // 2])
        remote.put_chunks(keys[n // 2:], pl[n // 2:])
        local.attach_peer(remote)
        got = local.match_prefix(req.tokens)
        assert got.shape[0] == n
        dest = make_dest(lay, n, "nhd", Bs=16, first_token=3, seed=5)
        want = oracle_result(lay, 41, req, dest)
        buf = sentinel_buffer(dest.size, device="cuda:0")
        desc = oc.build_descriptor(local, got, lay, lib_target(oc, dest, buf.data_ptr()))
        s, cons = torch.cuda.Stream(0), torch.cuda.Stream(0)
        runs = [dict(engine=oc.COPY_BULK), dict(engine=oc.COPY_LDST), dict(engine=oc.COPY_BULK, overlap=True),
                dict(engine=oc.COPY_BULK, mode=oc.FETCH_PER_LAYER), dict(engine=oc.COPY_BULK, max_ctas=4)]
        for opts in runs:
            with torch.cuda.stream(s):
                buf.fill_(0xA5)
            desc.fetch_layerwise(s, **opts)
            desc.wait_layer(lay.num_layers - 1, cons)
            cons.synchronize()
            s.synchronize()
            assert np.array_equal(buf.cpu().numpy(), want), opts
        # the same request in a WDRR batch (held rates) next to a local one
        b = oc.Batch([desc])
        with torch.cuda.stream(s):
            buf.fill_(0xA5)
        b.fetch(s, wdrr_weights=[5e10], hold_rates=True)
        s.synchronize()
        desc.sync_layer(lay.num_layers - 1)
        assert np.array_equal(buf.cpu().numpy(), want)
        b.close()
        desc.close()
        local.close()
        remote.close()


def _owner(q, done):
    import paper_2605_22850_b200 as oc
    from oracle.geometry import Layout
    from scenario import payload_stack, requests_family
    torch.cuda.set_device(1)
    lay = Layout(4, 8, 128, 2, 16)
    req = requests_family(lay, 32, 0, [40])[0]
    keys = oc.chunk_keys(req.tokens, 16)
    st = oc.Store(lay, capacity=40, device=1)
    st.put_chunks(keys, payload_stack(lay, 32, req.payload_ids))
    torch.cuda.synchronize()
    q.put(st.export())
    done.wait(180)
    st.close()


def test_ipc_store_from_another_process_and_gpu():
    import paper_2605_22850_b200 as oc
    from oracle.geometry import Layout
    from scenario import lib_target, make_dest, oracle_result, requests_family, sentinel_buffer
    ctx = mp.get_context("spawn")
    q, done = ctx.Queue(), ctx.Event()
    p = ctx.Process(target=_owner, args=(q, done))
    p.start()
    try:
        blob = q.get(timeout=180)
        torch.cuda.set_device(0)
        lay = Layout(4, 8, 128, 2, 16)
        req = requests_family(lay, 32, 0, [40])[0]
        peer = oc.Store.import_(blob, device=0)
        local = oc.Store(lay, capacity=1, device=0)
        local.attach_peer(peer)
        keys = local.match_prefix(req.tokens)
        assert keys.shape[0] == 40
        dest = make_dest(lay, 40, "nhd", Bs=16, first_token=0, seed=8)
        want = oracle_result(lay, 32, req, dest)
        buf = sentinel_buffer(dest.size, device="cuda:0")
        desc = oc.build_descriptor(local, keys, lay, lib_target(oc, dest, buf.data_ptr()))
        for engine in (oc.COPY_BULK, oc.COPY_LDST):
            buf.fill_(0xA5)
            torch.cuda.synchronize()
            desc.fetch_layerwise(torch.cuda.current_stream(), engine=engine)
            desc.sync_layer(lay.num_layers - 1)
            torch.cuda.synchronize()
            assert np.array_equal(buf.cpu().numpy(), want), engine
        desc.close()
        local.close()
        peer.close()
    finally:
        done.set()
        p.join(timeout=60)
    assert p.exitcode == 0
