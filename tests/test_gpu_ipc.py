"""Cross-process chunk homes (config 5's peer reads, on one GPU): rank A owns a store and exports it
(CUDA IPC handle + key table); rank B imports it as a read-only peer, resolves half of a request
through it and fetches -- parity with the oracle, byte for byte."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.multiprocessing as mp  # noqa: E402

pytestmark = pytest.mark.gpu


# the tiny layout (dense slots) and one whose HBM slots are padded (oc_slot_pitch: 1.25 MiB chunks,
# 40 granules of 32 KiB -> 41): the importer must use the exporter's pitch
LAYOUTS = [(2, 2, 64, 2, 16), (20, 8, 128, 2, 16)]


def _owner(q, done, lay_t):
    import paper_2605_22850_b200 as oc
    from oracle.geometry import Layout
    from scenario import payload_stack, requests_family
    torch.cuda.set_device(0)
    lay = Layout(*lay_t)
    req = requests_family(lay, 31, 0, [12])[0]
    keys = oc.chunk_keys(req.tokens, 16)
    st = oc.Store(lay, capacity=16)
    st.put_chunks(keys[6:], payload_stack(lay, 31, req.payload_ids[6:]))
    q.put(st.export())
    done.wait(120)
    st.close()


@pytest.mark.parametrize("lay_t", LAYOUTS)
def test_export_import_across_processes(lay_t):
    import paper_2605_22850_b200 as oc
    from oracle.geometry import Layout
    from scenario import lib_target, make_dest, oracle_result, payload_stack, requests_family, sentinel_buffer
    ctx = mp.get_context("spawn")
    q, done = ctx.Queue(), ctx.Event()
    p = ctx.Process(target=_owner, args=(q, done, lay_t))
    p.start()
    try:
        blob = q.get(timeout=120)
        lay = Layout(*lay_t)
        if lay_t == LAYOUTS[1]:
            assert oc.slot_pitch(lay_t, oc.TIER_HBM) == 41 * 32768 > oc.geometry(lay_t)[2]
        req = requests_family(lay, 31, 0, [12])[0]
        keys = oc.chunk_keys(req.tokens, 16)
        local = oc.Store(lay, capacity=16)
        local.put_chunks(keys[:6], payload_stack(lay, 31, req.payload_ids[:6]))
        # a blob whose capacity x pitch exceeds the mapped slab is refused (and its mapping closed)
        bad = bytearray(blob)
        cap = int.from_bytes(bad[32:40], "little")
        assert cap == 16 and int.from_bytes(bad[48:56], "little") == oc.slot_pitch(lay_t, oc.TIER_HBM)
        bad[32:40] = (cap * 4096).to_bytes(8, "little")
        with pytest.raises(oc.ObjcacheError):
            oc.Store.import_(bytes(bad), device=0)
        peer = oc.Store.import_(blob, device=0)
        assert peer.count == 6
        with pytest.raises(oc.ObjcacheError):
            peer.put_chunks(keys[:1], payload_stack(lay, 31, req.payload_ids[:1]))   # read-only
        local.attach_peer(peer)
        got_keys = local.match_prefix(req.tokens)
        assert got_keys.shape[0] == 12
        dest = make_dest(lay, 12, "nhd", Bs=16, first_token=4, seed=3)
        buf = sentinel_buffer(dest.size)
        for engine in (oc.COPY_LDST, oc.COPY_BULK):
            buf.fill_(0xA5)
            desc = oc.build_descriptor(local, got_keys, lay, lib_target(oc, dest, buf.data_ptr()))
            desc.fetch_layerwise(torch.cuda.current_stream(), engine=engine)
            desc.sync_layer(1)
            torch.cuda.synchronize()
            assert np.array_equal(buf.cpu().numpy(), oracle_result(lay, 31, req, dest))
            desc.close()
        local.close()
        peer.close()
    finally:
        done.set()
        p.join(timeout=60)
    assert p.exitcode == 0
