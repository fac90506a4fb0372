"""Small fetches of every engine/mode/target under compute-sanitizer (memcheck / racecheck / synccheck)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import numpy as np
import torch
import paper_2605_22850_b200 as oc
from oracle.geometry import Layout
from scenario import lib_target, make_dest, oracle_result, payload_stack, requests_family, sentinel_buffer

lay = Layout(2, 2, 64, 2, 16)
ok = 0
SECTIONS = os.environ.get("OC_SAN_SECTIONS", "1,2,3,4,5,6,7").split(",")
for kind in (("nhd", "hnd") if "1" in SECTIONS else ()):
    for engine in (oc.COPY_BULK, oc.COPY_LDST):
        for mode in (oc.FETCH_PERSISTENT, oc.FETCH_PER_LAYER):
            req = requests_family(lay, 3, 0, [5])[0]
            with oc.Store(lay, capacity=8) as st:
                keys = oc.chunk_keys(req.tokens, 16)
                st.put_chunks(keys, payload_stack(lay, 3, req.payload_ids))
                dest = make_dest(lay, 5, kind, Bs=8, first_token=3, seed=1)
                buf = sentinel_buffer(dest.size)
                d = oc.build_descriptor(st, keys, lay, lib_target(oc, dest, buf.data_ptr()))
                s = torch.cuda.Stream()
                d.fetch_layerwise(s, engine=engine, mode=mode, unit_bytes=1024)
                d.wait_layer(1, torch.cuda.current_stream())
                assert np.array_equal(buf.cpu().numpy(), oracle_result(lay, 3, req, dest))
                if engine == oc.COPY_BULK and mode == oc.FETCH_PERSISTENT:
                    b = oc.Batch([d])
                    b.fetch(s)
                    d.sync_layer(1)
                    b.fetch(s, wdrr_weights=[1e9], hold_rates=True, entry_units=3)   # WDRR order
                    d.sync_layer(1)
                    assert np.array_equal(buf.cpu().numpy(), oracle_result(lay, 3, req, dest))
                    b.close()
                    src = make_dest(lay, 5, kind, Bs=8, first_token=3, seed=1)
                    st2 = oc.Store(lay, capacity=8)
                    oc.put_from_paged(st2, keys, lay, lib_target(oc, src, buf.data_ptr()), s)
                    s.synchronize()
                    st2.close()
                d.close()
                ok += 1
# descriptors built and fetched back to back on several streams (pooled blocks recycled), each
# with a consumer that waits on its last layer and runs a compute-window spin
req = requests_family(lay, 4, 0, [6])[0]
with oc.Store(lay, capacity=8) as st:
  if "2" in SECTIONS:
      keys = oc.chunk_keys(req.tokens, 16)
      st.put_chunks(keys, payload_stack(lay, 4, req.payload_ids))
      streams = [torch.cuda.Stream() for _ in range(4)]
      cons = torch.cuda.Stream()
      stamps = torch.zeros(2, dtype=torch.int64, device="cuda")
      live = []
      for i in range(12):
          dest = make_dest(lay, 6, "nhd", Bs=16, seed=10 + i)
          buf = sentinel_buffer(dest.size)
          d = oc.build_descriptor(st, keys, lay, lib_target(oc, dest, buf.data_ptr()))
          s = streams[i % 4]
          s.wait_stream(torch.cuda.current_stream())
          d.fetch_layerwise(s)
          d.wait_layer(1, cons)
          oc.emulate_compute(1000, cons, stamps)
          live.append((d, buf, dest))
          if len(live) > 4:
              d0, b0, de0 = live.pop(0)
              d0.sync_layer(1)
              assert np.array_equal(b0.cpu().numpy(), oracle_result(lay, 4, req, de0))
              d0.close()
              ok += 1
      for d0, b0, de0 in live:
          d0.sync_layer(1)
          assert np.array_equal(b0.cpu().numpy(), oracle_result(lay, 4, req, de0))
          d0.close()
          ok += 1
# a WDRR batch of three requests with uneven weights and held rates
with oc.Store(lay, capacity=24) as st:
  if "3" in SECTIONS:
      items = []
      for seed, n in ((5, 3), (6, 7), (7, 2)):
          r = requests_family(lay, seed, 0, [n])[0]
          k = oc.chunk_keys(r.tokens, 16)
          st.put_chunks(k, payload_stack(lay, seed, r.payload_ids))
          dest = make_dest(lay, n, "nhd", Bs=16, seed=seed)
          buf = sentinel_buffer(dest.size)
          items.append((seed, r, dest, buf, oc.build_descriptor(st, k, lay, lib_target(oc, dest, buf.data_ptr()))))
      b = oc.Batch([it[4] for it in items])
      s = torch.cuda.Stream()
      s.wait_stream(torch.cuda.current_stream())  # the sentinel fills are on the current stream
      for hold in (False, True):
          b.fetch(s, unit_bytes=1024, wdrr_weights=[1e9, 3e9, 0.5e9], quantum_bytes=1024, hold_rates=hold)
          for i, it in enumerate(items):
              it[4].sync_layer(1)
              want = oracle_result(lay, it[0], it[1], it[2])
              got = it[3].cpu().numpy()
              if not np.array_equal(got, want):
                  diff = np.nonzero(got != want)[0]
                  torch.cuda.synchronize()
                  late = np.array_equal(it[3].cpu().numpy(), want)
                  t = it[4].layer_times().astype(np.int64)
                  raise AssertionError(f"WDRR hold={hold} request {i}: {len(diff)} bytes differ (first at "
                                       f"{diff[:4].tolist()}), equal after a device sync: {late}, layer "
                                       f"times {(t - t[0]).tolist()}")
              ok += 1
      b.close()
      for it in items:
          it[4].close()
# the copy-engine path from a pinned-host store (two runs of slots), and strict pacing
if "4" in SECTIONS:
    fam = requests_family(lay, 8, 4, [2, 3])
    with oc.Store(lay, capacity=16, tier=oc.TIER_PINNED_HOST) as st:
        ka, kb = (oc.chunk_keys(r.tokens, 16) for r in fam)
        st.put_chunks(ka, payload_stack(lay, 8, fam[0].payload_ids))
        st.put_chunks(kb, payload_stack(lay, 8, fam[1].payload_ids))
        dest = make_dest(lay, fam[1].n_chunks, "hnd", Bs=8, first_token=2, seed=9)
        buf = sentinel_buffer(dest.size)
        d = oc.build_descriptor(st, kb, lay, lib_target(oc, dest, buf.data_ptr()))
        s = torch.cuda.Stream()
        for opts in ({"engine": oc.COPY_CE}, {"pace_Bps": 2e9, "pace_strict": True}, {"engine": oc.COPY_CE}):
            with torch.cuda.stream(s):
                buf.fill_(0xA5)
            d.fetch_layerwise(s, **opts)
            d.sync_layer(1)
            s.synchronize()
            assert np.array_equal(buf.cpu().numpy(), oracle_result(lay, 8, fam[1], dest)), opts
            ok += 1
        d.close()
        fdest = make_dest(lay, fam[1].n_chunks, "flat")       # CE straight into the client buffer
        fbuf = sentinel_buffer(fdest.size)
        d = oc.build_descriptor(st, kb, lay, lib_target(oc, fdest, fbuf.data_ptr()))
        d.fetch_layerwise(s, engine=oc.COPY_CE)
        d.sync_layer(1)
        s.synchronize()
        assert np.array_equal(fbuf.cpu().numpy(), oracle_result(lay, 8, fam[1], fdest))
        ok += 1
        d.close()
# a pinned-host store mirroring layer 0 in HBM: split launches and CE mirror copies
if "4" in SECTIONS:
    fam = requests_family(lay, 9, 3, [2, 1])
    with oc.Store(lay, capacity=8, tier=oc.TIER_PINNED_HOST) as st:
        st.set_hot_layers(1)
        kf = oc.chunk_keys(fam[0].tokens, 16)
        st.put_chunks(kf, payload_stack(lay, 9, fam[0].payload_ids))
        dest = make_dest(lay, fam[0].n_chunks, "nhd", Bs=8, seed=4)
        buf = sentinel_buffer(dest.size)
        d = oc.build_descriptor(st, kf, lay, lib_target(oc, dest, buf.data_ptr()))
        s = torch.cuda.Stream()
        for engine in (oc.COPY_BULK, oc.COPY_LDST, oc.COPY_CE):
            with torch.cuda.stream(s):
                buf.fill_(0xA5)
            d.fetch_layerwise(s, engine=engine)
            d.sync_layer(1)
            s.synchronize()
            assert np.array_equal(buf.cpu().numpy(), oracle_result(lay, 9, fam[0], dest)), engine
            ok += 1
        d.close()
        # WDRR with held rates over two members of the mirrored store: mirrored units first (c25)
        kg = oc.chunk_keys(fam[1].tokens, 16)
        st.put_chunks(kg, payload_stack(lay, 9, fam[1].payload_ids))
        items = []
        for i, r in enumerate(fam):
            dst = make_dest(lay, r.n_chunks, "hnd" if i else "nhd", Bs=8, seed=5 + i)
            bb = sentinel_buffer(dst.size)
            items.append((r, dst, bb, oc.build_descriptor(st, st.match_prefix(r.tokens), lay,
                                                          lib_target(oc, dst, bb.data_ptr()))))
        b = oc.Batch([it[3] for it in items])
        b.fetch(s, wdrr_weights=[2e8, 6e8], hold_rates=True, entry_units=2)
        s.synchronize()
        for r, dst, bb, dd in items:
            assert np.array_equal(bb.cpu().numpy(), oracle_result(lay, 9, r, dst))
            ok += 1
        b.close()
        for it in items:
            it[3].close()
# chain keys of a ragged batch on the GPU
if "5" in SECTIONS:
    from oracle import keys as okeys
    streams = [np.arange(n, dtype=np.uint32) * 7 + n for n in (0, 15, 16, 47, 160)]
    got = oc.chunk_keys_batch(streams, 16)
    for t, g in zip(streams, got):
        want = b"".join(okeys.chunk_keys(t, 16))
        assert g.tobytes() == want
        ok += 1
if "6" in SECTIONS:
    # round 2: a fetch in layer ranges (oc_fetch_layers, lean ring) and the host mirror's fast path
    lay4 = Layout(4, 2, 64, 2, 16)
    req = requests_family(lay4, 6, 0, [7])[0]
    with oc.Store(lay4, capacity=8) as st:
        keys = oc.chunk_keys(req.tokens, 16)
        st.put_chunks(keys, payload_stack(lay4, 6, req.payload_ids))
        for engine, lean in ((oc.COPY_BULK, True), (oc.COPY_BULK, False), (oc.COPY_LDST, False)):
            dest = make_dest(lay4, 7, "nhd", Bs=8, first_token=3, seed=2)
            buf = sentinel_buffer(dest.size)
            d = oc.build_descriptor(st, keys, lay4, lib_target(oc, dest, buf.data_ptr()))
            s, cons = torch.cuda.Stream(), torch.cuda.Stream()
            for l0, l1 in ((0, 1), (1, 3), (3, 4)):
                d.fetch_layers(l0, l1, s, engine=engine, unit_bytes=1024, lean=lean)
            for l in range(4):
                d.wait_layer(l, cons)
            cons.synchronize()
            assert d.layers_ready() == 4
            assert np.array_equal(buf.cpu().numpy(), oracle_result(lay4, 6, req, dest))
            d.close()
            ok += 1
if "7" in SECTIONS:
    # the yield launch (layer 0 persistent, then one unit per CTA), waits through the opt-in relay
    # stream, and a store whose HBM slots are padded (oc_slot_pitch) filled by put_chunks + offload
    lay20 = Layout(20, 8, 128, 2, 16)                     # 1.25 MiB chunks -> 41-granule pitch
    r1, r2 = requests_family(lay20, 12, 0, [3, 3])
    with oc.Store(lay20, capacity=6) as st:
        k1, k2 = oc.chunk_keys(r1.tokens, 16), oc.chunk_keys(r2.tokens, 16)
        st.put_chunks(k1, payload_stack(lay20, 12, r1.payload_ids))
        dest = make_dest(lay20, 3, "nhd", Bs=16, seed=3)
        buf = sentinel_buffer(dest.size)
        d = oc.build_descriptor(st, k1, lay20, lib_target(oc, dest, buf.data_ptr()))
        s, cons = torch.cuda.Stream(), torch.cuda.Stream()
        os.environ["OC_WAIT_RELAY"] = "1"
        d.fetch_layerwise(s, yield_sms=True)
        for l in range(20):
            d.wait_layer(l, cons)
        cons.synchronize()
        os.environ.pop("OC_WAIT_RELAY")
        want = oracle_result(lay20, 12, r1, dest)
        assert np.array_equal(buf.cpu().numpy(), want)
        ok += 1
        # offload request 1's delivered blocks under request 2's keys into the padded slots, then
        # fetch them back: request 2's keys now hold request 1's bytes
        s.wait_stream(cons)
        assert oc.put_from_paged(st, k2, lay20, lib_target(oc, dest, buf.data_ptr()), s) == 3
        buf2 = sentinel_buffer(dest.size)
        d2 = oc.build_descriptor(st, k2, lay20, lib_target(oc, dest, buf2.data_ptr()))
        d2.fetch_layerwise(s)
        d2.sync_layer(19)
        assert np.array_equal(buf2.cpu().numpy(), want)
        ok += 1
        d.close()
        d2.close()
torch.cuda.synchronize()
print("sanitize workload ok", ok)
