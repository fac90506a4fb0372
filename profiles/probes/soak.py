"""Soak: back-to-back 4K fetches of 4 rotating requests for a fixed wall time, the launch shape drawn
at random per fetch (TMA or LD/ST engine, persistent with OC_FETCH_OVERLAP or stream order, PER_LAYER,
yield, layer ranges with a one-unit-per-CTA continuation, and -- rarely -- AUTO from a pinned-host
store with 32 MiB layers, i.e. the copy-engine + scatter path), every destination verified against the oracle's bytes (computed once per request) after a
random subset of fetches.  Reports fetches, bytes, verifications and mismatches."""
import json, os, random, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))), "tests"))
import numpy as np
import torch
import paper_2605_22850_b200 as oc
import synth
from oracle.geometry import Layout
from scenario import lib_target, make_dest, oracle_result, payload_stack, requests_family, sentinel_buffer
secs = float(sys.argv[1]) if len(sys.argv) > 1 else 120
lay = Layout(*synth.LLAMA3_8B.as_tuple())
N = 256
store = oc.Store(lay, capacity=4 * N)
sets = []
for r in range(4):
    req = requests_family(lay, 300 + r, 0, [N])[0]
    keys = oc.chunk_keys(req.tokens, 16)
    for b0 in range(0, N, 64):
        store.put_chunks(keys[b0:b0 + 64], payload_stack(lay, 300 + r, req.payload_ids[b0:b0 + 64]))
    kind = "nhd" if r % 2 == 0 else "hnd"
    dest = make_dest(lay, N, kind, Bs=16, first_token=0, seed=310 + r, pool_factor=1.25)
    buf = sentinel_buffer(dest.size)
    want = oracle_result(lay, 300 + r, req, dest)
    d = oc.build_descriptor(store, keys, lay, lib_target(oc, dest, buf.data_ptr()))
    sets.append((d, buf, want, kind))
# pinned-host requests with 32 MiB layers (N = 512): AUTO takes the copy engine + scatter path
pstore = oc.Store(lay, capacity=2 * 2 * N, tier=oc.TIER_PINNED_HOST)
psets = []
for r in range(2):
    req = requests_family(lay, 400 + r, 0, [2 * N])[0]
    keys = oc.chunk_keys(req.tokens, 16)
    for b0 in range(0, 2 * N, 64):
        pstore.put_chunks(keys[b0:b0 + 64], payload_stack(lay, 400 + r, req.payload_ids[b0:b0 + 64]))
    kind = "nhd" if r == 0 else "hnd"
    dest = make_dest(lay, 2 * N, kind, Bs=16, first_token=0, seed=410 + r, pool_factor=1.25)
    buf = sentinel_buffer(dest.size)
    want = oracle_result(lay, 400 + r, req, dest)
    psets.append((oc.build_descriptor(pstore, keys, lay, lib_target(oc, dest, buf.data_ptr())), buf, want, kind))
s, cons = torch.cuda.Stream(), torch.cuda.Stream()
rng = random.Random(1)
shapes = [dict(engine=oc.COPY_BULK, overlap=True), dict(engine=oc.COPY_LDST, overlap=True), dict(engine=oc.COPY_AUTO),
          dict(mode=oc.FETCH_PER_LAYER, overlap=True), dict(engine=oc.COPY_BULK, yield_sms=True),
          dict(ranged=True), dict(pinned_auto=True)]
n, checks, bad, t0 = 0, 0, 0, time.time()
while time.time() - t0 < secs:
    i = n % 4
    d, buf, want, kind = sets[i]
    sh = dict(rng.choice(shapes))
    if sh.pop("pinned_auto", False):
        if rng.random() < 0.9:                       # keep the slow (PCIe) shape rare
            sh = dict(engine=oc.COPY_BULK, overlap=True)
        else:
            d, buf, want, kind = psets[n % 2]
            sh = dict(engine=oc.COPY_AUTO)
    if kind == "hnd" and sh.get("engine") == oc.COPY_BULK:
        sh["engine"] = oc.COPY_LDST                  # TMA per-piece stores into HND are slow, not wrong
    if sh.pop("ranged", False):                      # layer ranges, the continuation one unit per CTA
        d.fetch_layers(0, 2, s)
        d.fetch_layers(2, lay.num_layers, s, **({"yield_sms": True} if kind == "nhd" else {}))
    else:
        d.fetch_layerwise(s, **sh)
    d.wait_layer(lay.num_layers - 1, cons)
    n += 1
    if rng.random() < 0.02:                          # verify this delivery (ordered after its last layer)
        cons.synchronize()
        got = buf.cpu().numpy()
        checks += 1
        bad += int(not np.array_equal(got, want))
        with torch.cuda.stream(s):
            buf.fill_(0xA5)                          # the next fetch of this request must rewrite everything
        s.synchronize()                              # (and before any later launch can overlap the fill)
    if n % 64 == 0:
        torch.cuda.synchronize()
torch.cuda.synchronize()
print(json.dumps({"seconds": round(time.time() - t0, 1), "fetches": n, "bytes_rw": n * 2 * N * lay.num_layers * 65536,
                  "verified": checks, "mismatches": bad, "shapes": len(shapes)}))
for d_, _, _, _ in sets + psets:
    d_.close()
store.close()
pstore.close()
