"""4K fetch GB/s into NHD vs HND paged targets (Llama-3-8B layout), bulk and LD/ST engines."""
import json, sys
sys.path.insert(0, ".")
import torch
import paper_2605_22850_b200 as oc
import synth
lay = synth.LLAMA3_8B.as_tuple()
L, G, Bs = lay[0], lay[4], 16
row, S, chunk = oc.geometry(lay)
hd = lay[2] * lay[3]
N = 256
store = oc.Store(lay, capacity=N)
(tok,), _ = synth.family_streams(1, G, 0, [N])
keys = oc.chunk_keys(tok, G)
store.put_chunks(keys, torch.randint(0, 256, (N, chunk), dtype=torch.uint8, device="cuda"))
need = N * G // Bs
pool = need + need // 4
bt = synth.block_table(7, need, pool)
cache = torch.empty(L * 2 * pool * Bs * row, dtype=torch.uint8, device="cuda")
base = cache.data_ptr()
per_kv = pool * Bs * row
nhd = oc.PagedTarget([base + l * 2 * per_kv for l in range(L)], [base + l * 2 * per_kv + per_kv for l in range(L)],
                     Bs * row, row, hd, Bs, bt, 0)
blk = 2 * lay[1] * Bs * hd                                  # HND: [L][pool][2][n_kv][Bs][d]
hnd = oc.PagedTarget([base + l * pool * blk for l in range(L)], [base + l * pool * blk + lay[1] * Bs * hd for l in range(L)],
                     blk, hd, Bs * hd, Bs, bt, 0)
s = torch.cuda.Stream()
for name, tgt in (("nhd", nhd), ("hnd", hnd)):
    d = oc.build_descriptor(store, keys, lay, tgt)
    for eng_name, eng in (("bulk", oc.COPY_BULK), ("ldst", oc.COPY_LDST), ("auto", oc.COPY_AUTO)):
        for _ in range(3):
            d.fetch_layerwise(s, engine=eng)
        s.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        for _ in range(20):
            d.fetch_layerwise(s, engine=eng)
        b.record(s)
        s.synchronize()
        ms = a.elapsed_time(b) / 20
        print(json.dumps({"target": name, "engine": eng_name, "us": round(ms * 1e3, 1),
                          "GBps": round(2 * N * S * L / ms / 1e6, 1)}), flush=True)
    d.close()
# batches of 4 requests into HND targets: TMA vs LD/ST (AUTO)
descs = [oc.build_descriptor(store, keys, lay, hnd) for _ in range(4)]
b = oc.Batch(descs)
for eng_name, eng in (("bulk", oc.COPY_BULK), ("auto", oc.COPY_AUTO)):
    for _ in range(3):
        b.fetch(s, engine=eng)
    s.synchronize()
    a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a0.record(s)
    for _ in range(10):
        b.fetch(s, engine=eng)
    a1.record(s)
    s.synchronize()
    ms = a0.elapsed_time(a1) / 10
    print(json.dumps({"target": "hnd", "batch": 4, "engine": eng_name, "us": round(ms * 1e3, 1),
                      "GBps": round(4 * 2 * N * S * L / ms / 1e6, 1)}), flush=True)
b.close()
for d in descs:
    d.close()
