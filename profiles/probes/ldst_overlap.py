"""Back-to-back 4K fetches (4 rotating requests, own caches) into NHD and HND paged targets, TMA and
LD/ST engines, stream order vs OC_FETCH_OVERLAP."""
import json, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2605_22850_b200 as oc
import synth
lay = synth.LLAMA3_8B.as_tuple()
L, G, Bs = lay[0], lay[4], 16
row, S, chunk = oc.geometry(lay)
hd = lay[2] * lay[3]
N = 256
store = oc.Store(lay, capacity=4 * N)
sets = []
for r in range(4):
    (tok,), _ = synth.family_streams(40 + r, G, 0, [N]); keys = oc.chunk_keys(tok, G)
    store.put_chunks(keys, torch.randint(0, 256, (N, chunk), dtype=torch.uint8, device="cuda"))
    need = N * G // Bs; pool = need + need // 4
    bt = synth.block_table(7 + r, need, pool)
    cache = torch.empty(L * 2 * pool * Bs * row, dtype=torch.uint8, device="cuda"); base = cache.data_ptr()
    per_kv = pool * Bs * row
    nhd = oc.PagedTarget([base + l * 2 * per_kv for l in range(L)], [base + l * 2 * per_kv + per_kv for l in range(L)],
                         Bs * row, row, hd, Bs, bt, 0)
    blk = 2 * lay[1] * Bs * hd
    hnd = oc.PagedTarget([base + l * pool * blk for l in range(L)], [base + l * pool * blk + lay[1] * Bs * hd for l in range(L)],
                         blk, hd, Bs * hd, Bs, bt, 0)
    sets.append((keys, nhd, hnd, cache))
s = torch.cuda.Stream()
for kind in ("nhd", "hnd"):
    descs = [oc.build_descriptor(store, k, lay, n if kind == "nhd" else h) for k, n, h, _ in sets]
    for eng_name, eng in (("bulk", oc.COPY_BULK), ("ldst", oc.COPY_LDST)):
        for ov in (False, True):
            for i in range(12):
                descs[i % 4].fetch_layerwise(s, engine=eng, overlap=ov)
            s.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            for i in range(100):
                descs[i % 4].fetch_layerwise(s, engine=eng, overlap=ov)
            b.record(s); s.synchronize()
            ms = a.elapsed_time(b) / 100
            print(json.dumps({"target": kind, "engine": eng_name, "overlap": ov, "us": round(ms * 1e3, 1),
                              "TBps": round(2 * N * S * L / ms / 1e9, 3)}), flush=True)
    for d in descs:
        d.close()
