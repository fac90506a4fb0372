"""Where the 4K fetch's first-layer latency (X0) goes: per-CTA ramp stamps (OC_TRACE=1,
oc_trace_read) of the bulk kernel on the bench workload (Llama-3-8B, 4K hit, N=256 and the stall
leg's N=224, fragmented NHD Bs=16), relative to the observer CTA's start t[0].  Also per-layer
ready times and the back-to-back launch time.  Usage: OC_TRACE=1 python profiles/probes/ramp_trace.py"""
import json, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2605_22850_b200 as oc, synth

lay = synth.LLAMA3_8B.as_tuple()
L, G, Bs = lay[0], lay[4], 16
row, S, chunk = oc.geometry(lay)
names = ["cta_start", "first_layer_retired", "claim1", "load1_issued", "unit1_in_smem", "stores1_issued",
         "first_layer_released", "signal1_published"]
out = {}
for N in (256, 224):
    store = oc.Store(lay, capacity=4 * N)
    descs, caches = [], []
    for r in range(4):
        (tok,), _ = synth.family_streams(50 + r, G, 0, [N])
        keys = oc.chunk_keys(tok, G)
        store.put_chunks(keys, torch.randint(0, 256, (N, chunk), dtype=torch.uint8, device="cuda"))
        need = N * G // Bs
        pool = need + need // 4
        cache = torch.empty((L, 2, pool, Bs, row), dtype=torch.uint8, device="cuda")
        per_kv = pool * Bs * row
        kb = [cache.data_ptr() + l * 2 * per_kv for l in range(L)]
        descs.append(oc.build_descriptor(store, keys, lay, oc.PagedTarget(
            kb, [x + per_kv for x in kb], Bs * row, row, lay[2] * lay[3], Bs, synth.block_table(7 + r, need, pool), 0)))
        caches.append(cache)
    s = torch.cuda.Stream()
    for i in range(12):
        descs[i % 4].fetch_layerwise(s)
    s.synchronize()
    rows = []
    x0 = []
    for i in range(8):
        d = descs[i % 4]
        torch.cuda.synchronize()
        d.fetch_layerwise(s)
        s.synchronize()
        t = d.layer_times().astype(np.int64)
        tr = oc.trace_read().astype(np.int64) if os.environ.get("OC_TRACE") == "1" else np.zeros((2048, 8), np.int64)
        live = tr[1:][tr[1:, 0] > 0]
        rel = np.where(live > 0, live - t[0], -1)
        rows.append(rel)
        x0.append(t[1] - t[0])
        ready = (t[1:] - t[0]) / 1e3
    rel = np.concatenate(rows)
    res = {"ctas": int(rows[0].shape[0]), "X0_us_median": float(np.median(x0)) / 1e3,
           "ready_us_last_run": [round(float(v), 2) for v in ready[:6]] + ["..."] + [round(float(ready[-1]), 2)]}
    for k, nm in enumerate(names):
        v = rel[:, k][rel[:, k] >= 0] / 1e3
        if v.size:
            res[nm] = {q: round(float(np.percentile(v, p)), 2) for q, p in (("p0", 0), ("p50", 50), ("p90", 90), ("p100", 100))}
    # back-to-back launch time (no trace influence on the mean is expected; stamps are a few stores)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for i in range(20):
        descs[i % 4].fetch_layerwise(s)
    b.record(s)
    s.synchronize()
    res["b2b_us_per_fetch"] = round(a.elapsed_time(b) * 1e3 / 20, 2)
    res["b2b_TBps"] = round(2 * N * S * L * 20 / (a.elapsed_time(b) / 1e3) / 1e12, 3)
    for _ in range(2):   # OC_FETCH_OVERLAP: each launch overlaps the previous one's tail
        a.record(s)
        for i in range(40):
            descs[i % 4].fetch_layerwise(s, overlap=True)
        b.record(s)
        s.synchronize()
    res["b2b_overlap_us_per_fetch"] = round(a.elapsed_time(b) * 1e3 / 40, 2)
    res["b2b_overlap_TBps"] = round(2 * N * S * L * 40 / (a.elapsed_time(b) / 1e3) / 1e12, 3)
    out[f"N{N}"] = res
    for d in descs:
        d.close()
    store.close()
    del caches
    torch.cuda.empty_cache()
print(json.dumps(out, indent=1))
