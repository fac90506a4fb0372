import json, os, sys
sys.path.insert(0, "/root/repo")
import numpy as np
import torch
import paper_2605_22850_b200 as oc
import synth
dev = torch.device("cuda", 0)
for L, N, scramble in ((80, 1792, False), (80, 1792, True), (32, 1792, False), (32, 1792, True), (40, 1792, True), (48, 1792, True)):
    lay_t = (L, 8, 128, 2, 16)
    G, Bs = 16, 16
    row, S, chunk = oc.geometry(lay_t)
    store = oc.Store(lay_t, capacity=2 * N, device=0)
    ds, caches = [], []
    for r in range(2):
        (tok,), _ = synth.family_streams(900 + r, G, 0, [N]); keys = oc.chunk_keys(tok, G)
        order = np.random.default_rng(r).permutation(N) if scramble else np.arange(N)
        for b0 in range(0, N, 256):
            sel = order[b0:b0 + 256]
            store.put_chunks(keys[sel], torch.randint(0, 256, (len(sel), chunk), dtype=torch.uint8, device=dev))
        need = N * G // Bs; pool = need + need // 4
        cache = torch.empty((L, 2, pool, Bs, row), dtype=torch.uint8, device=dev); per_kv = pool * Bs * row
        kb = [cache.data_ptr() + l * 2 * per_kv for l in range(L)]
        ds.append(oc.build_descriptor(store, keys, lay_t, oc.PagedTarget(kb, [x + per_kv for x in kb], Bs * row, row, 256, Bs, synth.block_table(5 + r, need, pool), 0)))
        caches.append(cache)
    s = torch.cuda.Stream()
    for i in range(4): ds[i % 2].fetch_layerwise(s, overlap=True)
    s.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 8
    a.record(s)
    for i in range(reps): ds[i % 2].fetch_layerwise(s, overlap=True)
    b.record(s); s.synchronize()
    ms = a.elapsed_time(b) / reps
    print(json.dumps({"L": L, "N": N, "scrambled_slots": scramble, "ms": round(ms, 3), "TBps": round(2 * N * S * L / ms / 1e9, 3)}), flush=True)
    for d in ds: d.close()
    store.close(); del caches; torch.cuda.empty_cache()
