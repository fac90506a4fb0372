"""PER_LAYER mode (one launch + one CUDA event per layer, successive layers' launches programmatic
dependents of each other): back-to-back 4K fetch rate vs the per-layer copy-CTA count, and the
persistent kernel for reference."""
import json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2605_22850_b200 as oc, synth
lay = synth.LLAMA3_8B.as_tuple(); L, G, Bs = lay[0], lay[4], 16
row, S, chunk = oc.geometry(lay)
N = 256
store = oc.Store(lay, capacity=4 * N)
descs, caches = [], []
for r in range(4):
    (tok,), _ = synth.family_streams(50 + r, G, 0, [N]); keys = oc.chunk_keys(tok, G)
    store.put_chunks(keys, torch.randint(0, 256, (N, chunk), dtype=torch.uint8, device="cuda"))
    need = N * G // Bs; pool = need + need // 4
    cache = torch.empty((L, 2, pool, Bs, row), dtype=torch.uint8, device="cuda"); per_kv = pool * Bs * row
    kb = [cache.data_ptr() + l * 2 * per_kv for l in range(L)]
    descs.append(oc.build_descriptor(store, keys, lay, oc.PagedTarget(kb, [x + per_kv for x in kb], Bs * row, row, lay[2] * lay[3], Bs, synth.block_table(7 + r, need, pool), 0)))
    caches.append(cache)
s = torch.cuda.Stream()
res = {}
for name, opts in [("persistent", {}), ("per_layer", {"mode": oc.FETCH_PER_LAYER})] + \
        [(f"per_layer_ctas{c}", {"mode": oc.FETCH_PER_LAYER, "max_ctas": c}) for c in (296, 222, 148)] + \
        [(f"per_layer_ctas{c}_u32k", {"mode": oc.FETCH_PER_LAYER, "max_ctas": c, "unit_bytes": 32768}) for c in (148, 111)]:
    for i in range(12):
        descs[i % 4].fetch_layerwise(s, overlap=True, **opts)
    s.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for i in range(40):
        descs[i % 4].fetch_layerwise(s, overlap=True, **opts)
    b.record(s); s.synchronize()
    res[name] = round(2 * N * S * L * 40 / (a.elapsed_time(b) / 1e3) / 1e12, 3)
print(json.dumps(res))
