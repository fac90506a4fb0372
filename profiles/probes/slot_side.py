"""Which side makes 5 MiB slots slow: gather into a FLAT target (contiguous destination) vs
scatter_flat (contiguous source, paged destination), L = 32 vs 80, N = 1792."""
import json, sys
sys.path.insert(0, "/root/repo")
import torch
import paper_2605_22850_b200 as oc
import synth
dev = torch.device("cuda", 0)
def timeit(fn, reps=8):
    s = torch.cuda.current_stream()
    for _ in range(3): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
for L in (32, 80, 64, 40):
    N = 1792
    lay_t = (L, 8, 128, 2, 16); G, Bs = 16, 16
    row, S, chunk = oc.geometry(lay_t)
    store = oc.Store(lay_t, capacity=N, device=0)
    (tok,), _ = synth.family_streams(900, G, 0, [N]); keys = oc.chunk_keys(tok, G)
    for b0 in range(0, N, 256):
        store.put_chunks(keys[b0:b0 + 256], torch.randint(0, 256, (min(N, b0 + 256) - b0, chunk), dtype=torch.uint8, device=dev))
    W = N * L * S
    flat = torch.empty(W, dtype=torch.uint8, device=dev)
    df = oc.build_descriptor(store, keys, lay_t, oc.FlatTarget(flat.data_ptr(), W))
    need = N * G // Bs; pool = need + need // 4
    cache = torch.empty((L, 2, pool, Bs, row), dtype=torch.uint8, device=dev); per_kv = pool * Bs * row
    kb = [cache.data_ptr() + l * 2 * per_kv for l in range(L)]
    dp = oc.build_descriptor(store, keys, lay_t, oc.PagedTarget(kb, [x + per_kv for x in kb], Bs * row, row, 256, Bs, synth.block_table(5, need, pool), 0))
    s = torch.cuda.current_stream()
    ms_gather_flat = timeit(lambda: df.fetch_layerwise(s, engine=oc.COPY_BULK))
    ms_paged = timeit(lambda: dp.fetch_layerwise(s, engine=oc.COPY_BULK))
    ms_scatter = timeit(lambda: dp.scatter_flat(flat.data_ptr(), W, s))
    f = lambda ms: round(2 * W / ms / 1e9, 3)
    print(json.dumps({"L": L, "gather_to_flat_TBps": f(ms_gather_flat), "gather_to_paged_TBps": f(ms_paged), "scatter_flat_to_paged_TBps": f(ms_scatter)}), flush=True)
    df.close(); dp.close(); store.close(); del flat, cache; torch.cuda.empty_cache()
