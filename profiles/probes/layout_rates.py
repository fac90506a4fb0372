"""Fetch rate across the BASELINE layouts and hit sizes, HBM store into a fragmented NHD paged cache
(Bs = 16): Llama-3-8B 4K / 64K and Llama-3-70B 32K at 87.5% hit (N = 1792, L = 80), 2 rotating
requests back to back with OC_FETCH_OVERLAP; first request verified in full against the oracle."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
import paper_2605_22850_b200 as oc
import synth
from benchlib import verify
from oracle.geometry import Layout
dev = torch.device("cuda", 0)
out = {}
for name, lay_t, N in (("llama3-8b_4k", synth.LLAMA3_8B.as_tuple(), 256), ("llama3-8b_64k", synth.LLAMA3_8B.as_tuple(), 4096),
                       ("llama3-70b_32k_87.5", (80, 8, 128, 2, 16), 1792)):
    L, G, Bs = lay_t[0], lay_t[4], 16
    row, S, chunk = oc.geometry(lay_t)
    store = oc.Store(lay_t, capacity=2 * N, device=0)
    sets = []
    for r in range(2):
        seed = 777 + r
        (tok,), (ids,) = synth.family_streams(seed, G, 0, [N])
        keys = oc.chunk_keys(tok, G)
        verify.fill_store([store], keys, seed, ids, chunk)
        need = N * G // Bs; pool = need + need // 4
        bt = synth.block_table(50 + r, need, pool)
        cache = torch.empty((L, 2, pool, Bs, row), dtype=torch.uint8, device=dev)
        per_kv = pool * Bs * row
        kb = [cache.data_ptr() + l * 2 * per_kv for l in range(L)]
        tgt = oc.PagedTarget(kb, [x + per_kv for x in kb], Bs * row, row, lay_t[2] * lay_t[3], Bs, bt, 0)
        sets.append((oc.build_descriptor(store, keys, lay_t, tgt), cache, seed, keys, ids, bt))
    s = torch.cuda.Stream()
    for i in range(4):
        sets[i % 2][0].fetch_layerwise(s, overlap=True)
    s.synchronize()
    reps = max(4, int(20 * 256 / N))
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for i in range(reps):
        sets[i % 2][0].fetch_layerwise(s, overlap=True)
    b.record(s); s.synchronize()
    ms = a.elapsed_time(b) / reps
    d0, cache0, seed0, keys0, ids0, bt0 = sets[0]
    d0.fetch_layerwise(s); s.synchronize()
    t = d0.layer_times().astype(np.int64)
    idx = verify.slot_index(torch, dev, bt0, N * G, Bs)
    layers = range(L) if N * L <= 256 * 32 else (0, L // 2, L - 1)
    ok, nbytes, t_or, _ = verify.full_check(torch, Layout(*lay_t), seed0, keys0, ids0, cache0, idx, layers)
    out[name] = {"L": L, "N": N, "GiB_per_fetch_rw": round(2 * N * S * L / 2**30, 2), "ms": round(ms, 3),
                 "TBps_rw": round(2 * N * S * L / ms / 1e9, 3), "X0_us": round((t[1] - t[0]) / 1e3, 1),
                 "verified_layers": len(layers), "bit_exact": ok}
    print(json.dumps({name: out[name]}), flush=True)
    for st_ in sets:
        st_[0].close()
    store.close(); del sets; torch.cuda.empty_cache()
