"""70B-layout fetch rate (L = 80, N = 1792, fragmented NHD paged cache, 2 rotating requests back to
back with OC_FETCH_OVERLAP) against the HBM slot pitch (OC_SLOT_PITCH_KIB override; 0 = the
library's oc_slot_pitch rule), plus the 8B 64K shape at its default pitch for comparison."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2605_22850_b200 as oc
import synth
from benchlib import verify
dev = torch.device("cuda", 0)


def rate(lay_t, N, pitch_kib):
    if pitch_kib:
        os.environ["OC_SLOT_PITCH_KIB"] = str(pitch_kib)
    else:
        os.environ.pop("OC_SLOT_PITCH_KIB", None)
    L, G, Bs = lay_t[0], lay_t[4], 16
    row, S, chunk = oc.geometry(lay_t)
    store = oc.Store(lay_t, capacity=2 * N, device=0)
    pitch = store.slab[1] // (2 * N)
    sets = []
    for r in range(2):
        seed = 777 + r
        (tok,), (ids,) = synth.family_streams(seed, G, 0, [N])
        keys = oc.chunk_keys(tok, G)
        verify.fill_store([store], keys, seed, ids, chunk)
        need = N * G // Bs
        pool = need + need // 4
        bt = synth.block_table(50 + r, need, pool)
        cache = torch.empty((L, 2, pool, Bs, row), dtype=torch.uint8, device=dev)
        per_kv = pool * Bs * row
        kb = [cache.data_ptr() + l * 2 * per_kv for l in range(L)]
        tgt = oc.PagedTarget(kb, [x + per_kv for x in kb], Bs * row, row, lay_t[2] * lay_t[3], Bs, bt, 0)
        sets.append((oc.build_descriptor(store, keys, lay_t, tgt), cache))
    s = torch.cuda.Stream()
    for i in range(4):
        sets[i % 2][0].fetch_layerwise(s, overlap=True)
    s.synchronize()
    reps = 8
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for i in range(reps):
        sets[i % 2][0].fetch_layerwise(s, overlap=True)
    b.record(s)
    s.synchronize()
    ms = a.elapsed_time(b) / reps
    for d, _ in sets:
        d.close()
    store.close()
    del sets
    torch.cuda.empty_cache()
    return {"L": L, "N": N, "chunk_KiB": chunk >> 10, "pitch_KiB": pitch >> 10, "granules": pitch // 32768,
            "ms": round(ms, 3), "TBps_rw": round(2 * N * S * L / ms / 1e9, 3)}


if len(sys.argv) > 1:   # L and granule counts: pitch_sweep.py L g1 g2 ...
    L = int(sys.argv[1])
    N = 1792 if L * 64 <= 5120 * 2 else 1024
    for g in sys.argv[2:]:
        print(json.dumps(rate((L, 8, 128, 2, 16), N, int(g) * 32)), flush=True)
else:
    for p in (5120, 0, 5184, 5216, 5248, 5280, 5376, 5632, 6144, 8192, 5120, 0):
        print(json.dumps(rate((80, 8, 128, 2, 16), 1792, p)), flush=True)
    print(json.dumps(rate(synth.LLAMA3_8B.as_tuple(), 4096, 0)), flush=True)
    print(json.dumps(rate((64, 8, 128, 2, 16), 1792, 0)), flush=True)
