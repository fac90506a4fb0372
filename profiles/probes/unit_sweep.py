"""4K and 64K fetch GB/s vs unit size and TMA CTAs per SM (OC_BULK_CTAS_PER_SM), HBM store."""
import json, os, subprocess, sys
code = r'''
import json, sys, torch
sys.path.insert(0, ".")
import paper_2605_22850_b200 as oc, synth
lay = synth.LLAMA3_8B.as_tuple(); L, G, Bs = lay[0], lay[4], 16
row, S, chunk = oc.geometry(lay)
res = {}
for N in (256, 4096):
    store = oc.Store(lay, capacity=N)
    (tok,), _ = synth.family_streams(5, G, 0, [N]); keys = oc.chunk_keys(tok, G)
    for b0 in range(0, N, 512):
        store.put_chunks(keys[b0:b0+512], torch.randint(0, 256, (min(512, N-b0), chunk), dtype=torch.uint8, device="cuda"))
    need = N * G // Bs
    cache = torch.empty((L, 2, need, Bs, row), dtype=torch.uint8, device="cuda"); per_kv = need * Bs * row
    kb = [cache.data_ptr() + l * 2 * per_kv for l in range(L)]
    d = oc.build_descriptor(store, keys, lay, oc.PagedTarget(kb, [x + per_kv for x in kb], Bs*row, row, lay[2]*lay[3], Bs, synth.block_table(2, need, need), 0))
    s = torch.cuda.Stream()
    for ub in (16384, 32768, 65536):
        for _ in range(3): d.fetch_layerwise(s, engine=oc.COPY_BULK, unit_bytes=ub)
        s.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 20 if N == 256 else 4
        a.record(s)
        for _ in range(reps): d.fetch_layerwise(s, engine=oc.COPY_BULK, unit_bytes=ub)
        b.record(s); s.synchronize()
        res[f"N{N}_u{ub//1024}K"] = round(2 * N * S * L * reps / a.elapsed_time(b) / 1e6, 1)
    d.close(); store.close(); del cache; torch.cuda.empty_cache()
print(json.dumps(res))
'''
for per_sm in (2, 3, 4):
    env = dict(os.environ, OC_BULK_CTAS_PER_SM=str(per_sm))
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True).stdout.strip().splitlines()
    print(json.dumps({"ctas_per_sm": per_sm, "GBps": json.loads(out[-1]) if out else None}), flush=True)
