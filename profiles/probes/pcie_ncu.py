"""A 4K-token hit from the pinned-host store, fetched by the SM zero-copy kernel (for ncu PCIe counters)."""
import sys
sys.path.insert(0, ".")
import torch
import paper_2605_22850_b200 as oc
import synth
lay = synth.LLAMA3_8B.as_tuple()
L, G, Bs = lay[0], lay[4], 16
row, S, chunk = oc.geometry(lay)
N = 256
store = oc.Store(lay, capacity=N, tier=oc.TIER_PINNED_HOST)
(tok,), _ = synth.family_streams(3, G, 0, [N])
keys = oc.chunk_keys(tok, G)
store.put_chunks(keys, torch.randint(0, 256, (N, chunk), dtype=torch.uint8, device="cuda"))
need = N * G // Bs
cache = torch.empty((L, 2, need, Bs, row), dtype=torch.uint8, device="cuda")
per_kv = need * Bs * row
kb = [cache.data_ptr() + l * 2 * per_kv for l in range(L)]
tgt = oc.PagedTarget(kb, [x + per_kv for x in kb], Bs * row, row, lay[2] * lay[3], Bs, synth.block_table(1, need, need), 0)
d = oc.build_descriptor(store, keys, lay, tgt)
s = torch.cuda.Stream()
for _ in range(4):
    d.fetch_layerwise(s, engine=oc.COPY_BULK)
s.synchronize()
print("bytes per fetch read from host:", N * S * L)
