"""Cost of the consumer's per-layer waits when they are enqueued before the layer is announced but
satisfied by the time the GPU reaches them: fetch behind a 1 ms spin on the copy stream; the consumer
waits (a) once on layer L-1, (b) on every layer, value waits; (c)/(d) the same with PER_LAYER events."""
import json, statistics, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2605_22850_b200 as oc
import synth
from flash_attn import flash_attn_func
dev = torch.device("cuda", 0); torch.cuda.set_device(0)
lay_t = synth.LLAMA3_8B.as_tuple()
L, G, Bs = lay_t[0], lay_t[4], 16
n_kv, d_h = lay_t[1], lay_t[2]
row, S, chunk = oc.geometry(lay_t)
w = [torch.randn(k, n, dtype=torch.bfloat16, device=dev) * 0.01 for k, n in ((4096, 6144), (4096, 4096), (4096, 28672), (14336, 4096))]
ctx = 4096; cached = ctx * 7 // 8; m = ctx - cached; N = cached // G
x = torch.randn(m, 4096, dtype=torch.bfloat16, device=dev)
need = N * G // Bs
cache = torch.zeros((L, 2, need, Bs, row), dtype=torch.uint8, device=dev)
kvb = cache.view(torch.bfloat16).view(L, 2, need * Bs, n_kv, d_h)
per_kv = need * Bs * row
kb = [cache.data_ptr() + l * 2 * per_kv for l in range(L)]
tgt = oc.PagedTarget(kb, [x_ + per_kv for x_ in kb], Bs * row, row, d_h * lay_t[3], Bs, synth.block_table(7, need, need), 0)
copy_s, cons_s = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
def layer_compute(l):
    qkv = torch.matmul(x, w[0])
    q = qkv[:, :4096].view(1, m, 32, d_h); kn = qkv[:, 4096:5120].view(1, m, n_kv, d_h); vn = qkv[:, 5120:].view(1, m, n_kv, d_h)
    a_hit = flash_attn_func(q, kvb[l, 0].unsqueeze(0), kvb[l, 1].unsqueeze(0), causal=False)
    a_new = flash_attn_func(q, kn, vn, causal=True)
    torch.matmul((a_hit + a_new).view(m, 4096), w[1])
    gu = torch.matmul(x, w[2])
    torch.matmul(gu[:, :14336], w[3])
store = oc.Store(lay_t, capacity=N, tier=oc.TIER_HBM, device=0)
(tok,), _ = synth.family_streams(9100 + N, G, 0, [N])
keys = oc.chunk_keys(tok, G)
store.put_chunks(keys, torch.randint(0, 256, (N, chunk), dtype=torch.uint8, device=dev))
d = oc.build_descriptor(store, keys, lay_t, tgt)
def chain(mode, all_waits, spin_ns=1_000_000):
    torch.cuda.synchronize()
    a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a0.record(copy_s); cons_s.wait_event(a0)
    oc.emulate_compute(spin_ns, copy_s)
    d.fetch_layerwise(copy_s, mode=mode)
    with torch.cuda.stream(cons_s):
        if not all_waits:
            d.wait_layer(L - 1, cons_s)
        for l in range(L):
            if all_waits:
                d.wait_layer(l, cons_s)
            layer_compute(l)
    a1.record(cons_s); torch.cuda.synchronize()
    return a0.elapsed_time(a1)
res = {}
for name, mode in (("value", oc.FETCH_PERSISTENT), ("events", oc.FETCH_PER_LAYER)):
    chain(mode, True); chain(mode, False)
    diffs = []
    for _ in range(9):
        one = chain(mode, False); allw = chain(mode, True)
        diffs.append(allw - one)
    diffs.sort()
    res[name] = {"extra_ms_for_31_waits_median": round(statistics.median(diffs), 4), "min": round(diffs[0], 4), "max": round(diffs[-1], 4),
                 "us_per_wait": round(statistics.median(diffs) * 1e3 / 31, 2)}
print(json.dumps(res), flush=True)
