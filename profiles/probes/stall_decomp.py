"""Decompose the added TTFT of the stall_gemm leg: the consumer's per-layer waits themselves (on a
descriptor whose layers are all announced already) vs no waits; then fetch variants."""
import json, statistics, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2605_22850_b200 as oc
import synth
from flash_attn import flash_attn_func
dev = torch.device("cuda", 0)
torch.cuda.set_device(0)
lay_t = synth.LLAMA3_8B.as_tuple()
L, G, Bs = lay_t[0], lay_t[4], 16
n_kv, d_h = lay_t[1], lay_t[2]
row, S, chunk = oc.geometry(lay_t)
w = [torch.randn(k, n, dtype=torch.bfloat16, device=dev) * 0.01 for k, n in ((4096, 6144), (4096, 4096), (4096, 28672), (14336, 4096))]
ctxs = [int(c) for c in (sys.argv[1] if len(sys.argv) > 1 else "4096,65536").split(",")]
for ctx in ctxs:
    cached = ctx * 7 // 8; m = ctx - cached; N = cached // G
    x = torch.randn(m, 4096, dtype=torch.bfloat16, device=dev)
    need = N * G // Bs
    cache = torch.zeros((L, 2, need, Bs, row), dtype=torch.uint8, device=dev)
    kvb = cache.view(torch.bfloat16).view(L, 2, need * Bs, n_kv, d_h)
    per_kv = need * Bs * row
    kb = [cache.data_ptr() + l * 2 * per_kv for l in range(L)]
    tgt = oc.PagedTarget(kb, [x_ + per_kv for x_ in kb], Bs * row, row, d_h * lay_t[3], Bs, synth.block_table(7, need, need), 0)
    copy_s, cons_s = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
    lo_s, hi_s = torch.cuda.Stream(device=dev, priority=0), torch.cuda.Stream(device=dev, priority=-1)
    def layer_compute(l):
        qkv = torch.matmul(x, w[0])
        q = qkv[:, :4096].view(1, m, 32, d_h); kn = qkv[:, 4096:5120].view(1, m, n_kv, d_h); vn = qkv[:, 5120:].view(1, m, n_kv, d_h)
        a_hit = flash_attn_func(q, kvb[l, 0].unsqueeze(0), kvb[l, 1].unsqueeze(0), causal=False)
        a_new = flash_attn_func(q, kn, vn, causal=True)
        torch.matmul((a_hit + a_new).view(m, 4096), w[1])
        gu = torch.matmul(x, w[2])
        torch.matmul(gu[:, :14336], w[3])
    def chain(d, fopts, waits, cs=None, ks=None):
        cs, ks = cs or copy_s, ks or cons_s
        torch.cuda.synchronize()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(cs); ks.wait_event(a0)
        if fopts is not None:
            d.fetch_layerwise(cs, **fopts)
        with torch.cuda.stream(ks):
            for l in range(L):
                if waits:
                    d.wait_layer(l, ks)
                layer_compute(l)
        a1.record(ks); torch.cuda.synchronize()
        return a0.elapsed_time(a1)
    store = oc.Store(lay_t, capacity=N, tier=oc.TIER_HBM, device=0)
    (tok,), _ = synth.family_streams(9100 + N, G, 0, [N])
    keys = oc.chunk_keys(tok, G)
    for b0 in range(0, N, 512):
        pl = torch.randint(0, 256, (min(N, b0 + 512) - b0, chunk), dtype=torch.uint8, device=dev)
        store.put_chunks(keys[b0:b0 + pl.shape[0]], pl); del pl
    d = oc.build_descriptor(store, keys, lay_t, tgt)
    d.fetch_layerwise(copy_s); torch.cuda.synchronize()
    chain(None, None, False)
    res = {"ctx": ctx}
    def paired(fn, n=7):
        r = []
        for _ in range(n):
            b = chain(None, None, False)
            r.append(fn() - b)
        r.sort(); r = r[1:-1]
        return {"mean": round(statistics.mean(r), 4), "min": round(r[0], 4), "max": round(r[-1], 4)}
    res["base_ms"] = round(chain(None, None, False), 3)
    res["waits_ready_value"] = paired(lambda: chain(d, None, True))           # all layers announced already
    d.fetch_layerwise(copy_s, mode=oc.FETCH_PER_LAYER); torch.cuda.synchronize()
    res["waits_ready_events"] = paired(lambda: chain(d, None, True))
    for name, fo, streams in (("full_gpu", {"engine": oc.COPY_BULK}, None),
                              ("per_layer", {"mode": oc.FETCH_PER_LAYER}, None),
                              ("yield_prio", {"engine": oc.COPY_BULK, "yield_sms": True}, (lo_s, hi_s)),
                              ("ctas16", {"engine": oc.COPY_BULK, "max_ctas": 16}, None)):
        cs, ks = streams if streams else (None, None)
        chain(d, fo, True, cs, ks)
        res[name] = paired(lambda: chain(d, fo, True, cs, ks))
        res[name + "_nowait_baseline_incl"] = None
    print(json.dumps(res), flush=True)
    d.close(); store.close(); del cache, kvb; torch.cuda.empty_cache()
