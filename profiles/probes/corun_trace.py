"""Device timeline (CUPTI kernel activity via torch.profiler; nsys is not in the image) of a prefix
fetch co-running with a shape-true Llama-3-8B prefill: the fetch kernel(s) on the copy stream and
the prefill's kernels on the consumer stream, 4K (default launch) and 64K (OC_FETCH_YIELD, copy
stream low / consumer high priority; first 3 layers).  Writes a compact JSON per case: every
kernel's stream, start and end (us from the fetch launch), and per layer the ready stamp."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
from torch.profiler import profile, ProfilerActivity
import paper_2605_22850_b200 as oc
import synth
from flash_attn import flash_attn_func
dev = torch.device("cuda", 0); torch.cuda.set_device(0)
lay_t = synth.LLAMA3_8B.as_tuple()
L, G, Bs = lay_t[0], lay_t[4], 16
n_kv, d_h = lay_t[1], lay_t[2]
row, S, chunk = oc.geometry(lay_t)
w = [torch.randn(k, n, dtype=torch.bfloat16, device=dev) * 0.01 for k, n in ((4096, 6144), (4096, 4096), (4096, 28672), (14336, 4096))]
out_dir = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out"
for name, ctx, fopts, prio, n_layers in (("4k_default", 4096, {"engine": oc.COPY_BULK}, False, L),
                                         ("64k_yield_prio", 65536, {"engine": oc.COPY_BULK, "yield_sms": True}, True, 3)):
    cached = ctx * 7 // 8; m = ctx - cached; N = cached // G
    x = torch.randn(m, 4096, dtype=torch.bfloat16, device=dev)
    need = N * G // Bs
    cache = torch.zeros((L, 2, need, Bs, row), dtype=torch.uint8, device=dev)
    kvb = cache.view(torch.bfloat16).view(L, 2, need * Bs, n_kv, d_h)
    per_kv = need * Bs * row
    kb = [cache.data_ptr() + l * 2 * per_kv for l in range(L)]
    tgt = oc.PagedTarget(kb, [x_ + per_kv for x_ in kb], Bs * row, row, d_h * lay_t[3], Bs, synth.block_table(7, need, need), 0)
    cs = torch.cuda.Stream(device=dev, priority=0)
    ks = torch.cuda.Stream(device=dev, priority=-1 if prio else 0)
    store = oc.Store(lay_t, capacity=N, tier=oc.TIER_HBM, device=0)
    (tok,), _ = synth.family_streams(9100 + N, G, 0, [N])
    keys = oc.chunk_keys(tok, G)
    for b0 in range(0, N, 512):
        pl = torch.randint(0, 256, (min(N, b0 + 512) - b0, chunk), dtype=torch.uint8, device=dev)
        store.put_chunks(keys[b0:b0 + pl.shape[0]], pl); del pl
    d = oc.build_descriptor(store, keys, lay_t, tgt)

    def chain():
        torch.cuda.synchronize()
        a0 = torch.cuda.Event(); a0.record(cs); ks.wait_event(a0)
        d.fetch_layerwise(cs, **fopts)
        with torch.cuda.stream(ks):
            for l in range(n_layers):
                d.wait_layer(l, ks)
                qkv = torch.matmul(x, w[0])
                q = qkv[:, :4096].view(1, m, 32, d_h); kn = qkv[:, 4096:5120].view(1, m, n_kv, d_h); vn = qkv[:, 5120:].view(1, m, n_kv, d_h)
                a = flash_attn_func(q, kvb[l, 0].unsqueeze(0), kvb[l, 1].unsqueeze(0), causal=False) + flash_attn_func(q, kn, vn, causal=True)
                torch.matmul(a.view(m, 4096), w[1])
                gu = torch.matmul(x, w[2]); torch.matmul(gu[:, :14336], w[3])
        torch.cuda.synchronize()
    chain(); chain()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        chain()
    t = d.layer_times().astype(np.int64)
    evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA and e.device_time_total > 0
           and not e.name.startswith("Memcpy") and not e.name.startswith("Memset")]
    # kernel records: name, start/end in us (profiler clock); t0 = the fetch kernel's first start
    recs = []
    for e in evs:
        recs.append({"name": e.name[:80], "start_us": e.time_range.start, "end_us": e.time_range.end})
    recs.sort(key=lambda r: r["start_us"])
    fetch = [r for r in recs if "fetch_bulk_kernel" in r["name"] or "fetch_ldst_kernel" in r["name"]]
    t0 = fetch[0]["start_us"] if fetch else recs[0]["start_us"]
    for r in recs:
        r["start_us"] = round(r["start_us"] - t0, 1); r["end_us"] = round(r["end_us"] - t0, 1)
        r["role"] = "fetch" if ("fetch_bulk_kernel" in r["name"] or "fetch_ldst_kernel" in r["name"]) else "prefill"
    ready_us = [round((t[1 + l] - t[0]) / 1e3, 1) for l in range(L)]
    out = {"case": name, "ctx": ctx, "layers_of_prefill_traced": n_layers, "fetch_opts": {k: (v if not isinstance(v, bool) else int(v)) for k, v in fopts.items()},
           "priorities": "copy 0 / consumer -1" if prio else "both 0",
           "clock": "CUPTI kernel activity via torch.profiler, us from the fetch kernel's start; ready_us from the kernel's %globaltimer stamps (since its start)",
           "layer_ready_us": ready_us, "kernels": recs}
    with open(os.path.join(out_dir, f"corun_trace_{name}.json"), "w") as f:
        json.dump(out, f)
    print(name, len(recs), "kernels; fetch kernels:", [(r["start_us"], r["end_us"]) for r in recs if r["role"] == "fetch"][:4], flush=True)
    d.close(); store.close(); del cache, kvb; torch.cuda.empty_cache()
