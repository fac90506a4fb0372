"""Where does a yield fetch (64K hit) run, and which prefill kernels does it slow?  Per-op CUDA events
on the consumer stream for layers 0-2, with and without the fetch, plus the fetch's layer-ready stamps."""
import json, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
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
ctx = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
variant = sys.argv[2] if len(sys.argv) > 2 else "yield_prio"
cached = ctx * 7 // 8; m = ctx - cached; N = cached // G
x = torch.randn(m, 4096, dtype=torch.bfloat16, device=dev)
need = N * G // Bs
cache = torch.zeros((L, 2, need, Bs, row), dtype=torch.uint8, device=dev)
kvb = cache.view(torch.bfloat16).view(L, 2, need * Bs, n_kv, d_h)
per_kv = need * Bs * row
kb = [cache.data_ptr() + l * 2 * per_kv for l in range(L)]
tgt = oc.PagedTarget(kb, [x_ + per_kv for x_ in kb], Bs * row, row, d_h * lay_t[3], Bs, synth.block_table(7, need, need), 0)
lo_s, hi_s = torch.cuda.Stream(device=dev, priority=0), torch.cuda.Stream(device=dev, priority=-1)
OPS = ["qkv", "attn_hit", "attn_new", "add", "o", "gate_up", "down"]
def layer_compute(l, rec):
    qkv = torch.matmul(x, w[0]); rec()
    q = qkv[:, :4096].view(1, m, 32, d_h); kn = qkv[:, 4096:5120].view(1, m, n_kv, d_h); vn = qkv[:, 5120:].view(1, m, n_kv, d_h)
    a_hit = flash_attn_func(q, kvb[l, 0].unsqueeze(0), kvb[l, 1].unsqueeze(0), causal=False); rec()
    a_new = flash_attn_func(q, kn, vn, causal=True); rec()
    a = a_hit + a_new; rec()
    torch.matmul(a.view(m, 4096), w[1]); rec()
    gu = torch.matmul(x, w[2]); rec()
    torch.matmul(gu[:, :14336], w[3]); rec()
store = oc.Store(lay_t, capacity=N, tier=oc.TIER_HBM, device=0)
(tok,), _ = synth.family_streams(9100 + N, G, 0, [N])
keys = oc.chunk_keys(tok, G)
for b0 in range(0, N, 512):
    pl = torch.randint(0, 256, (min(N, b0 + 512) - b0, chunk), dtype=torch.uint8, device=dev)
    store.put_chunks(keys[b0:b0 + pl.shape[0]], pl); del pl
d = oc.build_descriptor(store, keys, lay_t, tgt)
FO = {"yield_prio": {"engine": oc.COPY_BULK, "yield_sms": True}, "full_gpu": {"engine": oc.COPY_BULK},
      "yield_prio_u8k": {"engine": oc.COPY_BULK, "yield_sms": True, "unit_bytes": 8192}}[variant]
NL = 3
def chain(fetch):
    torch.cuda.synchronize()
    a0 = torch.cuda.Event(enable_timing=True); evs = []
    def rec():
        e = torch.cuda.Event(enable_timing=True); e.record(hi_s); evs.append(e)
    a0.record(lo_s); hi_s.wait_event(a0)
    if fetch: d.fetch_layerwise(lo_s, **FO)
    with torch.cuda.stream(hi_s):
        for l in range(NL):
            if fetch: d.wait_layer(l, hi_s)
            layer_compute(l, rec)
    torch.cuda.synchronize()
    t = np.array([a0.elapsed_time(e) for e in evs]).reshape(NL, len(OPS))
    return t
chain(False); chain(True)
base = np.median([chain(False) for _ in range(3)], axis=0)
runs = []
for _ in range(3):
    t = chain(True)
    lt = d.layer_times().astype(np.int64)
    runs.append((t, (lt[1:] - lt[0]) / 1e6))
t = np.median([r[0] for r in runs], axis=0)
ready = np.median([r[1] for r in runs], axis=0)
def durs(tt):
    flat = tt.reshape(-1); prev = np.concatenate([[0.0], flat[:-1]]); return (flat - prev).reshape(tt.shape)
db, df = durs(base), durs(t)
out = {"ctx": ctx, "variant": variant, "ops": OPS,
       "base_end_ms": np.round(base, 3).tolist(), "fetch_end_ms": np.round(t, 3).tolist(),
       "op_slowdown_ms": np.round(df - db, 4).tolist(),
       "ready_ms": np.round(ready, 3).tolist()}
print(json.dumps(out), flush=True)
