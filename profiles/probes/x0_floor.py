"""Floor for X0: a plain contiguous device copy of one 4K layer's bytes (16 MiB read + 16 MiB written),
timed alone with CUDA events, vs the fetch's X0 (layer 0 announced after the kernel's start)."""
import json, statistics, torch
dev = torch.device("cuda", 0)
res = {}
for mib in (8, 16, 32):
    n = mib << 20
    a = torch.empty(n, dtype=torch.uint8, device=dev).fill_(1); b = torch.empty_like(a)
    big = torch.empty(1 << 30, dtype=torch.uint8, device=dev)
    ts = []
    for i in range(60):
        big.fill_(i & 255)                       # flush L2 between runs
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); b.copy_(a); e1.record(); torch.cuda.synchronize()
        if i >= 10: ts.append(e0.elapsed_time(e1) * 1e3)
    res[f"copy_{mib}MiB_us"] = {"median": round(statistics.median(ts), 2), "min": round(min(ts), 2)}
    del a, b, big
print(json.dumps(res))
