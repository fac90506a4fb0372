"""Probe: copy-engine H2D of layer slices with a 2D strided copy (width = S, pitch = chunk bytes)
from a pinned slab into a contiguous HBM staging buffer, vs the SM zero-copy fetch kernel."""
import json, time
import torch
from cuda.bindings import runtime as rt

L, S = 32, 65536
chunk = L * S
N = 256
slab = torch.empty(N * chunk, dtype=torch.uint8).pin_memory()
slab.random_(0, 256) if False else None
stage = torch.empty(N * S * 2, dtype=torch.uint8, device="cuda")
s = torch.cuda.Stream()
H2D = rt.cudaMemcpyKind.cudaMemcpyHostToDevice
def run(layers, width_chunks=N):
    for l in range(layers):
        for c0 in range(0, N, width_chunks):
            h = min(width_chunks, N - c0)
            src = slab.data_ptr() + c0 * chunk + l * S
            dst = stage.data_ptr() + (l % 2) * N * S + c0 * S
            err, = rt.cudaMemcpy2DAsync(dst, S, src, chunk, S, h, H2D, s.cuda_stream)
            assert err == rt.cudaError_t.cudaSuccess, err
for w in (N, 64, 16, 4, 1):
    run(2, w); s.synchronize()
    best = None
    for rep in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t = time.perf_counter()
        e0.record(s)
        run(L, w)
        e1.record(s)
        host = time.perf_counter() - t
        s.synchronize()
        ms = e0.elapsed_time(e1)
        best = min(best or 1e9, ms)
    print(json.dumps({"probe": "ce_2d", "runs_per_layer": -(-N // w), "GBps": round(N * S * L / best / 1e6, 1),
                      "ms": round(best, 3), "host_submit_ms": round(host * 1e3, 3)}), flush=True)
# contiguous reference
big = torch.empty(N * S * L, dtype=torch.uint8).pin_memory()
dst = torch.empty(N * S * L, dtype=torch.uint8, device="cuda")
for _ in range(2):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    with torch.cuda.stream(s):
        dst.copy_(big, non_blocking=True)
    e1.record(s); s.synchronize()
print(json.dumps({"probe": "ce_contiguous", "GBps": round(N * S * L / e0.elapsed_time(e1) / 1e6, 1)}))
