"""Probe: do two or four copy streams (each a share of every layer's strided transfer) beat one?"""
import json
import torch
from cuda.bindings import runtime as rt

L, S = 32, 65536
chunk = L * S
N = 256
slab = torch.empty(N * chunk, dtype=torch.uint8).pin_memory()
stage = torch.empty(N * S * 2, dtype=torch.uint8, device="cuda")
H2D = rt.cudaMemcpyKind.cudaMemcpyHostToDevice
for nstreams in (1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(nstreams)]
    def run(layers):
        per = N // nstreams
        for l in range(layers):
            for k, s in enumerate(streams):
                c0 = k * per
                src = slab.data_ptr() + c0 * chunk + l * S
                dst = stage.data_ptr() + (l % 2) * N * S + c0 * S
                err, = rt.cudaMemcpy2DAsync(dst, S, src, chunk, S, per, H2D, s.cuda_stream)
                assert err == rt.cudaError_t.cudaSuccess
    run(2); torch.cuda.synchronize()
    best = 1e9
    for rep in range(3):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(streams[0])
        for s in streams[1:]:
            s.wait_event(e0)
        run(L)
        for s in streams[1:]:
            streams[0].wait_stream(s)
        e1.record(streams[0])
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print(json.dumps({"probe": "ce_2d_streams", "streams": nstreams, "GBps": round(N * S * L / best / 1e6, 1)}), flush=True)
