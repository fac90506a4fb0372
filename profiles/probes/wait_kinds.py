"""Device cost of a consumer-stream wait whose condition already holds when the GPU reaches it but
not when the host enqueued it: 32 x (wait + 20 us spin kernel) on the consumer stream, the waits'
producer being a 2 ms spin on another stream that every wait is enqueued behind.  Kinds: none,
cuStreamWaitValue32 (GEQ) on a word the producer stream sets, cudaStreamWaitEvent on events the
producer stream records."""
import json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from cuda.bindings import driver as cu
import paper_2605_22850_b200 as oc
dev = torch.device("cuda", 0); torch.cuda.set_device(0)
word = torch.zeros(4, dtype=torch.int32, device=dev)
prod, cons = torch.cuda.Stream(), torch.cuda.Stream()
L = 32
evs = [torch.cuda.Event() for _ in range(L)]
def chain(kind, epoch):
    torch.cuda.synchronize()
    a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a0.record(prod); cons.wait_event(a0)
    oc.emulate_compute(2_000_000, prod)                      # the "fetch": everything lands after 2 ms
    if kind == "value":
        cu.cuStreamWriteValue32(prod.cuda_stream, word.data_ptr(), epoch, 0)
    elif kind == "event":
        for e in evs:
            e.record(prod)
    oc.emulate_compute(2_100_000, cons)                      # consumer's first window covers the producer
    for l in range(L):
        if kind == "value":
            cu.cuStreamWaitValue32(cons.cuda_stream, word.data_ptr(), epoch, cu.CUstreamWaitValue_flags.CU_STREAM_WAIT_VALUE_GEQ)
        elif kind == "event":
            cons.wait_event(evs[l])
        oc.emulate_compute(20_000, cons)
    a1.record(cons); torch.cuda.synchronize()
    return a0.elapsed_time(a1)
res, ep = {}, 1
for kind in ("none", "value", "event"):
    chain(kind, ep); ep += 1
for rep in range(9):
    for kind in ("none", "value", "event"):
        res.setdefault(kind, []).append(chain(kind, ep)); ep += 1
base = statistics.median(res["none"])
print(json.dumps({k: {"median_ms": round(statistics.median(v), 4), "us_per_wait_over_none":
                      round((statistics.median(v) - base) * 1e3 / L, 2)} for k, v in res.items()}))
