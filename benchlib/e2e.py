"""End-to-end legs through the public C-ABI calls, in the serving node's call order (P:720-729:
match -> descriptor -> layer-ready waits).

hbm_tier (`e2e.hbm_tier`): the chunk store is the HBM cache itself (the tier the bench's `value`
measures) -- the control-plane cost of the serving call order against the device rate.  Every step, for the next request of a rotating set: its tokens (host) are hashed and
matched (oc_match_prefix: SHA-256 chain + probe, host), its descriptor is built (key resolution,
block table, one H2D upload of the descriptor block from pinned staging), the fetch is launched,
the consumer stream waits on the last layer, and the layer-ready stamps come back to pinned host
memory (oc_layer_times_async, D2H).  Control is pipelined as a serving node would run it: request
i+1's hashing and descriptor build run on the host while request i's fetch runs on the GPU; the
host blocks only on request i-1's stamps.  Timed by the host wall clock from the first match to the
last stamps in host memory; host microseconds per stage are reported.

pcie_tier (the contract's `e2e`: the step's inputs come from HOST buffers): the same call order with
the store in pinned host memory -- every step the request's N*S*L chunk bytes cross PCIe (copy
engine into an HBM stage + the scatter kernel) and the layer stamps come back.  `value` is the
bench metric (read + write bytes, 2*N*S*L per step, / wall time); since the rate is bounded by
PCIe, the payload rate over the link (`pcie_read_GBps`, N*S*L per step) is reported against an
in-harness pinned -> device copy of the same size.
"""
import statistics
import time

import numpy as np

from .common import N_CHUNKS_4K, ROTATE, UNIT
from .headline import build_sets


def descriptor_upload_bytes(N, L, n_blocks):
    """Bytes of the descriptor block uploaded per build (descriptor.cpp block_layout, 16-byte
    aligned parts): src[N] u64, k_base/v_base[L] u64, ts[L+1] u64, unit_cnt[L] u32, ready/next, bt."""
    a = lambda x: (x + 15) & ~15
    return a(N * 8) + 2 * a(L * 8) + a((L + 1) * 8) + a(L * 4) + 16 + a(n_blocks * 4)


def hbm_tier(args, oc, torch, dev, lay_t, ws=1, rank=0, dist=None, backend="nccl"):
    L, G, Bs = lay_t[0], lay_t[4], 16
    row, S, chunk = oc.geometry(lay_t)
    N = N_CHUNKS_4K
    store, sets = build_sets(oc, torch, dev, lay_t, N, rank, seed_base=2000)
    copy_s, cons_s = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
    steps = max(8, min(args.steps, 200))
    stamps = [torch.zeros(L + 1, dtype=torch.int64).pin_memory() for _ in range(4)]
    done = [torch.cuda.Event() for _ in range(4)]
    host = {"match": [], "build": [], "fetch": [], "wait": [], "readback_wait": []}

    def run(n, record=True):
        pend = []                                   # (step, descriptor) whose stamps are in flight
        bad = 0
        for i in range(n + 1):
            if i < n:
                st = sets[i % ROTATE]
                t0 = time.perf_counter()
                keys = store.match_prefix(st["tokens"])                     # host: SHA-256 chain + probe
                t1 = time.perf_counter()
                d = oc.build_descriptor(store, keys, lay_t, st["target"])   # host: resolve + H2D upload
                t2 = time.perf_counter()
                d.fetch_layerwise(copy_s, overlap=True)                     # GPU: gather + paged scatter
                t3 = time.perf_counter()
                d.wait_layer(L - 1, cons_s)                                 # consumer: all layers ready
                d.layer_times_async(stamps[i % 4], cons_s)                  # D2H of the result
                done[i % 4].record(cons_s)
                t4 = time.perf_counter()
                if record:
                    host["match"].append(t1 - t0)
                    host["build"].append(t2 - t1)
                    host["fetch"].append(t3 - t2)
                    host["wait"].append(t4 - t3)
                pend.append((i, d))
            while len(pend) >= 3 or (i == n and pend):  # request i-2's stamps are back (two requests in flight)
                j, dj = pend.pop(0)
                t5 = time.perf_counter()
                done[j % 4].synchronize()
                if record:
                    host["readback_wait"].append(time.perf_counter() - t5)
                t = stamps[j % 4].numpy()
                bad += int(not np.all(np.diff(t[1:]) >= 0) or t[1] < t[0])
                dj.close()
        return bad

    run(min(3, args.warmup) + 2, record=False)
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    t0 = time.perf_counter()
    bad = run(steps)
    torch.cuda.synchronize()
    secs = time.perf_counter() - t0
    if ws > 1:
        from paper_2605_22850_b200 import dist as odist
        secs = odist.max_over_ranks(secs, device=dev if backend == "nccl" else None)
    store.close()
    del sets
    torch.cuda.empty_cache()
    bytes_per_step = 2 * N * S * L
    nb = N * G // Bs + (N * G // Bs) // 4
    return {"value": ws * bytes_per_step * steps / secs / 1e9, "unit": UNIT,
            "h2d_bytes_per_step": ws * descriptor_upload_bytes(N, L, nb), "d2h_bytes_per_step": ws * (L + 1) * 8,
            "steps": steps, "ms_per_step": secs / steps * 1e3, "tier": "hbm (the chunk store is the HBM cache)",
            "host_us_per_step": {k: round(statistics.mean(v) * 1e6, 1) for k, v in host.items() if v},
            "stamps_monotone": bad == 0,
            "timing": "host wall clock from the first match_prefix to the last request's stamps in pinned host "
                      "memory; control pipelined two requests ahead of the GPU (max over ranks)"}


def pcie_tier(args, oc, torch, dev, lay_t, fopts, ws=1, backend="nccl"):
    """Public API end to end with the chunk store in pinned host memory (wall clock)."""
    import synth
    from . import verify
    L, G, Bs = lay_t[0], lay_t[4], 16
    row, S, chunk = oc.geometry(lay_t)
    N = N_CHUNKS_4K
    store = oc.Store(lay_t, capacity=ROTATE * N, tier=oc.TIER_PINNED_HOST, device=dev.index)
    reqs = []
    for r in range(ROTATE):
        (tok,), (ids,) = synth.family_streams(500 + r, G, 0, [N])
        verify.fill_store([store], oc.chunk_keys(tok, G), 500 + r, ids, chunk)
        need = N * G // Bs
        pool = need + need // 4
        bt = synth.block_table(91 + r, need, pool)
        cache = torch.empty((L, 2, pool, Bs, row), dtype=torch.uint8, device=dev)
        per_kv = pool * Bs * row
        kb = [cache.data_ptr() + l * 2 * per_kv for l in range(L)]
        tgt = oc.PagedTarget(kb, [x + per_kv for x in kb], Bs * row, row, lay_t[2] * lay_t[3], Bs, bt, 0)
        reqs.append((tok, oc.PreparedTarget(tgt, lay_t), cache))
    copy_s, cons_s = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
    stamps = [torch.zeros(L + 1, dtype=torch.int64).pin_memory() for _ in range(3)]
    done = [torch.cuda.Event() for _ in range(3)]

    def run(n):
        """n requests in the serving call order, the host control of request i+1 (hashing,
        descriptor build and upload, launch) issued while request i's transfer runs; the host
        blocks only on request i-1's stamps.  Returns the number of non-monotone stamp sets."""
        pend, bad = [], 0
        for i in range(n + 1):
            if i < n:
                tok, tgt, _ = reqs[i % ROTATE]
                keys = store.match_prefix(tok)                       # host: SHA-256 chain + probe
                d = oc.build_descriptor(store, keys, lay_t, tgt)     # host: resolve + one H2D upload
                d.fetch_layerwise(copy_s, **fopts)                   # GPU reads the host slab over PCIe
                d.wait_layer(L - 1, cons_s)
                d.layer_times_async(stamps[i % 3], cons_s)           # D2H of the result (layer-ready stamps)
                done[i % 3].record(cons_s)
                pend.append((i, d))
            if len(pend) >= 2 or (i == n and pend):
                j, dj = pend.pop(0)
                done[j % 3].synchronize()
                t = stamps[j % 3].numpy()
                bad += int(not np.all(np.diff(t[1:]) >= 0) or t[1] < t[0])
                dj.close()
        return bad

    steps = max(4, min(args.steps, 40))
    run(min(3, args.warmup) + 1)
    torch.cuda.synchronize()
    if ws > 1:
        torch.distributed.barrier()
    t0 = time.perf_counter()
    bad = run(steps)
    torch.cuda.synchronize()
    secs = time.perf_counter() - t0
    if ws > 1:                                      # whole job: all ranks' bytes / the slowest rank
        from paper_2605_22850_b200 import dist as odist
        secs = odist.max_over_ranks(secs, device=dev if backend == "nccl" else None)
    store.close()
    del reqs
    torch.cuda.empty_cache()
    pcie = N * S * L                                # payload bytes crossing PCIe per step
    # in-harness PCIe reference: a pinned -> device copy_ of the same payload size, best of 8
    h = torch.empty(pcie, dtype=torch.uint8).pin_memory()
    dd = torch.empty(pcie, dtype=torch.uint8, device=dev)
    h2d = 0.0
    for _ in range(8):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        dd.copy_(h, non_blocking=True)
        b.record()
        torch.cuda.synchronize()
        h2d = max(h2d, pcie / a.elapsed_time(b) / 1e6)
    del h, dd
    torch.cuda.empty_cache()
    pcie_GBps = ws * pcie * steps / secs / 1e9
    return {"value": ws * 2 * pcie * steps / secs / 1e9, "unit": UNIT,
            "h2d_bytes_per_step": pcie + descriptor_upload_bytes(N, L, N * G // Bs),
            "d2h_bytes_per_step": (L + 1) * 8,
            "pcie_read_GBps": round(pcie_GBps, 2), "h2d_copy_GBps": round(h2d, 1),
            "pcie_frac_of_h2d_copy": round(pcie_GBps / ws / h2d, 3) if h2d else None,
            "ms_per_step": round(secs / steps * 1e3, 3), "steps": steps, "stamps_monotone": bad == 0,
            "tier": ("pinned_host (copy engine: one strided transfer per layer into an HBM stage, then "
                     "the scatter kernel)" if fopts.get("engine") == oc.COPY_CE else
                     "pinned_host (PCIe zero-copy reads by the fetch kernel)"),
            "timing": "host wall clock from the first match_prefix to the last request's stamps in pinned host "
                      "memory; control pipelined one request ahead of the GPU (max over ranks)"}
