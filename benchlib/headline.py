"""The N=1 workload (BASELINE configs[1]): Llama-3-8B KV layout, one request per step with a 4K-token
prefix hit (N = 256 chunks of G = 16 tokens), delivered into a fragmented vLLM-style paged cache
(Bs = 16, NHD).  A step is one whole fetch_layerwise of the request -- the layer-major gather +
paged scatter of all 32 layers (Alg. A1), the layers announced in order -- and the consumer
stream's wait on the last announcement.  ROTATE independent requests (own chunks, own cache)
rotate so that consecutive steps touch 4 GiB > L2.  Steps are launched back to back with
OC_FETCH_OVERLAP (the requests are independent, so each launch may start during the previous
one's tail); `--no-overlap` launches them in plain stream order.

value     = 2*N*S*L bytes per step x steps / device time of the timed region (CUDA events:
            copy-stream start -> consumer-stream end), whole job (all ranks), max over ranks
roofline  = the fetch kernel alone: the same bytes / the copy stream's span over the K launches
            (events on the copy stream around the launches, i.e. the mean launch duration in the
            pipelined steady state), against MEASURED_PEAKS.json hbm_gbs
verified  = after the timed region, request 0's delivered bytes (all 32 layers, read back through
            its block table) against the oracle's Alg. A1 gather, byte for byte
"""
import statistics
import time

import numpy as np

from .common import N_CHUNKS_4K, ROTATE, ClockSampler, in_harness_copy, ncu_traffic, peaks
from . import verify


def build_sets(oc, torch, dev, lay_t, n_chunks, rank, seed_base=1000, tier=None, rotate=ROTATE):
    """ROTATE request sets in one store: synth payloads (regenerable by the oracle) put in one seeded
    random interleaving, so every request's chunks sit at random slab positions (SURVEY 8(d)
    config 2), each request with its own fragmented paged cache (pool = 1.25 x the blocks needed)
    and prepared target."""
    import synth
    L, G, Bs = lay_t[0], lay_t[4], 16
    row, S, chunk = oc.geometry(lay_t)
    store = oc.Store(lay_t, capacity=rotate * n_chunks, tier=oc.TIER_HBM if tier is None else tier,
                     device=dev.index)
    sets, reqs = [], []
    for r in range(rotate):
        seed = seed_base * rank + 1000 + r
        (tok,), (ids,) = synth.family_streams(seed, G, 0, [n_chunks])
        reqs.append((oc.chunk_keys(tok, G), seed, ids, tok))
    verify.fill_store_scattered(store, [q[:3] for q in reqs], chunk, order_seed=seed_base * rank + 7)
    for r, (keys, seed, ids, tok) in enumerate(reqs):
        need = n_chunks * G // Bs
        pool = need + need // 4
        bt = synth.block_table(77 + r, need, pool)
        cache = torch.empty((L, 2, pool, Bs, row), dtype=torch.uint8, device=dev)
        per_kv = pool * Bs * row
        kb = [cache.data_ptr() + l * 2 * per_kv for l in range(L)]
        tgt = oc.PagedTarget(kb, [x + per_kv for x in kb], Bs * row, row, lay_t[2] * lay_t[3], Bs, bt, 0)
        sets.append({"seed": seed, "tokens": tok, "ids": ids, "keys": keys, "bt": bt, "cache": cache,
                     "target": oc.PreparedTarget(tgt, lay_t)})
    torch.cuda.synchronize()
    return store, sets


def run(args, oc, torch, dev, lay_t, ws, rank, dist=None, backend="nccl"):
    from oracle.geometry import Layout
    L, G = lay_t[0], lay_t[4]
    row, S, chunk = oc.geometry(lay_t)
    N = N_CHUNKS_4K
    store, sets = build_sets(oc, torch, dev, lay_t, N, rank)
    descs = [oc.build_descriptor(store, st["keys"], lay_t, st["target"]) for st in sets]
    copy_s = torch.cuda.Stream(device=dev)
    cons_s = torch.cuda.Stream(device=dev)
    bytes_per_step = 2 * N * S * L                    # read + write
    overlap = not args.no_overlap
    fopts = {"overlap": overlap}
    if args.engine == "ldst":
        fopts = {"engine": oc.COPY_LDST}
    if args.mode == "per_layer":
        fopts = {"mode": oc.FETCH_PER_LAYER, "overlap": overlap}

    def step(i):
        d = descs[i % ROTATE]
        d.fetch_layerwise(copy_s, **fopts)
        # the consumer waits on the last layer: layers are announced strictly in order, so this
        # completes after every layer's ready signal (per-layer waits interleaved with compute are
        # the stall legs' subject)
        d.wait_layer(L - 1, cons_s)

    clocks = ClockSampler(dev.index)
    if not args.profile:
        clocks.start()
        time.sleep(0.3)
    for i in range(args.warmup):
        step(i)
    t_soak = time.perf_counter()
    i = 0
    while not args.profile and time.perf_counter() - t_soak < 1.0:   # keep the GPU loaded while sampling
        step(i)
        i += 1
        if i % 64 == 0:
            torch.cuda.synchronize()
    torch.cuda.synchronize()
    t_start, t_copy_end, t_end = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t_start.record(copy_s)
    cons_s.wait_event(t_start)
    for i in range(args.steps):
        step(i)
    t_copy_end.record(copy_s)
    t_end.record(cons_s)
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    clk = clocks.stop()
    elapsed_ms = t_start.elapsed_time(t_end)
    copy_ms = t_start.elapsed_time(t_copy_end)
    if ws > 1:
        t = torch.tensor([elapsed_ms], device=dev if backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)                # max over ranks
        elapsed_ms = float(t.item())
    ms_per_step = elapsed_ms / args.steps
    value = ws * bytes_per_step * args.steps / (elapsed_ms / 1e3) / 1e9
    peak, peak_src = peaks()
    achieved = bytes_per_step * args.steps / (copy_ms / 1e3) / 1e9
    traffic, traffic_fresh = ncu_traffic()

    # diagnostics outside the timed region: isolated launches (stream order, no overlap)
    iso = []
    for i in range(min(args.steps, 40)):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        d = descs[i % ROTATE]
        a.record(copy_s)
        d.fetch_layerwise(copy_s, **{k: v for k, v in fopts.items() if k != "overlap"})
        b.record(copy_s)
        iso.append((a, b))
    torch.cuda.synchronize()
    iso_us = [a.elapsed_time(b) * 1e3 for a, b in iso]
    x0_us = []
    for i in range(ROTATE):
        descs[i].fetch_layerwise(copy_s, **{k: v for k, v in fopts.items() if k != "overlap"})
        t = descs[i].layer_times().astype(np.int64)
        x0_us.append((t[1] - t[0]) / 1e3)
    harness_copy = in_harness_copy(torch, dev, copy_s, bytes_per_step // 2) if not args.profile else None

    # verification of the timed launch configuration: request 0 in full against the oracle
    ver = None
    if rank == 0 and not args.profile:
        st = sets[0]
        lay = Layout(*lay_t)
        idx = verify.slot_index(torch, dev, st["bt"], N * G, 16)
        ok, nbytes, t_or, t_all = verify.full_check(torch, lay, st["seed"], st["keys"], st["ids"], st["cache"],
                                                    idx, range(L))
        ver = {"request0_all_layers_bit_exact": ok, "bytes_compared": nbytes, "oracle_s": round(t_or, 2),
               "oracle_s_per_GB": round(t_or / (nbytes / 1e9), 2)}
    for d in descs:
        d.close()
    store.close()
    del sets
    torch.cuda.empty_cache()
    return {
        "value": value, "ms_per_step": ms_per_step, "clocks": clk,
        "gpu_launches": args.steps * (L if args.mode == "per_layer" else 1),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "frac_of_spec": round(achieved / 8000.0, 4),   # both denominators (8 TB/s spec)
                     "traffic": traffic if traffic_fresh else None,
                     "traffic_source": ("profiles/ncu_full_summary.json (ncu --set full of the current kernel "
                                        "sources)" if traffic_fresh else
                                        "none: the committed capture is of older kernel sources"),
                     "peak_source": peak_src, "kernel": "fetch_bulk_kernel<0>",
                     "bytes_per_launch": bytes_per_step,
                     "mean_launch_us": copy_ms * 1e3 / args.steps,
                     "timing": "CUDA events on the copy stream around the K back-to-back launches"},
        "isolated_launch_us": {q: round(float(np.percentile(iso_us, p)), 2) for q, p in
                               (("p10", 10), ("p50", 50), ("p90", 90))},
        "X0_us_isolated": round(statistics.median(x0_us), 2),
        "in_harness_copy": None if harness_copy is None else {
            "GBps": round(harness_copy, 1), "kernel_frac": round(achieved / harness_copy, 4),
            "method": "torch copy_ of %d MiB device to device, read + write counted, median of 20 after 3 "
                      "warm-ups" % (bytes_per_step // 2 >> 20)},
        "verified": ver,
        "launch": ("back-to-back fetches of rotating requests with OC_FETCH_OVERLAP (programmatic dependent "
                   "launch)" if fopts.get("overlap") else "stream order") +
                  (", one launch + CUDA event per layer" if args.mode == "per_layer" else ""),
    }
