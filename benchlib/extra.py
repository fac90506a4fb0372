"""Optional legs (flags of bench.py): granularity, offload, sensitivity, crossover, co-run, rate sweep,
batches, hashing, the tenant pool, the old weak-scaling serve leg, and the cross-GPU p2p leg."""
import json
import os
import statistics
import sys
import time

import numpy as np

from .common import (METRIC, N_CHUNKS_4K, ROTATE, TABLE_A5_T_TOTAL_MS, UNIT, ClockSampler, bench_config,  # noqa: F401
                     cores_used, dist_env, in_harness_copy, peaks, prefill_window_s, sched_workloads)
from .stall import stall_leg  # noqa: E402


def p2p_leg(args, oc, torch, dev, lay_t, ws, rank, backend="nccl"):
    """SURVEY 8(a) a11 / config 5's cross-GPU reads: rank r's store holds a 4K-token request's
    chunks in its HBM; the stores are exchanged once (CUDA IPC export blobs over all_gather_object)
    and rank r fetches the request homed on rank (r+1) mod N into its own paged cache -- the same
    fused kernel, its TMA loads crossing NVLink.  All ranks fetch concurrently; time = max over
    ranks of the device time of K fetches.  GB/s counts r+w (2*N*S*L) per fetch; the NVLink
    ingress per GPU is half of it.  Rank 0 checks two sampled layers byte for byte against the
    payload regenerated from the peer's seed."""
    import synth
    from paper_2605_22850_b200 import dist as odist
    L, G, Bs = lay_t[0], lay_t[4], 16
    row, S, chunk = oc.geometry(lay_t)
    N = N_CHUNKS_4K
    seed_of = lambda r: 31000 + r
    store = oc.Store(lay_t, capacity=N, tier=oc.TIER_HBM, device=dev.index)
    (tok,), (ids,) = synth.family_streams(seed_of(rank), G, 0, [N])
    store.put_chunks(oc.chunk_keys(tok, G), torch.from_numpy(synth.payloads(seed_of(rank), ids, chunk)).to(dev))
    torch.cuda.synchronize()
    blobs = odist.exchange_blobs(store.export())
    src_rank = (rank + 1) % ws
    peer = oc.Store.import_(blobs[src_rank], device=dev.index)
    local = oc.Store(lay_t, capacity=1, tier=oc.TIER_HBM, device=dev.index)   # resolves through its peer
    local.attach_peer(peer)
    (ptok,), (pids,) = synth.family_streams(seed_of(src_rank), G, 0, [N])
    keys = local.match_prefix(ptok)
    need = N * G // Bs
    bt = synth.block_table(55 + rank, need, need + need // 4)
    cache = torch.empty((L, 2, need + need // 4, Bs, row), dtype=torch.uint8, device=dev)
    per_kv = cache.shape[2] * Bs * row
    kb = [cache.data_ptr() + l * 2 * per_kv for l in range(L)]
    tgt = oc.PagedTarget(kb, [x + per_kv for x in kb], Bs * row, row, lay_t[2] * lay_t[3], Bs, bt, 0)
    d = oc.build_descriptor(local, keys, lay_t, tgt)
    s = torch.cuda.Stream(device=dev)
    steps = max(5, min(args.steps, 50))
    for _ in range(3):
        d.fetch_layerwise(s)
    s.synchronize()
    ok = None
    if rank == 0:                                   # sampled check of what crossed NVLink
        pl = synth.payloads(seed_of(src_rank), pids, chunk)
        slots = bt[np.arange(N * G) // Bs].astype(np.int64) * Bs + np.arange(N * G) % Bs
        ok = True
        for l in (0, L - 1):
            want = pl[:, l * S:(l + 1) * S].reshape(N, 2, G, row)
            for kv in (0, 1):
                got = cache[l, kv].reshape(-1, row)[torch.from_numpy(slots).to(dev)].cpu().numpy()
                ok &= bool(np.array_equal(got, want[:, kv].reshape(N * G, row)))
    if ws > 1:
        torch.distributed.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(steps):
        d.fetch_layerwise(s)
    b.record(s)
    s.synchronize()
    ms = odist.max_over_ranks(a.elapsed_time(b), device=dev if backend == "nccl" else None)
    # in-harness P2P reference: a copy-engine copy of the peer's slab into local HBM
    from cuda.bindings import runtime as cudart
    pbase, pbytes = peer.slab
    nb = int(min(pbytes, 1 << 30))
    scratch = torch.empty(nb, dtype=torch.uint8, device=dev)
    best = 0.0
    for _ in range(3):
        a.record(s)
        err, = cudart.cudaMemcpyAsync(scratch.data_ptr(), pbase, nb, cudart.cudaMemcpyKind.cudaMemcpyDefault,
                                      s.cuda_stream)
        b.record(s)
        s.synchronize()
        if err == cudart.cudaError_t.cudaSuccess:
            best = max(best, nb / a.elapsed_time(b) / 1e6)
    del scratch
    d.close()
    if ws > 1:
        torch.distributed.barrier()                 # peers done reading before any store goes away
    local.close()
    peer.close()
    store.close()
    del cache
    torch.cuda.empty_cache()
    rw = 2 * N * S * L
    return {"workload": f"each rank fetches a 4K-token hit (N={N}) homed on the next rank's GPU",
            "ranks": ws, "steps": steps, "GBps_rw_aggregate": round(ws * rw * steps / ms / 1e6, 1),
            "nvlink_ingress_GBps_per_gpu": round(rw / 2 * steps / ms / 1e6, 1),
            "ms_per_fetch_max_over_ranks": round(ms / steps, 4), "rank0_sampled_layers_bit_exact": ok,
            "p2p_copy_engine_GBps_rank0": round(best, 1),
            "ingress_frac_of_p2p_copy": round(rw / 2 * steps / ms / 1e6 / best, 3) if best else None,
            "peers_share_one_gpu": torch.cuda.device_count() < ws}


def serve_leg(args, oc, torch, dev, lay_t, ws=1, rank=0, backend="nccl"):
    """Config 5: a stream of concurrent mixed requests through the public API
    into a bounded paged KV pool.  Corpus: 32 x 4K-token + 4 x 64K-token prefix families (48 GiB
    in all); requests pick 4K/64K 50/50, a family by Zipf(1.1), hit 50% or 87.5%.  The pool
    (48 GiB of [L][2][blocks][Bs][row] per GPU) hands out blocks from a free list in FIFO
    admission order (a fragmented, seeded initial order); a request is admitted when its blocks
    are free, gets a descriptor over its blocks, is fetched on one of 8 streams, and its blocks
    return to the free list when its fetch's completion event fires.
    With N ranks (weak scaling, R requests per rank): family g is homed on rank g mod N, each
    rank's store holds its home families, the stores are exchanged once at setup (CUDA IPC blobs,
    all_gather_object) and attached as peers, and a rank's requests pick a local family with
    probability p_aff = 0.875 -- the rest read their chunks from a peer GPU inside the same fetch
    kernel (NVLink P2P loads).  No collective on the data path.  GB/s = 2*N*S*L summed over all
    requests / the max over ranks of the device time from the first launch to the last
    completion."""
    import collections
    import synth
    from paper_2605_22850_b200 import dist as odist
    L, G, Bs = lay_t[0], lay_t[4], 16
    row, S, chunk = oc.geometry(lay_t)
    R = args.serve
    fam_short, fam_long = (int(x) for x in os.environ.get("OC_SERVE_FAMILIES", "32,4").split(","))
    n_short, n_long = 4096 // G, 65536 // G
    home_of = lambda long, f: (f + fam_short * int(long)) % ws
    mine = [(lg, f, n) for lg, nf, n in ((False, fam_short, n_short), (True, fam_long, n_long))
            for f in range(nf) if home_of(lg, f) == rank]
    store = oc.Store(lay_t, capacity=max(1, sum(n for _, _, n in mine)), tier=oc.TIER_HBM, device=dev.index)
    gen = torch.Generator(device=dev).manual_seed(5 + rank)
    fam_keys = {}
    for long, nf, n in ((False, fam_short, n_short), (True, fam_long, n_long)):
        for f in range(nf):
            (tok,), _ = synth.family_streams(8000 + 100 * long + f, G, 0, [n])
            keys = oc.chunk_keys(tok, G)
            fam_keys[(long, f)] = keys
            if home_of(long, f) != rank:
                continue
            for b0 in range(0, n, 512):
                pl = torch.randint(0, 256, (min(n, b0 + 512) - b0, chunk), dtype=torch.uint8, device=dev, generator=gen)
                store.put_chunks(keys[b0:b0 + pl.shape[0]], pl)
                del pl
    peers = []
    if ws > 1:                                     # setup only: exchange store handles, attach peers
        torch.cuda.synchronize()
        blobs = odist.exchange_blobs(store.export())
        for r, blob in enumerate(blobs):
            if r != rank:
                p = oc.Store.import_(blob, device=dev.index)
                store.attach_peer(p)
                peers.append(p)
    pool_blocks = (int(os.environ.get("OC_SERVE_POOL_GIB", "48")) << 30) // (L * 2 * Bs * row)
    cache = torch.empty((L, 2, pool_blocks, Bs, row), dtype=torch.uint8, device=dev)
    per_kv = pool_blocks * Bs * row
    kb = [cache.data_ptr() + l * 2 * per_kv for l in range(L)]
    vb = [x + per_kv for x in kb]
    reqs = synth.serving_requests(11 + rank, R, fam_short, fam_long, home_of=home_of if ws > 1 else None, rank=rank)
    remote_bytes = sum(2 * (int((65536 if lg else 4096) * h) // G) * S * L for lg, f, h in reqs if home_of(lg, f) != rank)
    streams = [torch.cuda.Stream(device=dev) for _ in range(8)]
    start = torch.cuda.Event(enable_timing=True)

    def run():
        free = collections.deque(int(b) for b in synth.block_table(3, pool_blocks, pool_blocks))
        pending = collections.deque(enumerate(reqs))
        inflight = []
        total_bytes, fetch_us, wait_blocks, n_done = 0, [], 0, 0
        torch.cuda.synchronize()
        if ws > 1:
            torch.distributed.barrier()
        start.record(streams[0])
        for s in streams[1:]:
            s.wait_event(start)
        ends = []
        t_host = time.perf_counter()
        while pending or inflight:
            still = []
            for ev, d, blocks, nb in inflight:
                if ev.query():
                    t = d.layer_times().astype(np.int64)
                    fetch_us.append((t[L] - t[0]) / 1e3)
                    d.close()
                    free.extend(blocks)
                    n_done += 1
                else:
                    still.append((ev, d, blocks, nb))
            inflight = still
            admitted = False
            while pending:
                i, (long, fam, hit) = pending[0]
                n = int((65536 if long else 4096) * hit) // G
                need = n * G // Bs
                if len(free) < need:
                    wait_blocks += 1
                    break
                pending.popleft()
                blocks = [free.popleft() for _ in range(need)]
                tgt = oc.PagedTarget(kb, vb, Bs * row, row, lay_t[2] * lay_t[3], Bs, np.asarray(blocks, np.int32), 0)
                try:
                    d = oc.build_descriptor(store, fam_keys[(long, fam)][:n], lay_t, tgt)
                    s = streams[i % len(streams)]
                    d.fetch_layerwise(s)
                except oc.ObjcacheError:
                    print(f"serve: request {i} (long={long}, family={fam}, hit={hit}, N={n}, "
                          f"blocks {min(blocks)}..{max(blocks)}, {len(inflight)} in flight) failed",
                          file=sys.stderr)
                    raise
                ev = torch.cuda.Event(enable_timing=True)
                ev.record(s)
                ends.append(ev)
                inflight.append((ev, d, blocks, n))
                total_bytes += 2 * n * S * L
                admitted = True
            if not admitted and inflight:
                inflight[0][0].synchronize()
        torch.cuda.synchronize()
        host_s = time.perf_counter() - t_host
        dev_ms = max(start.elapsed_time(e) for e in ends)
        return total_bytes, dev_ms, host_s, fetch_us, wait_blocks

    def run_batched(max_batch=64):
        """The same admission, but every admission step launches the requests it admitted as ONE
        position-major batch (oc.BATCH_BY_POSITION): requests of one prefix family read their
        shared chunks together.  Blocks return when the batch's completion event fires."""
        free = collections.deque(int(b) for b in synth.block_table(3, pool_blocks, pool_blocks))
        pending = collections.deque(enumerate(reqs))
        inflight = []
        total_bytes, n_batches, sizes = 0, 0, []
        torch.cuda.synchronize()
        if ws > 1:
            torch.distributed.barrier()
        start.record(streams[0])
        for s in streams[1:]:
            s.wait_event(start)
        ends = []
        t_host = time.perf_counter()
        while pending or inflight:
            still = []
            for ev, b, ds, blocks in inflight:
                if ev.query():
                    b.close()
                    for d in ds:
                        d.close()
                    free.extend(blocks)
                else:
                    still.append((ev, b, ds, blocks))
            inflight = still
            ds, blocks_all = [], []
            while pending and len(ds) < max_batch:
                i, (long, fam, hit) = pending[0]
                n = int((65536 if long else 4096) * hit) // G
                need = n * G // Bs
                if len(free) < need:
                    break
                pending.popleft()
                blocks = [free.popleft() for _ in range(need)]
                tgt = oc.PagedTarget(kb, vb, Bs * row, row, lay_t[2] * lay_t[3], Bs, np.asarray(blocks, np.int32), 0)
                ds.append(oc.build_descriptor(store, fam_keys[(long, fam)][:n], lay_t, tgt))
                blocks_all += blocks
                total_bytes += 2 * n * S * L
            if ds:
                b = oc.Batch(ds, order=oc.BATCH_BY_POSITION)
                s = streams[n_batches % len(streams)]
                b.fetch(s)
                ev = torch.cuda.Event(enable_timing=True)
                ev.record(s)
                ends.append(ev)
                inflight.append((ev, b, ds, blocks_all))
                n_batches += 1
                sizes.append(len(ds))
            elif inflight:
                inflight[0][0].synchronize()
        torch.cuda.synchronize()
        host_s = time.perf_counter() - t_host
        dev_ms = max(start.elapsed_time(e) for e in ends)
        return total_bytes, dev_ms, host_s, n_batches, sizes

    run()                                               # warm-up pass (descriptor pool, modules)
    total_bytes, dev_ms, host_s, fetch_us, waits = run()
    mb = int(os.environ.get("OC_SERVE_MAX_BATCH", "16"))    # profiles/r01_serve.json: 4..64 swept
    run_batched(mb)
    tb_b, dev_ms_b, host_s_b, n_batches, sizes = run_batched(mb)
    red_dev = dev if backend == "nccl" else None
    max_ms = odist.max_over_ranks(dev_ms, device=red_dev)
    all_bytes = odist.sum_over_ranks(total_bytes, device=red_dev)
    all_remote = odist.sum_over_ranks(remote_bytes, device=red_dev)
    res = {"requests_per_rank": R, "ranks": ws,
           "mix": f"4K/64K 50/50, Zipf(1.1) over {fam_short} + {fam_long} families, hit 50%/87.5%"
                  + (f", family g homed on rank g mod {ws}, p_aff 0.875" if ws > 1 else ""),
           "pool_GiB_per_rank": pool_blocks * L * 2 * Bs * row / 2**30, "bytes_rw": all_bytes,
           "remote_byte_fraction": round(all_remote / all_bytes, 4),
           "GBps_device": round(all_bytes / max_ms / 1e6, 1),
           "GBps_rank0_host_wall": round(total_bytes / host_s / 1e9, 1),
           "device_ms_max_over_ranks": round(max_ms, 2),
           "fetch_us_p50_rank0": round(float(np.percentile(fetch_us, 50)), 1),
           "fetch_us_p99_rank0": round(float(np.percentile(fetch_us, 99)), 1),
           "admission_stalls_rank0": waits}
    max_ms_b = odist.max_over_ranks(dev_ms_b, device=red_dev)
    res["batched_by_position"] = {
        "how": f"each admission step launches its admitted requests (<= {mb}) as one position-major batch",
        "GBps_device": round(odist.sum_over_ranks(tb_b, device=red_dev) / max_ms_b / 1e6, 1),
        "GBps_rank0_host_wall": round(tb_b / host_s_b / 1e9, 1),
        "device_ms_max_over_ranks": round(max_ms_b, 2), "batches_rank0": n_batches,
        "batch_size_median_rank0": float(np.median(sizes)) if sizes else 0}
    del cache
    if ws > 1:
        torch.distributed.barrier()                # peers' fetches done before any store goes away
    store.close()
    for p in peers:
        p.close()
    torch.cuda.empty_cache()
    return res


def offload_leg(args, oc, torch, dev, lay_t):
    """Offload path: put_from_paged of 4K-token requests (N = 256 chunks)
    from a fragmented paged cache into fresh slots of an HBM store -- the inverse gather.  Each
    iteration offloads a new key set (no dedup); 10 offloads are issued back to back on one stream
    and timed with CUDA events around them.  GB/s = 2*N*S*L per offload / device time per
    offload; host_us = one call's host time (key reservation + descriptor upload + launch)."""
    import synth
    L, G, Bs = lay_t[0], lay_t[4], 16
    row, S, chunk = oc.geometry(lay_t)
    N = N_CHUNKS_4K
    iters = 12
    store = oc.Store(lay_t, capacity=iters * N, tier=oc.TIER_HBM, device=dev.index)
    need = N * G // Bs
    pool = need + need // 4
    cache = torch.randint(0, 256, (L, 2, pool, Bs, row), dtype=torch.uint8, device=dev)
    per_kv = pool * Bs * row
    kb = [cache.data_ptr() + l * 2 * per_kv for l in range(L)]
    tgt = oc.PagedTarget(kb, [x + per_kv for x in kb], Bs * row, row, lay_t[2] * lay_t[3], Bs,
                         synth.block_table(21, need, pool), 0)
    key_sets = []
    for i in range(iters):
        (tok,), _ = synth.family_streams(6000 + i, G, 0, [N])
        key_sets.append(oc.chunk_keys(tok, G))
    s = torch.cuda.Stream(device=dev)
    torch.cuda.synchronize()
    for i in range(2):                              # warm-up (pools, module load)
        assert oc.put_from_paged(store, key_sets[i], lay_t, tgt, s) == N
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    host_us = []
    a.record(s)
    for i in range(2, iters):                       # back to back: the host enqueues ahead of the GPU
        t0 = time.perf_counter()
        n_new = oc.put_from_paged(store, key_sets[i], lay_t, tgt, s)
        host_us.append((time.perf_counter() - t0) * 1e6)
        assert n_new == N
    b.record(s)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / (iters - 2)
    res = {"N": N, "bytes_rw_per_offload": 2 * N * S * L, "GBps": round(2 * N * S * L / ms / 1e6, 1),
           "ms_per_offload": round(ms, 4), "offloads_timed": iters - 2,
           "host_us_median": round(float(np.median(host_us)), 1),
           "engine": os.environ.get("OC_OFFLOAD_ENGINE", "bulk")}
    store.close()
    del cache
    torch.cuda.empty_cache()
    return res


def sensitivity_leg(args, oc, torch, dev, lay_t):
    """Fig. 14 analog: TTFT increase when the transfer path is capped at 10 Gbps
    instead of 100 Gbps, layerwise vs chunkwise, for the Table A5 cells (4K/64K x 50%/87.5%, A100
    windows).  Chunks in the pinned host tier; the cap is the fetch's pacer (layer l released at
    t0 + l*s/r; chunkwise = the same paced transfer with every wait on the whole prefix).  Model:
    Eq. 3 with uniform X = s/r (layerwise), L*X + L*C (chunkwise)."""
    import synth
    L, G, Bs = lay_t[0], lay_t[4], 16
    row, S, chunk = oc.geometry(lay_t)
    out = {}
    for ctx, hit in ((4096, 0.5), (4096, 0.875), (65536, 0.5), (65536, 0.875)):
        N = int(ctx * hit) // G
        c = TABLE_A5_T_TOTAL_MS[(ctx, hit)] / L / 1e3                 # A100 windows
        s = N * S
        store = oc.Store(lay_t, capacity=N, tier=oc.TIER_PINNED_HOST, device=dev.index)
        (tok,), _ = synth.family_streams(77 + N, G, 0, [N])
        keys = oc.chunk_keys(tok, G)
        gen = torch.Generator(device=dev).manual_seed(N)
        for b0 in range(0, N, 512):
            pl = torch.randint(0, 256, (min(N, b0 + 512) - b0, chunk), dtype=torch.uint8, device=dev, generator=gen)
            store.put_chunks(keys[b0:b0 + pl.shape[0]], pl)
            del pl
        need = N * G // Bs
        cache = torch.empty((L, 2, need, Bs, row), dtype=torch.uint8, device=dev)
        per_kv = need * Bs * row
        kb = [cache.data_ptr() + l * 2 * per_kv for l in range(L)]
        tgt = oc.PagedTarget(kb, [x + per_kv for x in kb], Bs * row, row, lay_t[2] * lay_t[3], Bs,
                             synth.block_table(9, need, need), 0)
        descs = {"layerwise": oc.build_descriptor(store, keys, lay_t, tgt),
                 "chunkwise": oc.build_descriptor(store, keys, lay_t, tgt, oc.DELIVER_CHUNK_MAJOR)}
        copy_s, cons_s = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)

        def chain(d, rate):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            a.record(copy_s)
            cons_s.wait_event(a)
            d.fetch_layerwise(copy_s, pace_Bps=rate)
            for l in range(L):
                d.wait_layer(l, cons_s)
                oc.emulate_compute(int(c * 1e9), cons_s)
            b.record(cons_s)
            torch.cuda.synchronize()
            return a.elapsed_time(b)

        for d in descs.values():           # warm-up (module load, wait entry point), untimed
            d.fetch_layerwise(copy_s)
            for l in range(L):
                d.wait_layer(l, cons_s)
                oc.emulate_compute(0, cons_s)
            torch.cuda.synchronize()
        cell = {"N": N, "s_MiB": s / 2**20, "C_ms": round(c * 1e3, 3), "r_star_GBps": round(s / c / 1e9, 3)}
        for mode, d in descs.items():
            t = {g: chain(d, g * 1e9 / 8) for g in (100, 10)}
            model = {}
            for g in (100, 10):
                X = s / (g * 1e9 / 8)
                model[g] = (X + (L - 1) * max(X, c) + c) if mode == "layerwise" else L * X + L * c
            cell[mode] = {"ttft_100G_ms": round(t[100], 2), "ttft_10G_ms": round(t[10], 2),
                          "increase_pct": round(100 * (t[10] / t[100] - 1), 2),
                          "model_increase_pct": round(100 * (model[10] / model[100] - 1), 2)}
        out[f"{ctx // 1024}K,{hit:g}"] = cell
        for d in descs.values():
            d.close()
        store.close()
        del cache
        torch.cuda.empty_cache()
    return out


def granularity_leg(args, oc, torch, dev, lay_t, fopts):
    """Config 2's chunk-size sweep: the 4K-token hit at G = 16, 64, 256
    (N = 256, 64, 16) through the fused kernel, plus the unfused comparison at G = 16: the same
    kernel into the paper's flat client buffer [L][N*S] (Alg. A1's B_l), then the client-side
    scatter into the paged cache (oc scatter_flat; a torch index_copy_ per layer beside it) --
    4*N*S bytes per layer instead of 2*N*S.  GB/s are
    algorithmic (2*N*S*L) over device time, best of 20 after warm-up, rotating 2 request sets."""
    import synth
    L, Bs = lay_t[0], 16
    out = {}
    for G in (16, 64, 256):
        lay = synth.with_chunk_tokens(synth.LLAMA3_8B, G).as_tuple()
        row, S, chunk = oc.geometry(lay)
        N = 4096 // G
        store = oc.Store(lay, capacity=2 * N, tier=oc.TIER_HBM, device=dev.index)
        sets = []
        for r in range(2):
            (tok,), _ = synth.family_streams(300 + r, G, 0, [N])
            keys = oc.chunk_keys(tok, G)
            store.put_chunks(keys, torch.randint(0, 256, (N, chunk), dtype=torch.uint8, device=dev))
            need = N * G // Bs
            cache = torch.empty((L, 2, need, Bs, row), dtype=torch.uint8, device=dev)
            per_kv = need * Bs * row
            kb = [cache.data_ptr() + l * 2 * per_kv for l in range(L)]
            bt = synth.block_table(40 + r, need, need)
            tgt = oc.PagedTarget(kb, [x + per_kv for x in kb], Bs * row, row, lay[2] * lay[3], Bs, bt, 0)
            d = oc.build_descriptor(store, keys, lay, tgt)
            flat = None
            if G == 16:
                flat = torch.empty((L, N * S), dtype=torch.uint8, device=dev)
                df = oc.build_descriptor(store, keys, lay, oc.FlatTarget(flat.data_ptr(), flat.numel()))
                slots = torch.from_numpy((np.asarray(bt, dtype=np.int64)[np.arange(N * G) // Bs] * Bs
                                          + np.arange(N * G) % Bs)).to(dev)
                flat = (flat, df, slots)
            sets.append((d, cache, flat))
        s = torch.cuda.Stream(device=dev)

        def timed(fn):
            for i in range(4):
                fn(i)
            best = None
            for i in range(20):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(s)
                fn(i)
                b.record(s)
                torch.cuda.synchronize()
                ms = a.elapsed_time(b)
                best = ms if best is None else min(best, ms)
            return best

        ms = timed(lambda i: sets[i % 2][0].fetch_layerwise(s, **fopts))
        x0 = [float(t[1] - t[0]) / 1e3 for t in [sets[1][0].layer_times().astype(np.int64)]][0]
        cell = {"N": N, "S_KiB": S // 1024, "GBps": round(2 * N * S * L / ms / 1e6, 1), "ms": round(ms, 4),
                "X0_us": round(x0, 2)}
        if G == 16:
            def unfused(i):
                d, cache, (flatb, df, slots) = sets[i % 2]
                df.fetch_layerwise(s, **fopts)
                with torch.cuda.stream(s):
                    for l in range(L):
                        src = flatb[l].view(N, 2, G, row).permute(1, 0, 2, 3).reshape(2, N * G, row)
                        cache[l].view(2, -1, row).index_copy_(1, slots, src)
            def unfused_ours(i):                  # the same two steps, both in our kernels
                d, cache, (flatb, df, slots) = sets[i % 2]
                df.fetch_layerwise(s, **fopts)
                d.scatter_flat(flatb.data_ptr(), flatb.numel(), s)
            ms_u = timed(unfused)
            ms_o = timed(unfused_ours)
            cell["unfused_flat_then_scatter"] = {"GBps_algorithmic": round(2 * N * S * L / ms_o / 1e6, 1),
                                                 "ms": round(ms_o, 4), "traffic_bytes": 4 * N * S * L,
                                                 "scatter": "oc scatter_flat (bulk kernel, flat source)",
                                                 "torch_scatter_GBps_algorithmic": round(2 * N * S * L / ms_u / 1e6, 1),
                                                 "torch_scatter": "torch permute+index_copy_ per layer"}
            # correctness of the comparison paths: same bytes as the fused kernel
            d, cache, _ = sets[0]
            same = True
            for fn in (unfused, unfused_ours):
                with torch.cuda.stream(s):
                    cache.zero_()
                fn(0)
                torch.cuda.synchronize()
                ref = cache.clone()
                d.fetch_layerwise(s, **fopts)
                torch.cuda.synchronize()
                same &= bool(torch.equal(ref, cache))
            cell["unfused_equals_fused"] = same
        out[f"G{G}"] = cell
        for d, cache, flat in sets:
            d.close()
            if flat is not None:
                flat[1].close()
        del sets
        store.close()
        torch.cuda.empty_cache()
    return out


def crossover_leg(args, oc, torch, dev, lay_t, fopts):
    """Eq. 2 / Fig. 13 analog: added TTFT of layerwise vs chunkwise
    delivery across context lengths (87.5% hit, B200 compute windows), per tier.  Theta_B200 is the
    smallest payload W at which layerwise is not worse than chunkwise."""
    ctxs = [128, 256, 512, 1024, 2048, 4096, 8192, 16384, 32768, 65536]
    cells = [(f"{c}t", c, c * 7 // 8, None) for c in ctxs]
    res = stall_leg(args, oc, torch, dev, lay_t, fopts, cells=cells, windows_sel=("b200",), timelines=False,
                    optlocal=False)
    out = {"windows": "b200 FLOP model, 87.5% hit", "cells": {}}
    row, S, chunk = oc.geometry(lay_t)
    for tier in ("hbm", "pinned_host"):
        theta = None
        for c in reversed(ctxs):            # smallest W from which layerwise is never worse
            r = res[f"{c}t_{tier}_b200win"]
            W = r["N"] * chunk
            out["cells"][f"{c}t_{tier}"] = {"W_MiB": W / 2**20, "layerwise_ms": r["added_ms"],
                                            "chunkwise_ms": r["added_ms_chunkwise"],
                                            "C_ms": r["C_ms_per_layer"], "X0_ms": r["X0_ms"]}
            if r["added_ms"] > r["added_ms_chunkwise"]:
                break
            theta = W
        out[f"theta_{tier}_MiB"] = None if theta is None else theta / 2**20
    return out


def corun_leg(args, oc, torch, dev, lay_t):
    """Prefill compute and KV delivery share the GPU (hard part 2): a stream of bf16
    8192^3 GEMMs (torch.matmul, the compute stand-in) runs concurrently with back-to-back 4K fetches
    on another stream.  Reported per copy-CTA budget: fetch GB/s and GEMM TFLOP/s alone and together."""
    import synth
    L, G, Bs = lay_t[0], lay_t[4], 16
    row, S, chunk = oc.geometry(lay_t)
    N = N_CHUNKS_4K
    store = oc.Store(lay_t, capacity=2 * N, tier=oc.TIER_HBM, device=dev.index)
    descs = []
    for r in range(2):
        (tok,), _ = synth.family_streams(600 + r, G, 0, [N])
        keys = oc.chunk_keys(tok, G)
        store.put_chunks(keys, torch.randint(0, 256, (N, chunk), dtype=torch.uint8, device=dev))
        need = N * G // Bs
        cache = torch.empty((L, 2, need, Bs, row), dtype=torch.uint8, device=dev)
        per_kv = need * Bs * row
        kb = [cache.data_ptr() + l * 2 * per_kv for l in range(L)]
        tgt = oc.PagedTarget(kb, [x + per_kv for x in kb], Bs * row, row, lay_t[2] * lay_t[3], Bs,
                             synth.block_table(r, need, need), 0)
        descs.append((oc.build_descriptor(store, keys, lay_t, tgt), cache))
    a = torch.randn(8192, 8192, dtype=torch.bfloat16, device=dev)
    b = torch.randn(8192, 8192, dtype=torch.bfloat16, device=dev)
    cbuf = torch.empty(8192, 8192, dtype=torch.bfloat16, device=dev)
    gs, fs = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
    n_gemm, n_fetch = 40, 200
    flops = 2 * 8192 ** 3

    def run(do_gemm, do_fetch, fopts):
        torch.cuda.synchronize()
        e = {k: torch.cuda.Event(enable_timing=True) for k in ("g0", "g1", "f0", "f1")}
        if do_gemm:
            e["g0"].record(gs)
            with torch.cuda.stream(gs):
                for _ in range(n_gemm):
                    torch.matmul(a, b, out=cbuf)
            e["g1"].record(gs)
        if do_fetch:
            e["f0"].record(fs)
            for i in range(n_fetch):
                descs[i % 2][0].fetch_layerwise(fs, **fopts)
            e["f1"].record(fs)
        torch.cuda.synchronize()
        res = {}
        if do_gemm:
            res["gemm_tflops"] = round(n_gemm * flops / e["g0"].elapsed_time(e["g1"]) / 1e9, 1)
        if do_fetch:
            res["fetch_GBps"] = round(n_fetch * 2 * N * S * L / e["f0"].elapsed_time(e["f1"]) / 1e6, 1)
        return res

    run(True, True, {})                                     # warm up cuBLAS and the fetch path
    out = {"gemm_alone": run(True, False, {})}
    for engine, name in ((oc.COPY_BULK, "bulk"), (oc.COPY_LDST, "ldst")):
        for mc in (0, 148, 64, 32, 16):
            fo = {"engine": engine, "max_ctas": mc, "unit_bytes": int(os.environ.get("OC_CORUN_UNIT", "0"))}
            alone = run(False, True, fo)
            both = run(True, True, fo)
            out[f"{name}_ctas{mc or 'auto'}"] = {"fetch_alone_GBps": alone["fetch_GBps"],
                                                 "fetch_corun_GBps": both["fetch_GBps"],
                                                 "gemm_corun_tflops": both["gemm_tflops"]}
    for d, _ in descs:
        d.close()
    store.close()
    del a, b, cbuf, descs
    torch.cuda.empty_cache()
    return out


def sweep_leg(args, oc, torch, dev, lay_t):
    """Fig. 15 analog: one request from the pinned host tier, paced at f * r*, with
    the Table A5 A100 compute windows; added TTFT against the resident-KV chain and against Eq. 3
    with uniform X = s/r, C = c (added = X + (L-1) max(0, X - C)).  The knee sits at f = 1."""
    import synth
    L, G, Bs = lay_t[0], lay_t[4], 16
    row, S, chunk = oc.geometry(lay_t)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(1000)
    e0.record()
    torch.cuda._sleep(20_000_000)
    e1.record()
    torch.cuda.synchronize()
    cyc_per_ms = 20_000_000 / e0.elapsed_time(e1)
    out = {}
    for ctx, hit in ((16384, 0.875), (65536, 0.875)):
        N = int(ctx * hit) // G
        c = TABLE_A5_T_TOTAL_MS[(ctx, hit)] / L / 1e3
        s = N * S
        rstar = s / c
        store = oc.Store(lay_t, capacity=N, tier=oc.TIER_PINNED_HOST, device=dev.index)
        (tok,), _ = synth.family_streams(31 + N, G, 0, [N])
        keys = oc.chunk_keys(tok, G)
        gen = torch.Generator(device=dev).manual_seed(N)
        for b0 in range(0, N, 512):
            pl = torch.randint(0, 256, (min(N, b0 + 512) - b0, chunk), dtype=torch.uint8, device=dev, generator=gen)
            store.put_chunks(keys[b0:b0 + pl.shape[0]], pl)
            del pl
        need = N * G // Bs
        cache = torch.empty((L, 2, need, Bs, row), dtype=torch.uint8, device=dev)
        per_kv = need * Bs * row
        kb = [cache.data_ptr() + l * 2 * per_kv for l in range(L)]
        tgt = oc.PagedTarget(kb, [x + per_kv for x in kb], Bs * row, row, lay_t[2] * lay_t[3], Bs,
                             synth.block_table(3, need, need), 0)
        d = oc.build_descriptor(store, keys, lay_t, tgt)
        copy_s, cons_s = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)

        def chain(pace):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            a.record(copy_s)
            cons_s.wait_event(a)
            if pace is not None:
                d.fetch_layerwise(copy_s, pace_Bps=pace)
            for l in range(L):
                if pace is not None:
                    d.wait_layer(l, cons_s)
                with torch.cuda.stream(cons_s):
                    torch.cuda._sleep(int(c * 1e3 * cyc_per_ms))
            b.record(cons_s)
            torch.cuda.synchronize()
            return a.elapsed_time(b)

        base = min(chain(None) for _ in range(2))
        pts = []
        for f in (0.25, 0.5, 0.75, 0.9, 1.0, 1.1, 1.25, 1.5, 2.0, 4.0):
            r = f * rstar
            added = chain(r) - base
            X = s / r
            pts.append({"f": f, "rate_GBps": round(r / 1e9, 3), "added_ms": round(added, 3),
                        "eq3_added_ms": round((X + (L - 1) * max(0.0, X - c)) * 1e3, 3)})
        out[f"{ctx // 1024}K,{hit:g}"] = {"r_star_GBps": round(rstar / 1e9, 3), "C_ms": round(c * 1e3, 3),
                                          "payload_per_layer_MiB": s / 2**20, "points": pts}
        d.close()
        store.close()
        del cache
        torch.cuda.empty_cache()
    return out


def batch_leg(args, oc, torch, dev, lay_t):
    """Config 5 on one GPU: concurrent mixed 4K/64K requests (Llama-3-8B layout) whose prefixes
    come from a few shared families (Zipf-like reuse), each delivered into its own paged cache.
    Compares one batched launch (layer-major across requests) with one launch per request on one
    stream and with one launch per request on its own stream.  GB/s = r+w bytes of all requests /
    device time; per-request X0 (layer-0 ready after the launch) summarises latency."""
    import synth
    n4, n64 = (int(x) for x in args.batch.lower().split("x"))
    L, G, Bs = lay_t[0], lay_t[4], 16
    row, S, chunk = oc.geometry(lay_t)
    fam4, fam64 = 4, 2
    N4, N64 = 4096 // G, 65536 // G
    store = oc.Store(lay_t, capacity=fam4 * N4 + fam64 * N64, tier=oc.TIER_HBM, device=dev.index)
    fam_keys = []
    gen = torch.Generator(device=dev).manual_seed(55)
    for f, n in [(f, N4) for f in range(fam4)] + [(fam4 + f, N64) for f in range(fam64)]:
        (tok,), _ = synth.family_streams(7000 + f, G, 0, [n])
        keys = oc.chunk_keys(tok, G)
        for b0 in range(0, n, 512):
            pl = torch.randint(0, 256, (min(n, b0 + 512) - b0, chunk), dtype=torch.uint8, device=dev, generator=gen)
            store.put_chunks(keys[b0:b0 + pl.shape[0]], pl)
            del pl
        fam_keys.append(keys)
    reqs = []
    for i in range(n4 + n64):
        big = i >= n4
        keys = fam_keys[fam4 + (i % fam64)] if big else fam_keys[i % fam4]
        n = keys.shape[0]
        need = n * G // Bs
        cache = torch.empty((L, 2, need, Bs, row), dtype=torch.uint8, device=dev)
        per_kv = need * Bs * row
        kb = [cache.data_ptr() + l * 2 * per_kv for l in range(L)]
        tgt = oc.PagedTarget(kb, [x + per_kv for x in kb], Bs * row, row, lay_t[2] * lay_t[3], Bs,
                             synth.block_table(100 + i, need, need), 0)
        reqs.append((oc.build_descriptor(store, keys, lay_t, tgt), cache, n))
    descs = [r[0] for r in reqs]
    total_bytes = sum(2 * n * S * L for _, _, n in reqs)
    batch = oc.Batch(descs)
    batch_pos = oc.Batch(descs, order=oc.BATCH_BY_POSITION)
    s0 = torch.cuda.Stream(device=dev)
    streams = [torch.cuda.Stream(device=dev) for _ in descs]

    def timed(fn, reps=3):
        best = None
        for _ in range(reps + 1):
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s0)
            fn(a)
            for st in streams:
                s0.wait_stream(st)
            b.record(s0)
            torch.cuda.synchronize()
            ms = a.elapsed_time(b)
            x0 = [float(t[1] - t[0]) / 1e6 for t in (d.layer_times().astype(np.int64) for d in descs)]
            if best is None or ms < best[0]:
                best = (ms, x0)
        return {"GBps": round(total_bytes / best[0] / 1e6, 1), "ms": round(best[0], 3),
                "x0_ms_4k_median": round(float(np.median(best[1][:n4])), 4) if n4 else None,
                "x0_ms_64k_median": round(float(np.median(best[1][n4:])), 4) if n64 else None}

    res = {"requests": f"{n4} x 4K + {n64} x 64K (families: {fam4} x 4K, {fam64} x 64K)",
           "bytes_rw": total_bytes,
           "batched_one_launch": timed(lambda a: batch.fetch(s0)),
           # position-major inside each layer: members sharing a family prefix read each shared
           # slice together (HBM once, L2 for the rest)
           "batched_by_position": timed(lambda a: batch_pos.fetch(s0)),
           # WDRR claim order (Alg. A2 line 7), weights = each request's bytes (equal finish times)
           "batched_wdrr_by_size": timed(lambda a: batch.fetch(s0, wdrr_weights=[float(n) for _, _, n in reqs])),
           "per_request_one_stream": timed(lambda a: [d.fetch_layerwise(s0) for d in descs]),
           "per_request_own_streams": timed(lambda a: [(st.wait_event(a), d.fetch_layerwise(st))
                                                       for d, st in zip(descs, streams)])}
    batch.close()
    batch_pos.close()
    for d, _, _ in reqs:
        d.close()
    del reqs
    store.close()
    torch.cuda.empty_cache()
    return res


def hash_leg(args, oc, torch, dev, G=16, ctx=4096):
    """Chain keys (reading c1) of R requests of 4K tokens (256 keys each): one GPU launch
    (oc_chunk_keys_batch, one thread per chain; device time from CUDA events around the launch
    alone) vs the host library's loop over oc_chunk_keys (SHA extensions, one core)."""
    import synth
    R = args.hash
    streams = [synth.tokens(77000 + i, ctx) for i in range(R)]
    t = time.perf_counter()
    for st in streams:
        oc.chunk_keys(st, G)
    host_s = time.perf_counter() - t
    flat = torch.from_numpy(np.concatenate(streams).view(np.int32)).to(dev)
    off = torch.from_numpy((np.arange(R, dtype=np.int64) * ctx)).to(dev)
    lens = torch.full((R,), ctx, dtype=torch.int64, device=dev)
    koff = torch.from_numpy(np.arange(R, dtype=np.int64) * (ctx // G)).to(dev)
    out = torch.empty((R * (ctx // G), 32), dtype=torch.uint8, device=dev)
    s = torch.cuda.Stream(device=dev)
    run = lambda: oc._check(oc._lib.oc_chunk_keys_batch(flat.data_ptr(), off.data_ptr(), lens.data_ptr(), R, G, None,
                                                       out.data_ptr(), koff.data_ptr(), s.cuda_stream))
    run()
    s.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    run()
    b.record(s)
    s.synchronize()
    gpu_ms = a.elapsed_time(b)
    same = bool(np.array_equal(out[:ctx // G].cpu().numpy(), oc.chunk_keys(streams[0], G)))
    keys = R * (ctx // G)
    return {"requests": R, "keys": keys, "host_ms": round(host_s * 1e3, 2), "gpu_ms": round(gpu_ms, 3),
            "host_keys_per_s": round(keys / host_s), "gpu_keys_per_s": round(keys / (gpu_ms / 1e3)),
            "first_request_equal": same}


def pool_leg(args, oc, torch, dev, lay_t, epoch_s=0.1, cap_gbps=50.0, delta_gbps=5.0):
    """Alg. A2 as a running system (Sec. 3.6): requests arrive over time (Poisson) and
    are submitted to an oc.TenantPool; every 100 ms (reading c16) the host calls pool.epoch(), which
    retires finished requests, admits the waiting ones under the cap the running ones leave (rates
    from the policy), and launches them -- as independently paced fetches, or as one WDRR batch per
    epoch with held rates.  Chunks live in the pinned-host tier (PCIe as the shared link); each
    request's consumer runs wait_layer(l) + a compute window c_i per layer (Table A5 windows).
    TTFT_i = end of its last window - its arrival, both stamped on the GPU clock; the no-limit TTFT
    is L * c_i.  Reported per (policy, dispatch): mean / p50 / p90 TTFT and the sum of added TTFT."""
    import synth
    GB = 1e9 / 8
    L, G, Bs = lay_t[0], lay_t[4], 16
    row, S, chunk = oc.geometry(lay_t)
    cells = [(16384, 0.5), (16384, 0.875), (32768, 0.5), (32768, 0.875), (65536, 0.5), (65536, 0.875)]
    R = args.pool
    rng = np.random.default_rng(2605)
    kinds = [cells[i % len(cells)] for i in rng.permutation(R)]
    bytes_total = sum(int(c * h) // G * S * L for c, h in kinds)
    mean_gap = bytes_total / (cap_gbps * GB) / R / 0.9      # offered load ~0.9 of the cap
    arrivals = np.cumsum(rng.exponential(mean_gap, R))
    arrivals -= arrivals[0]
    n_max = max(int(c * h) // G for c, h in kinds)
    store = oc.Store(lay_t, capacity=n_max, tier=oc.TIER_PINNED_HOST, device=dev.index)
    (tok,), _ = synth.family_streams(4343, G, 0, [n_max])
    keys = oc.chunk_keys(tok, G)
    gen = torch.Generator(device=dev).manual_seed(4343)
    for b0 in range(0, n_max, 128):
        b1 = min(n_max, b0 + 128)
        pl = torch.randint(0, 256, (b1 - b0, chunk), dtype=torch.uint8, device=dev, generator=gen)
        store.put_chunks(keys[b0:b0 + pl.shape[0]], pl)
        del pl
    caches = {}
    for c, h in set(kinds):                                  # one destination per kind, reused
        N = int(c * h) // G
        need = N * G // Bs
        cache = torch.empty((L, 2, need, Bs, row), dtype=torch.uint8, device=dev)
        per_kv = need * Bs * row
        kb = [cache.data_ptr() + l * 2 * per_kv for l in range(L)]
        caches[(c, h)] = (cache, oc.PagedTarget(kb, [x + per_kv for x in kb], Bs * row, row, lay_t[2] * lay_t[3],
                                                Bs, synth.block_table(N, need, need), 0))
    copy_streams = [torch.cuda.Stream(device=dev) for _ in range(R)]
    cons_streams = [torch.cuda.Stream(device=dev) for _ in range(R)]
    stamps = torch.zeros((R, L + 1, 2), dtype=torch.int64, device=dev)

    def run(policy, dispatch):
        pool = oc.TenantPool(policy, cap_gbps * GB, delta_gbps * GB, 0, dispatch=dispatch)
        torch.cuda.synchronize()
        descs, tickets, chained = [None] * R, [None] * R, [False] * R
        c_of = [TABLE_A5_T_TOTAL_MS[k] / L / 1e3 for k in kinds]
        t0 = time.perf_counter()
        nxt, next_epoch = 0, 0.0
        while True:
            now = time.perf_counter() - t0
            while nxt < R and arrivals[nxt] <= now:
                i = nxt
                c, h = kinds[i]
                N = int(c * h) // G
                descs[i] = oc.build_descriptor(store, keys[:N], lay_t, caches[(c, h)][1])
                oc.emulate_compute(0, cons_streams[i], stamps[i, 0])          # arrival stamp
                tickets[i] = pool.submit(descs[i], c_of[i], copy_streams[i])
                nxt += 1
            if now >= next_epoch:
                pool.epoch()
                next_epoch += epoch_s
                for i in range(nxt):
                    if not chained[i] and pool.status(tickets[i])[0] != oc.TENANT_WAITING:
                        for l in range(L):                    # prefill of layer l after its KV
                            descs[i].wait_layer(l, cons_streams[i])
                            oc.emulate_compute(int(c_of[i] * 1e9), cons_streams[i], stamps[i, 1 + l])
                        chained[i] = True
            if nxt == R and all(chained):
                break
            time.sleep(0.002)
        torch.cuda.synchronize()
        st = stamps.cpu().numpy().astype(np.int64)
        ttft = (st[:, L, 1] - st[:, 0, 0]) / 1e6
        base = np.array([L * c * 1e3 for c in c_of])
        pool.close()
        for d in descs:
            d.close()
        return {"ttft_ms_mean": round(float(ttft.mean()), 1), "ttft_ms_p50": round(float(np.median(ttft)), 1),
                "ttft_ms_p90": round(float(np.percentile(ttft, 90)), 1),
                "added_ms_sum": round(float((ttft - base).sum()), 1)}

    out = {"requests": R, "cap_gbps": cap_gbps, "delta_gbps": delta_gbps, "epoch_ms": epoch_s * 1e3,
           "offered_load_of_cap": 0.9, "mix": "Workload C cells (16K/32K/64K x 50%/87.5%), Table A5 windows",
           "runs": {}}
    for policy in ("equal", "stall_opt", "cal_stall_opt"):
        for dname, disp in (("independent", oc.DISPATCH_INDEPENDENT), ("wdrr", oc.DISPATCH_WDRR)):
            out["runs"][f"{policy}/{dname}"] = run(policy, disp)
    store.close()
    del caches
    torch.cuda.empty_cache()
    return out
