"""BASELINE config 5: Llama-3-8B layout, concurrent mixed 4K / 64K requests over
1/2/4/8 GPUs with NVLink P2P reads of chunks homed on another GPU.  STRONG scaling: the corpus and
the request set are the same at every N; only their placement changes.

Corpus   16 prefix families of 4K tokens (256 chunks, 512 MiB each) + 2 of 64K tokens (4096 chunks,
         8 GiB each) = 24 GiB of synth chunk payloads; family g is homed on rank g mod N (its
         chunks live in that GPU's HBM store).
Requests 128, from synth.serving_requests (4K/64K 50/50, family by Zipf(1.1), hit 50% or 87.5%);
         request q is served by its family's home rank with probability p_aff = 0.875, otherwise by
         a uniformly drawn rank (seeded per request) -- then its chunks are read from the peer GPU
         inside the same fetch kernel (store handles exchanged once over CUDA IPC, attached as
         peers).  No collective on the data path.
Serving  per rank: a bounded paged pool (40 GiB of [L][2][blocks][Bs][row]), FIFO admission by
         free blocks, 8 copy streams, blocks returned when a fetch's completion event fires.
Timing   device time from a common start event to the last completion, max over ranks;
         GB/s = 2*N*S*L summed over all requests / that time (aggregate), / N per GPU.
Remote   remote_byte_fraction = bytes of requests served off their family's home / all bytes;
         NVLink ingress per GPU = the payload those requests read (N*S*L each) / the time, against
         an in-harness cudaMemcpyPeer-style copy of 1 GiB from the next rank's slab (copy engine).
Verified a second, identical pass checks every request on completion: all per-layer digests
         against the oracle (benchlib.verify); rank 0 also checks one 4K request in full and one
         64K request's first and last layers byte for byte.
Batched  `batched_by_position`: the same passes with each admission step's requests (at most 16)
         fetched as one position-major batch (oc.BATCH_BY_POSITION: prefix-family members read
         their shared chunks together), timed and digest-verified the same way.

Run as `python -m benchlib.config5` under the bench's rank environment (bench.py spawns one child
per rank on its own port, so a fault here cannot take the contract line with it); rank 0 prints
one JSON object.
"""
import collections
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

N_SHORT, N_LONG = 16, 2
R_REQUESTS = 128
P_AFF = 0.875
POOL_GIB = 40
BATCH_MAX = 16


def route(reqs, ws, home_of, seed=5):
    """Serving rank of every request: the family's home with probability P_AFF, else uniform."""
    out = []
    for q, (long, fam, _) in enumerate(reqs):
        rng = np.random.Generator(np.random.PCG64([seed, 0xA77, q]))
        out.append(home_of(long, fam) if rng.random() < P_AFF or ws == 1 else int(rng.integers(0, ws)))
    return out


def main():
    if os.environ.get("OC_HANG_DUMP_S"):               # debugging support: stacks of a stuck rank
        import faulthandler
        faulthandler.dump_traceback_later(float(os.environ["OC_HANG_DUMP_S"]), exit=True)
    import torch
    import torch.distributed as dist

    import paper_2605_22850_b200 as oc
    import synth
    from paper_2605_22850_b200 import dist as odist
    from benchlib import verify
    from oracle.geometry import Layout

    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # OC_BENCH_DIST_BACKEND=gloo: several ranks share one GPU (the N>1 code path on a one-GPU box;
    # NCCL refuses duplicate GPUs); peer stores are then IPC-imported from the same device
    backend = os.environ.get("OC_BENCH_DIST_BACKEND", "nccl")
    if backend != "nccl":
        local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    comm = {"world_size": ws, "backend": None}
    if ws > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
        comm = {"world_size": dist.get_world_size(), "backend": dist.get_backend()}
        if backend == "nccl":
            comm["nccl_version"] = ".".join(str(x) for x in torch.cuda.nccl.version())
        else:
            comm["peers_share_one_gpu"] = True
    lay_t = synth.LLAMA3_8B.as_tuple()
    L, G, Bs = lay_t[0], lay_t[4], 16
    row, S, chunk = oc.geometry(lay_t)
    n_short, n_long = 4096 // G, 65536 // G
    home_of = lambda long, f: (f + N_SHORT * int(long)) % ws
    fam_seed = lambda long, f: 8000 + 100 * int(long) + f
    fams = {}
    for long, nf, n in ((False, N_SHORT, n_short), (True, N_LONG, n_long)):
        for f in range(nf):
            (tok,), (ids,) = synth.family_streams(fam_seed(long, f), G, 0, [n])
            fams[(long, f)] = {"keys": oc.chunk_keys(tok, G), "ids": ids, "seed": fam_seed(long, f)}
    mine = [k for k in fams if home_of(*k) == rank]
    cap = max(1, sum(len(fams[k]["ids"]) for k in mine))
    store = oc.Store(lay_t, capacity=cap, tier=oc.TIER_HBM, device=local)
    t0 = time.perf_counter()
    for k in mine:
        verify.fill_store([store], fams[k]["keys"], fams[k]["seed"], fams[k]["ids"], chunk)
    fill_s = time.perf_counter() - t0
    peers = []
    p2p_GBps = None
    if ws > 1:                                     # setup only: exchange store handles, attach peers
        torch.cuda.synchronize()
        blobs = odist.exchange_blobs(store.export())
        for r, blob in enumerate(blobs):
            if r != rank:
                p = oc.Store.import_(blob, device=local)
                store.attach_peer(p)
                peers.append((r, p))
        # in-harness NVLink reference: copy-engine copy of 1 GiB of the next rank's slab
        from cuda.bindings import runtime as cudart
        nxt = dict(peers)[(rank + 1) % ws]
        pbase, pbytes = nxt.slab
        nb = int(min(pbytes, 1 << 30))
        scratch = torch.empty(nb, dtype=torch.uint8, device=dev)
        s = torch.cuda.Stream(device=dev)
        best = 0.0
        for _ in range(3):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            err, = cudart.cudaMemcpyAsync(scratch.data_ptr(), pbase, nb, cudart.cudaMemcpyKind.cudaMemcpyDefault,
                                          s.cuda_stream)
            b.record(s)
            s.synchronize()
            if err == cudart.cudaError_t.cudaSuccess:
                best = max(best, nb / a.elapsed_time(b) / 1e6)
        p2p_GBps = best
        del scratch
        dist.barrier()
    pool_blocks = (POOL_GIB << 30) // (L * 2 * Bs * row)
    cache = torch.empty((L, 2, pool_blocks, Bs, row), dtype=torch.uint8, device=dev)
    per_kv = pool_blocks * Bs * row
    kb = [cache.data_ptr() + l * 2 * per_kv for l in range(L)]
    vb = [x + per_kv for x in kb]
    reqs_all = synth.serving_requests(5, R_REQUESTS, N_SHORT, N_LONG)
    served_by = route(reqs_all, ws, home_of)
    reqs = [(q, lg, f, h) for q, ((lg, f, h), r) in enumerate(zip(reqs_all, served_by)) if r == rank]
    n_of = lambda lg, h: int((65536 if lg else 4096) * h) // G
    remote_bytes = sum(2 * n_of(lg, h) * S * L for _, lg, f, h in reqs if home_of(lg, f) != rank)
    streams = [torch.cuda.Stream(device=dev) for _ in range(8)]
    start = torch.cuda.Event(enable_timing=True)
    T = verify.digest_table(S)
    T_dev = torch.from_numpy(T.view(np.int64)).to(dev)
    checks = {"digest_requests": 0, "digest_ok": 0, "full": {}}
    expect = {}

    def check_member(d, blocks, q, lg, f, n):
        idx = verify.slot_index(torch, dev, blocks, n * G, Bs)
        got = verify.gpu_digests(torch, cache, idx, n, G, T_dev)
        checks["digest_requests"] += 1
        checks["digest_ok"] += int(np.array_equal(got, expect[(lg, f)].request(n)))
        if rank == 0 and ("short" if not lg else "long") not in checks["full"]:
            fam = fams[(lg, f)]
            layers = range(L) if not lg else (0, L - 1)
            ok, nbytes, t_or, _ = verify.full_check(torch, Layout(*lay_t), fam["seed"], fam["keys"][:n],
                                                    fam["ids"][:n], cache, idx, layers)
            checks["full"]["short" if not lg else "long"] = {
                "request": q, "layers": len(layers), "bit_exact": ok, "bytes": nbytes, "oracle_s": round(t_or, 2)}

    def run(check=False, batch=0):
        """One pass over this rank's requests.  batch = 0: one fetch_layerwise per request (8 copy
        streams); batch = B > 0: the requests admitted in one admission step (at most B) are fetched
        as ONE position-major batch (oc.BATCH_BY_POSITION), so members of one prefix family read
        their shared chunks together; blocks return when the whole batch completes."""
        free = collections.deque(int(b) for b in synth.block_table(3, pool_blocks, pool_blocks))
        pending = collections.deque(reqs)
        inflight = []                               # (event, Batch or None, members)
        total, n_launch = 0, 0
        torch.cuda.synchronize()
        if ws > 1:
            dist.barrier()
        start.record(streams[0])
        for s in streams[1:]:
            s.wait_event(start)
        ends = []
        t_host = time.perf_counter()
        while pending or inflight:
            still = []
            for ev, bt_, members in inflight:
                if ev.query():
                    for m in members:
                        if check:
                            check_member(*m)
                        free.extend(m[1])
                    if bt_ is not None:
                        bt_.close()
                    for m in members:
                        m[0].close()
                else:
                    still.append((ev, bt_, members))
            inflight = still
            step, admitted = [], False
            while pending and (batch == 0 or len(step) < batch):
                q, lg, f, h = pending[0]
                n = n_of(lg, h)
                need = n * G // Bs
                if len(free) < need:
                    break
                pending.popleft()
                blocks = [free.popleft() for _ in range(need)]
                tgt = oc.PagedTarget(kb, vb, Bs * row, row, lay_t[2] * lay_t[3], Bs, np.asarray(blocks, np.int32), 0)
                d = oc.build_descriptor(store, fams[(lg, f)]["keys"][:n], lay_t, tgt)
                total += 2 * n * S * L
                admitted = True
                if batch == 0:
                    s = streams[q % len(streams)]
                    d.fetch_layerwise(s)
                    ev = torch.cuda.Event(enable_timing=True)
                    ev.record(s)
                    ends.append(ev)
                    inflight.append((ev, None, [(d, blocks, q, lg, f, n)]))
                else:
                    step.append((d, blocks, q, lg, f, n))
            if step:
                bt_ = oc.Batch([m[0] for m in step], order=oc.BATCH_BY_POSITION)
                s = streams[n_launch % len(streams)]
                n_launch += 1
                bt_.fetch(s)
                ev = torch.cuda.Event(enable_timing=True)
                ev.record(s)
                ends.append(ev)
                inflight.append((ev, bt_, step))
            if not admitted:
                if inflight:
                    inflight[0][0].synchronize()
                elif pending:
                    raise RuntimeError("config5: a request needs more blocks than the pool holds")
        torch.cuda.synchronize()
        host_s = time.perf_counter() - t_host
        dev_ms = max((start.elapsed_time(e) for e in ends), default=0.0)
        return total, dev_ms, host_s

    run()                                           # warm-up pass
    total, dev_ms, host_s = run()                   # timed pass
    red = dev if backend == "nccl" else "cpu"
    max_ms = odist.max_over_ranks(dev_ms, device=red)
    all_bytes = odist.sum_over_ranks(total, device=red)
    per_rank = [odist.sum_over_ranks(total if r == rank else 0, device=red) for r in range(ws)]  # load balance
    all_remote = odist.sum_over_ranks(remote_bytes, device=red)
    # verification pass: the oracle's digests of every family prefix this rank's requests use
    t0 = time.perf_counter()
    need_n = collections.defaultdict(int)
    for _, lg, f, h in reqs:
        need_n[(lg, f)] = max(need_n[(lg, f)], n_of(lg, h))
    oracle_bytes = 0
    for k, n in need_n.items():
        expect[k] = verify.FamilyDigests(fams[k]["seed"], fams[k]["ids"], n, L, S, T)
        oracle_bytes += expect[k].bytes
    t_oracle = time.perf_counter() - t0
    run(check=True)
    ok_all = odist.sum_over_ranks(checks["digest_ok"], device=red)
    n_all = odist.sum_over_ranks(checks["digest_requests"], device=red)
    # the same requests with each admission step fetched as one position-major batch (at most
    # BATCH_MAX members; profiles/r01_serve.json swept 4..64 and found 16 best), timed, then verified
    run(batch=BATCH_MAX)                            # warm-up pass
    _, dev_ms_b, _ = run(batch=BATCH_MAX)
    max_ms_b = odist.max_over_ranks(dev_ms_b, device=red)
    c_ok, c_n = checks["digest_ok"], checks["digest_requests"]
    run(check=True, batch=BATCH_MAX)
    ok_b = odist.sum_over_ranks(checks["digest_ok"] - c_ok, device=red)
    n_b = odist.sum_over_ranks(checks["digest_requests"] - c_n, device=red)
    t_oracle_max = odist.max_over_ranks(t_oracle, device=red)
    oracle_bytes_all = odist.sum_over_ranks(oracle_bytes, device=red)
    if ws > 1:
        dist.barrier()                              # peers' fetches done before any store goes away
    res = {"workload": (f"llama3-8b layout, {R_REQUESTS} requests over {N_SHORT} x 4K + {N_LONG} x 64K prefix "
                        f"families (24 GiB corpus, family g homed on rank g mod N), 4K/64K 50/50, Zipf(1.1), hit "
                        f"50%/87.5%, p_aff {P_AFF}; the same corpus and requests at every N (strong scaling)"),
           "n_gpus": ws, "comm": comm,
           "requests_per_rank_rank0": len(reqs), "bytes_rw": all_bytes,
           "bytes_rw_per_rank": per_rank,
           "busiest_rank_share": round(max(per_rank) / all_bytes, 4) if all_bytes else None,
           "GBps_aggregate": round(all_bytes / max_ms / 1e6, 1),
           "GBps_per_gpu": round(all_bytes / max_ms / 1e6 / ws, 1),
           "device_ms_max_over_ranks": round(max_ms, 2),
           "remote_byte_fraction": round(all_remote / all_bytes, 4) if all_bytes else 0.0,
           "nvlink_ingress_GBps_per_gpu": round(all_remote / 2 / ws / max_ms / 1e6, 1) if ws > 1 else 0.0,
           "p2p_copy_GBps_rank0": round(p2p_GBps, 1) if p2p_GBps else None,
           "pool_GiB_per_gpu": POOL_GIB, "corpus_fill_s_rank0": round(fill_s, 1),
           "verified": {"requests_digest_equal": int(ok_all), "requests": int(n_all),
                        "all_layers_all_requests": int(ok_all) == int(n_all) and n_all > 0,
                        "rank0_full": checks["full"],
                        "oracle_digest_s_max_over_ranks": round(t_oracle_max, 1),
                        "oracle_s_per_verified_GB": round(t_oracle_max * ws / (oracle_bytes_all / 1e9), 3)
                        if oracle_bytes_all else None}}
    res["batched_by_position"] = {
        "max_members": BATCH_MAX, "GBps_aggregate": round(all_bytes / max_ms_b / 1e6, 1),
        "GBps_per_gpu": round(all_bytes / max_ms_b / 1e6 / ws, 1), "device_ms_max_over_ranks": round(max_ms_b, 2),
        "note": "algorithmic bytes (2*N*S*L per request) as above; members of one prefix family read shared chunks "
                "once, so this is delivered bandwidth, not DRAM traffic",
        "verified": {"requests_digest_equal": int(ok_b), "requests": int(n_b),
                     "all_layers_all_requests": int(ok_b) == int(n_b) and n_b > 0}}
    if ws > 1 and p2p_GBps:
        res["nvlink_ingress_frac_of_p2p_copy"] = round(res["nvlink_ingress_GBps_per_gpu"] / p2p_GBps, 3)
    del cache
    store.close()
    for _, p in peers:
        p.close()
    if ws > 1:
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(res), flush=True)


def spawn(ws, rank, local, timeout=420):
    """Run this leg as a child process of a bench rank (its own process group on MASTER_PORT + 17).
    Returns the parsed JSON (rank 0) or {"error": ...}."""
    import subprocess
    # Not inherited: torchrun's TORCHELASTIC_* variables -- TORCHELASTIC_USE_AGENT_STORE makes the
    # child's env:// rendezvous connect to an agent store on the new port that nobody serves (a hang
    # until the timeout, seen with two ranks).
    base = {k: v for k, v in os.environ.items() if not k.startswith("TORCHELASTIC_")}
    env = dict(base, WORLD_SIZE=str(ws), RANK=str(rank), LOCAL_RANK=str(local),
               MASTER_ADDR=os.environ.get("MASTER_ADDR", "127.0.0.1"),
               MASTER_PORT=str(int(os.environ.get("MASTER_PORT", "29500")) + 17))
    try:
        p = subprocess.run([sys.executable, "-m", "benchlib.config5"], cwd=ROOT, env=env, capture_output=True,
                           text=True, timeout=timeout)
    except subprocess.TimeoutExpired:
        return {"error": f"timeout after {timeout} s"}
    if p.returncode != 0:
        return {"error": f"rc={p.returncode}: " + (p.stderr or "")[-600:]}
    if rank != 0:
        return None
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    return json.loads(lines[-1]) if lines else {"error": "no output: " + (p.stderr or "")[-400:]}


if __name__ == "__main__":
    main()
