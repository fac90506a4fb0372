"""The reference arm of this tier: the oracle (tests-only CPU code, oracle/) timed on host cores --
`bench.py --impl reference` and the `cpu_baseline` objects.  The only bench code that executes oracle/."""
import json
import os
import statistics
import sys
import time

import numpy as np

from .common import (METRIC, N_CHUNKS_4K, ROTATE, TABLE_A5_T_TOTAL_MS, UNIT, ClockSampler, bench_config,  # noqa: F401
                     cores_used, dist_env, in_harness_copy, peaks, prefill_window_s, sched_workloads)


# ---- the reference arm: the oracle, timed on host cores ---------------------------------------------
class OracleWorkload:
    """The oracle's Alg. A1 gather + paged scatter on one seeded request (setup untimed)."""

    def __init__(self, seed, n_chunks, lay):
        import synth
        from oracle import keys as okeys
        from oracle.descriptor import PagedTarget, build_descriptor
        from oracle.geometry import chunk_bytes, chunk_layer_bytes, row_bytes, head_bytes
        from oracle.store import ChunkStore
        G = lay.chunk_tokens
        (t,), (ids,) = synth.family_streams(seed, G, 0, [n_chunks])
        keys = okeys.chunk_keys(t, G)
        self.st = ChunkStore(lay)
        self.st.put(keys, synth.payloads(seed, ids, chunk_bytes(lay)))
        row, self.S, Bs = row_bytes(lay), chunk_layer_bytes(lay), 16
        need = -(-n_chunks * G // Bs)
        pool = need + need // 4
        bt = synth.block_table(seed, need, pool).tolist()
        per_kv = pool * Bs * row
        k = [l * 2 * per_kv for l in range(lay.num_layers)]
        tgt = PagedTarget(k, [x + per_kv for x in k], Bs * row, row, head_bytes(lay), Bs, bt, 0)
        self.dst = synth.sentinel(lay.num_layers * 2 * per_kv)
        self.desc = build_descriptor(self.st, keys, lay, tgt)
        self.n = n_chunks

    def run(self, layers):
        """Returns (algorithmic read+write bytes, seconds)."""
        from oracle.assemble import gather_layer, scatter_paged
        t0 = time.perf_counter()
        for l in layers:
            scatter_paged(gather_layer(self.st, self.desc, l), l, self.desc, self.dst)
        return 2 * self.n * self.S * len(layers), time.perf_counter() - t0


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    import synth
    from oracle.geometry import Layout
    lay = Layout(*synth.LLAMA3_8B.as_tuple())
    # one step = one layer of the full 4K request (N = 256 chunks: 16 MiB read + 16 MiB written)
    wl = OracleWorkload(1, N_CHUNKS_4K, lay)
    for i in range(args.warmup):
        wl.run([i % lay.num_layers])
    tot_b, tot_s = 0, 0.0
    for i in range(args.steps):
        b, s = wl.run([i % lay.num_layers])
        tot_b += b
        tot_s += s
    v = tot_b / tot_s / 1e9
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": tot_s / args.steps * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": bench_config(args, synth.LLAMA3_8B.as_tuple(), ws),
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle",
                         "sample": f"{args.steps} steps, each one layer of the 4K request (256 chunks, G=16, "
                                   "Bs=16): Alg. A1 gather + paged scatter, single-threaded numpy"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def cpu_baseline_leg():
    import synth
    from oracle.geometry import Layout
    lay = Layout(*synth.LLAMA3_8B.as_tuple())
    wl = OracleWorkload(1, N_CHUNKS_4K, lay)
    layers = []
    tot_b, tot_s = 0, 0.0
    l = 0
    while tot_s < 10.0 and l < lay.num_layers:
        b, s = wl.run([l])
        tot_b += b
        tot_s += s
        layers.append(l)
        l += 1
    c, ncpu = cores_used()
    return {"value": tot_b / tot_s / 1e9, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"{len(layers)} of 32 layers of the 4K request (N=256, G=16, Bs=16), "
                      f"{tot_s:.1f} s, single-threaded Python+numpy (host has {ncpu} cpus, affinity {c})"}


def cpu_config3_leg():
    """The oracle on one layer of the config-3 request (N = 4096 chunks, 256 MiB per layer): the
    per-layer work depends on N and S only, so the layout is truncated to one layer to keep the
    host copy of the store at 256 MiB instead of 8 GiB."""
    import synth
    from oracle.geometry import Layout
    L8 = synth.LLAMA3_8B.as_tuple()
    wl = OracleWorkload(3, 4096, Layout(1, *L8[1:]))
    b, t = wl.run([0])
    c, ncpu = cores_used()
    return {"value": round(b / t / 1e9, 3), "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"1 layer of the 64K request (N=4096, 512 MiB read+write), {t:.1f} s, single-threaded "
                      f"Python+numpy (host has {ncpu} cpus, affinity {c})"}
