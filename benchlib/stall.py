"""Added TTFT (the metric's second half): timer-spin compute windows and real prefill compute."""
import json
import os
import statistics
import sys
import time

import numpy as np

from .common import (METRIC, N_CHUNKS_4K, ROTATE, TABLE_A5_T_TOTAL_MS, UNIT, ClockSampler, bench_config,  # noqa: F401
                     cores_used, dist_env, in_harness_copy, peaks, prefill_window_s, sched_workloads)


def stall_leg(args, oc, torch, dev, lay_t, fopts, cells=None, tiers=None, windows_sel=("a100", "b200"),
              timelines=True, optlocal=True):
    """Added TTFT of a prefix hit over per-layer compute windows (Eq. 3).

    The consumer stream waits on layer l (wait_layer), then runs the compute window C_l as a
    %globaltimer spin (oc.emulate_compute) that stamps its start/end on the clock of the fetch's
    layer-ready stamps.  TTFT runs from the fetch launch to the end of the last layer's compute
    (free-running copy stream, reading c14).  Baselines: (i) the same consumer chain, waits
    included, with the KV already delivered (resident KV); (ii) the paper's opt-local-LW analog
    (P:1000-1003): a pre-aggregated layer-major buffer copied contiguously layer by layer (one
    cudaMemcpyAsync + event per layer).  added = TTFT - TTFT(resident).  Per-layer device stalls:
    stall_0 = start_0 - launch, stall_l = start_l - end_(l-1), minus the resident chain's gaps.
    a8 check: the free-running recurrence start_l = max(ready_l, end_(l-1) + gap) with the
    measured ready_l, C_l and resident gaps predicts the measured last end."""
    import synth
    L, G, Bs = lay_t[0], lay_t[4], 16
    row, S, chunk = oc.geometry(lay_t)
    stamps = torch.zeros((L, 2), dtype=torch.int64, device=dev)
    cur = {"fo": fopts}                            # fetch options of the tier being measured

    def chain(copy_s, cons_s, d, C_ns, fetch=True, events=None):
        """Returns (TTFT ms from the launch event, stamps [L,2] ns)."""
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record(copy_s)
        cons_s.wait_event(a)
        if d is not None and fetch:
            d.fetch_layerwise(copy_s, **cur["fo"])
        elif events is not None:
            events(copy_s)
        for l in range(L):
            if d is not None:
                d.wait_layer(l, cons_s)
            elif events is not None:
                cons_s.wait_event(events.ev[l])
            oc.emulate_compute(C_ns, cons_s, stamps[l])
        b.record(cons_s)
        torch.cuda.synchronize()
        return a.elapsed_time(b), stamps.cpu().numpy().copy()

    res = {"timelines": {}}
    if cells is None:
        cells = [("4k", 4096, 3584, 63.47)] + ([("64k", 65536, 57344, 2423.90)] if args.stall64k else [])
    if tiers is None:
        tiers = (("hbm", oc.TIER_HBM), ("pinned_host", oc.TIER_PINNED_HOST), ("pinned_host_ce", oc.TIER_PINNED_HOST),
                 ("pinned_host_hot1", oc.TIER_PINNED_HOST))
    for name, ctx, cached, t_total_ms in cells:
        N = cached // G
        windows = {"a100": t_total_ms / L if t_total_ms else None,             # Table A5 (A100)
                   "b200": prefill_window_s("llama3-8b", ctx, cached / ctx) * 1e3}  # FLOP model
        windows = {k: v for k, v in windows.items() if k in windows_sel and v is not None}
        need = N * G // Bs
        cache = torch.empty((L, 2, need, Bs, row), dtype=torch.uint8, device=dev)
        per_kv = need * Bs * row
        kb = [cache.data_ptr() + l * 2 * per_kv for l in range(L)]
        bt = synth.block_table(5, need, need)
        tgt = oc.PagedTarget(kb, [x + per_kv for x in kb], Bs * row, row, lay_t[2] * lay_t[3], Bs, bt, 0)
        copy_s, cons_s = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
        for tier_name, tier in tiers:
            cur["fo"] = {"engine": oc.COPY_CE} if tier_name.endswith("_ce") else fopts
            store = oc.Store(lay_t, capacity=N, tier=tier, device=dev.index)
            if tier_name.endswith("_hot1"):            # layer 0 of every chunk mirrored in HBM
                store.set_hot_layers(1)
            (tok,), _ = synth.family_streams(9000 + N, G, 0, [N])
            keys = oc.chunk_keys(tok, G)
            gen = torch.Generator(device=dev).manual_seed(N)
            for b0 in range(0, N, 512):
                pl = torch.randint(0, 256, (min(N, b0 + 512) - b0, chunk), dtype=torch.uint8, device=dev,
                                   generator=gen)
                store.put_chunks(keys[b0:b0 + pl.shape[0]], pl)
                del pl
            d = oc.build_descriptor(store, keys, lay_t, tgt)
            d_cw = oc.build_descriptor(store, keys, lay_t, tgt, oc.DELIVER_CHUNK_MAJOR)
            ol = None
            if optlocal:
                # opt-local-LW analog: layer-major pre-aggregated source [L][N*S] on the same tier
                src = torch.empty((L, N * S), dtype=torch.uint8, device=dev) if tier == oc.TIER_HBM else \
                    torch.empty((L, N * S), dtype=torch.uint8, pin_memory=True)
                dst = torch.empty((L, N * S), dtype=torch.uint8, device=dev)

                class _OL:
                    ev = [torch.cuda.Event() for _ in range(L)]

                    def __call__(self, s):
                        with torch.cuda.stream(s):
                            for l in range(L):
                                dst[l].copy_(src[l], non_blocking=True)
                                self.ev[l].record(s)
                ol = _OL()
            for wname, C_ms in windows.items():
                C_ns = int(round(C_ms * 1e6))
                d.fetch_layerwise(copy_s, **cur["fo"])
                torch.cuda.synchronize()
                base_runs = [chain(copy_s, cons_s, d, C_ns, fetch=False) for _ in range(3)]
                base, bst = min(base_runs, key=lambda r: r[0])
                gaps = (bst[1:, 0] - bst[:-1, 1]).astype(np.float64)       # resident-chain gap between windows
                gap_ns = float(np.median(gaps))
                runs = []
                for it in range(3):
                    ttft, st = chain(copy_s, cons_s, d, C_ns)
                    t = d.layer_times().astype(np.int64)
                    runs.append((ttft - base, ttft, t, st))
                best = min(runs, key=lambda r: r[0])
                _, ttft, t, st = best
                ready = t[1:] - t[0]
                start, end = st[:, 0] - t[0], st[:, 1] - t[0]
                stall = np.empty(L)
                stall[0] = start[0]
                stall[1:] = start[1:] - end[:-1] - gap_ns
                # a8 free-running recurrence with the measured ready_l, C_l and resident gaps
                e_prev = None
                for l in range(L):
                    s_l = ready[l] if e_prev is None else max(ready[l], e_prev + gap_ns)
                    e_prev = s_l + (end[l] - start[l])
                cw = min(chain(copy_s, cons_s, d_cw, C_ns)[0] for _ in range(2)) - base
                key = f"{name}_{tier_name}" + ("" if wname == "a100" else "_b200win")
                cell = {"N": N, "window": wname, "C_ms_per_layer": round(C_ms, 4), "added_ms": round(best[0], 4),
                        "added_per_layer_ms": round(best[0] / L, 5),
                        "X0_ms": round(ready[0] / 1e6, 4), "transfer_ms": round(ready[-1] / 1e6, 4),
                        "ttft_ms": round(ttft, 3), "baseline_ttft_ms": round(base, 3),
                        "resident_gap_us": round(gap_ns / 1e3, 2),
                        "device_stall_ms": {"layer0": round(stall[0] / 1e6, 4),
                                            "layers_1_to_L-1": round(float(stall[1:].sum()) / 1e6, 4),
                                            "max_layer": round(float(stall[1:].max()) / 1e6, 4) if L > 1 else 0.0},
                        "a8_model_end_ms": round(e_prev / 1e6, 4), "measured_end_ms": round(end[-1] / 1e6, 4),
                        "added_ms_chunkwise": round(cw, 4), "payload_MiB": N * S * L / 2**20}
                if ol is not None:
                    ol(copy_s)
                    torch.cuda.synchronize()
                    cell["added_ms_opt_local_lw"] = round(min(chain(copy_s, cons_s, None, C_ns, events=ol)[0]
                                                              for _ in range(2)) - base, 4)
                res[key] = cell
                if timelines and name == "4k":  # per-layer device timeline (the overlap evidence)
                    res["timelines"][key] = {"layer_ready_ms": [round(x / 1e6, 4) for x in ready],
                                             "compute_start_ms": [round(x / 1e6, 4) for x in start],
                                             "compute_end_ms": [round(x / 1e6, 4) for x in end]}
            d_cw.close()
            d.close()
            store.close()
            del ol
            torch.cuda.empty_cache()
        del cache
        torch.cuda.empty_cache()
    res["windows"] = ("a100: Table A5 per-layer compute (P:2706-2713); b200: FLOP model at half the measured "
                      "sustained bf16 rate; %globaltimer spin (oc.emulate_compute); baseline = the same chain "
                      "(waits included) with the KV already delivered; opt_local_lw = pre-aggregated layer-major "
                      "buffer on the same tier, one contiguous copy + event per layer; times relative to the "
                      "fetch kernel's start")
    return res


def stall_gemm_leg(args, oc, torch, dev, lay_t):
    """Added TTFT with real prefill compute sharing the GPU ("a shape-true Llama
    layer (random bf16 weights; only shapes matter) over the miss tokens").  Per layer the consumer
    stream waits for the layer's KV (wait_layer) and then runs the layer's prefill over the m miss
    tokens: the QKV projection (4096x6144), attention of the m queries over the h fetched hit tokens
    -- read straight from the paged cache the fetch just filled (all hit keys are visible to every
    query, so their block order does not matter) -- plus causal attention over the m new tokens
    (flash-attn, GQA 32/8 heads; the two partial outputs are summed, not LSE-merged: timing shape
    only), the O projection (4096x4096), gate+up (4096x28672) and down (14336x4096) GEMMs.

    Timing: CUDA events after every layer on the consumer stream, from an event on the copy stream
    just before the fetch launch.  Each measurement is a PAIR run back to back on the same streams:
    the chain with the fetch, and the same chain on resident KV without waits; added = the
    difference.  `pairs` pairs per variant; median, min, max reported.
      added_ms       at the last layer (TTFT)
      added_settled  at the end of the first layer whose compute ends after the fetch's last layer
                     was announced, plus one: from there on the two chains run the same kernels on
                     the same resident KV, so later layers add only the compute's own run-to-run
                     noise (at 64K, +-1 ms over 688 ms) -- the low-noise estimate of the same
                     quantity
    Decomposition (medians): X0 (the fetch's first-layer announcement after its start, device
    stamps), waits (the same consumer chain on a descriptor whose layers are all announced: the
    wait_layer calls alone), contention = added_settled - X0 - waits (the copy's SM and HBM use
    slowing the co-running prefill).

    Variants of the HBM-tier fetch: full_gpu (default launch: the fetch holds every SM until it is
    done), per_layer (one launch + event per layer), yield (OC_FETCH_YIELD: layer 0 with the whole
    GPU, then one unit per CTA so the prefill's kernels take SMs back as copy CTAs retire) with the
    copy stream at low and the consumer at high priority (yield_prio) or both at default priority,
    and gated_u32k (oc_fetch_layers: layers 0-1 at once, layer l+2 requested on a highest-priority
    stream after the consumer's attention of layer l, so it runs beside the MLP GEMMs)."""
    import synth
    from flash_attn import flash_attn_func
    L, G, Bs = lay_t[0], lay_t[4], 16
    n_kv, d_h = lay_t[1], lay_t[2]
    row, S, chunk = oc.geometry(lay_t)
    w = [torch.randn(k, n, dtype=torch.bfloat16, device=dev) * 0.01
         for k, n in ((4096, 6144), (4096, 4096), (4096, 28672), (14336, 4096))]
    out = {"model": "llama3-8b layer: QKV, flash attention over the fetched hit KV + causal over the miss "
                    "tokens, O, gate+up, down (random bf16 weights)",
           "method": "paired chains (fetch, resident-no-wait) back to back; CUDA events per layer on the consumer "
                     "stream; median over pairs"}
    cells = [("4k", 4096, 11)] + ([("64k", 65536, 5)] if getattr(args, "stall64k", 1) else [])
    keep = set(getattr(args, "stall_gemm_cells", "4k,64k").split(","))
    cells = [c for c in cells if c[0] in keep]
    for name, ctx, pairs in cells:
        cached = ctx * 7 // 8
        m = ctx - cached
        N = cached // G
        x = torch.randn(m, 4096, dtype=torch.bfloat16, device=dev)
        need = N * G // Bs
        cache = torch.zeros((L, 2, need, Bs, row), dtype=torch.uint8, device=dev)
        kvb = cache.view(torch.bfloat16).view(L, 2, need * Bs, n_kv, d_h)
        per_kv = need * Bs * row
        kb = [cache.data_ptr() + l * 2 * per_kv for l in range(L)]
        tgt = oc.PagedTarget(kb, [x_ + per_kv for x_ in kb], Bs * row, row, lay_t[2] * lay_t[3], Bs,
                             synth.block_table(7, need, need), 0)
        copy_s, cons_s = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
        lo_s, hi_s = torch.cuda.Stream(device=dev, priority=0), torch.cuda.Stream(device=dev, priority=-1)

        gate_s = torch.cuda.Stream(device=dev, priority=-2)   # clamped to the device's highest priority

        def layer_compute(l, after_attn=None):
            qkv = torch.matmul(x, w[0])
            q = qkv[:, :4096].view(1, m, 32, d_h)
            kn = qkv[:, 4096:5120].view(1, m, n_kv, d_h)
            vn = qkv[:, 5120:].view(1, m, n_kv, d_h)
            a_hit = flash_attn_func(q, kvb[l, 0].unsqueeze(0), kvb[l, 1].unsqueeze(0), causal=False)
            a_new = flash_attn_func(q, kn, vn, causal=True)
            if after_attn is not None:
                after_attn(l)
            torch.matmul((a_hit + a_new).view(m, 4096), w[1])
            gu = torch.matmul(x, w[2])
            torch.matmul(gu[:, :14336], w[3])

        def chain(d, fopts, cs, ks, waits=True):
            """Per-layer end times (ms after the launch event) of one consumer chain."""
            torch.cuda.synchronize()
            a0 = torch.cuda.Event(enable_timing=True)
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(L)]
            a0.record(cs)
            ks.wait_event(a0)
            hook = None
            if fopts is not None and "gated" in fopts:
                # co-run schedule through oc_fetch_layers: the first k0 layers at once with the whole
                # GPU; layer l + k0 on a highest-priority stream gated on the consumer's attention of
                # layer l, so it runs beside layer l's MLP GEMMs (lean CTAs fit beside a GEMM CTA)
                g = dict(fopts["gated"])
                k0 = g.pop("k0")
                gs = cs if g.pop("low", False) else gate_s
                d.fetch_layers(0, k0, cs, unit_bytes=g.get("unit_bytes", 0))

                def hook(l):
                    if l + k0 < L:
                        e = torch.cuda.Event()
                        e.record(ks)
                        gs.wait_event(e)
                        d.fetch_layers(l + k0, l + k0 + 1, gs, **g)
            elif fopts is not None:
                d.fetch_layerwise(cs, **fopts)
            with torch.cuda.stream(ks):
                for l in range(L):
                    if d is not None and waits:
                        d.wait_layer(l, ks)
                    layer_compute(l, hook)
                    ev[l].record(ks)
            torch.cuda.synchronize()
            return np.array([a0.elapsed_time(e) for e in ev])

        def med(v):
            v = sorted(v)
            return {"median": round(statistics.median(v), 4), "min": round(v[0], 4), "max": round(v[-1], 4)}

        chain(None, None, copy_s, cons_s)
        base0 = chain(None, None, copy_s, cons_s)
        res = {"miss_tokens": m, "hit_chunks": N, "pairs": pairs, "compute_ms_resident": round(float(base0[-1]), 3),
               "compute_ms_per_layer": round(float(base0[-1]) / L, 4),
               "r_star_GBps": round(N * S / (float(base0[-1]) / L / 1e3) / 1e9, 1)}
        tiers = [("hbm", oc.TIER_HBM, (("full_gpu", {"engine": oc.COPY_BULK}, None),
                                       ("per_layer", {"mode": oc.FETCH_PER_LAYER}, None),
                                       ("yield", {"engine": oc.COPY_BULK, "yield_sms": True}, None),
                                       ("yield_prio", {"engine": oc.COPY_BULK, "yield_sms": True}, (lo_s, hi_s)),
                                       # finer units: smaller copy CTAs, more of them per SM in a tail
                                       ("yield_prio_u16k", {"engine": oc.COPY_BULK, "yield_sms": True,
                                                            "unit_bytes": 16384}, (lo_s, hi_s)),
                                       ("yield_prio_u8k", {"engine": oc.COPY_BULK, "yield_sms": True,
                                                           "unit_bytes": 8192}, (lo_s, hi_s)),
                                       # the co-run schedule through oc_fetch_layers (measured worse:
                                       # profiles/r02_stall_gemm_gated.json)
                                       ("gated_u32k", {"gated": {"k0": 2, "engine": oc.COPY_BULK, "max_ctas": 148,
                                                                 "unit_bytes": 32768}}, None),
                                       # the same gating on a LOW-priority copy stream with one unit per
                                       # CTA: layer l+2's copy waits for layer l's attention to end, then
                                       # fills the SMs the O/MLP GEMMs leave free
                                       ("gated_low_yield", {"gated": {"k0": 2, "engine": oc.COPY_BULK,
                                                                      "yield_sms": True, "low": True}},
                                        (lo_s, hi_s))))]
        sel = [v for v in getattr(args, "stall_gemm_variants", "").split(",") if v]
        if sel:
            tiers = [(tn, t, tuple(v for v in vs if v[0] in sel)) for tn, t, vs in tiers]
        if not getattr(args, "stall_gemm_hbm_only", False):
            tiers += [("pinned_host", oc.TIER_PINNED_HOST, (("sm", {"engine": oc.COPY_BULK}, None),
                                                            ("ce", {"engine": oc.COPY_CE}, None)))]
        for tier_name, tier, variants in tiers:
            store = oc.Store(lay_t, capacity=N, tier=tier, device=dev.index)
            (tok,), _ = synth.family_streams(9100 + N, G, 0, [N])
            keys = oc.chunk_keys(tok, G)
            for b0 in range(0, N, 512):
                pl = torch.randint(0, 256, (min(N, b0 + 512) - b0, chunk), dtype=torch.uint8, device=dev)
                store.put_chunks(keys[b0:b0 + pl.shape[0]], pl)
                del pl
            d = oc.build_descriptor(store, keys, lay_t, tgt)
            if tier == oc.TIER_HBM:
                # the waits alone: every layer already announced when the chain is enqueued
                d.fetch_layerwise(copy_s)
                torch.cuda.synchronize()
                wv = []
                for _ in range(pairs):
                    b_ = chain(None, None, copy_s, cons_s)
                    wv.append(float(chain(d, None, copy_s, cons_s)[-1] - b_[-1]))
                res["waits_only_ms"] = med(wv)
            for vname, fopts, streams in variants:
                cs, ks = streams if streams else (copy_s, cons_s)
                chain(d, fopts, cs, ks)
                added, settled, x0, span = [], [], [], []
                for _ in range(pairs):
                    b_ = chain(None, None, cs, ks)
                    f_ = chain(d, fopts, cs, ks)
                    t_ = d.layer_times().astype(np.int64)
                    span_ms = (t_[L] - t_[0]) / 1e6
                    k = int(np.searchsorted(b_, span_ms, side="right"))   # first layer ending after it
                    k = min(k + 1, L - 1)
                    added.append(float(f_[-1] - b_[-1]))
                    settled.append(float(f_[k] - b_[k]))
                    x0.append((t_[1] - t_[0]) / 1e6)
                    span.append(span_ms)
                cell = {"added_ms": med(added), "added_settled_ms": med(settled),
                        "X0_ms": round(statistics.median(x0), 4), "fetch_span_ms": round(statistics.median(span), 3)}
                if tier == oc.TIER_HBM:
                    cell["decomposition_ms"] = {
                        "X0": cell["X0_ms"], "waits": res["waits_only_ms"]["median"],
                        "contention": round(statistics.median(settled) - cell["X0_ms"] - res["waits_only_ms"]["median"], 4)}
                res[f"{tier_name}_{vname}"] = cell
            d.close()
            store.close()
        out[name] = res
        del cache, kvb
        torch.cuda.empty_cache()
    return out
