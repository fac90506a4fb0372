"""Benchmark of the ObjectCache hot path on B200 (contract: one JSON line on rank 0).

Workload (BASELINE.json configs[1]): Llama-3-8B KV layout (32 layers, 8 KV heads, d = 128, bf16),
one request per step with a 4K-token prefix hit (N = 256 chunks of G = 16 tokens), delivered into
a fragmented vLLM-style paged cache (Bs = 16, NHD): the layer-major gather + paged scatter of all
32 layers (Alg. A1), announced layer by layer; details in benchlib/headline.py.

  value         read + write HBM bytes (2*N*S*L per step) / device time of the timed region, whole
                job (every rank fetches its own requests: weak scaling), max over ranks
  roofline      the fetch kernel (fetch_bulk_kernel<0>): the same bytes / the copy stream's span
                over the K launches, vs MEASURED_PEAKS.json hbm_gbs
  e2e           the same metric through the public C-ABI calls from HOST buffers: the chunk store in
                pinned host memory (match -> build -> fetch, the payload crossing PCIe -> wait -> D2H
                of the layer stamps), with the PCIe payload rate against an in-harness H2D copy;
                `e2e.hbm_tier`: the same call order with the HBM store, pipelined (control-plane
                cost against the device `value`)
  cpu_baseline  the oracle (tests-only CPU code) on a bounded sample, 1 core
  legs          stall (added TTFT at 4K/64K), config3 (64K hit, verified), config5 (mixed requests
                over the job's GPUs, strong scaling, NVLink peer reads, verified); optional legs by flag

--impl reference runs the oracle itself as the reference arm (rank 0 only).
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from benchlib.common import METRIC, UNIT, bench_config, dist_env  # noqa: E402


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=200)
    p.add_argument("--warmup", type=int, default=10)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--mode", default="persistent", choices=["persistent", "per_layer"])
    p.add_argument("--engine", default="bulk", choices=["bulk", "ldst"])
    p.add_argument("--no-overlap", action="store_true", help="headline launches in plain stream order "
                   "(no OC_FETCH_OVERLAP)")
    p.add_argument("--no-stall", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-config3", action="store_true", help="skip BASELINE config 3 (64K-token hit, 8 GiB)")
    p.add_argument("--no-config5", action="store_true", help="skip config 5 (mixed requests over the job's GPUs)")
    p.add_argument("--stall64k", type=int, default=1)
    p.add_argument("--profile", action="store_true", help="headline only, no soak / clock sampling (ncu runs)")
    p.add_argument("--stall-gemm", action="store_true", help="added TTFT with real prefill (GEMMs + attention)")
    p.add_argument("--stall-gemm-hbm-only", action="store_true")
    p.add_argument("--stall-gemm-cells", default="4k,64k", help="comma list of stall-gemm cells (4k, 64k)")
    p.add_argument("--stall-gemm-variants", default="", help="comma list of HBM-tier variants (default: all)")
    p.add_argument("--sched", default="", help="comma list of scheduler workloads (A,B,C,70B; 70B = config 4)")
    p.add_argument("--corun", action="store_true")
    p.add_argument("--granularity", action="store_true", help="G = 16/64/256 and the unfused flow")
    p.add_argument("--serve", type=int, default=0, help="old weak-scaling serving leg with this many requests")
    p.add_argument("--offload", action="store_true")
    p.add_argument("--p2p", action="store_true")
    p.add_argument("--sensitivity", action="store_true")
    p.add_argument("--crossover", action="store_true")
    p.add_argument("--sweep", action="store_true")
    p.add_argument("--pool", type=int, default=0)
    p.add_argument("--hash", type=int, default=0)
    p.add_argument("--batch", default="")
    return p.parse_args()


def main_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2605_22850_b200 as oc
    import synth
    from benchlib import configs, e2e, extra, headline, reference, stall

    ws, rank, local = dist_env()
    # OC_BENCH_DIST_BACKEND=gloo lets several ranks share one GPU to exercise the N>1 code path
    # (NCCL refuses duplicate GPUs); real multi-GPU runs use NCCL with one GPU per rank.
    backend = os.environ.get("OC_BENCH_DIST_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count()) if backend != "nccl" else local
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    lay_t = synth.LLAMA3_8B.as_tuple()
    head = headline.run(args, oc, torch, dev, lay_t, ws, rank, dist, backend)
    out = {
        "metric": METRIC, "value": head["value"], "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": head["ms_per_step"], "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u8", "data": "synthetic (seeded PCG64 chunk bytes, Llama-3 vocab tokens)",
        "config": dict(bench_config(args, lay_t, ws), launch=head["launch"]),
        "gpu_launches": head["gpu_launches"], "roofline": head["roofline"], "clocks": head["clocks"],
        "kernel": {k: head[k] for k in ("isolated_launch_us", "X0_us_isolated", "in_harness_copy", "verified")},
    }
    legs = {}
    if not args.no_e2e and not args.profile:
        # the contract's e2e: HOST buffers (pinned-host chunk store, the payload crosses PCIe every
        # step); next to it the HBM-tier serving call order (control-plane cost vs the device rate)
        e = e2e.pcie_tier(args, oc, torch, dev, lay_t, {"engine": oc.COPY_CE}, ws, backend)
        hb = e2e.hbm_tier(args, oc, torch, dev, lay_t, ws, rank, dist, backend)
        if rank == 0:
            hb["frac_of_value"] = round(hb["value"] / head["value"], 4)
            e["hbm_tier"] = hb
            out["e2e"] = e
    if rank == 0 and not args.no_stall and not args.profile:
        legs["stall"] = stall.stall_leg(args, oc, torch, dev, lay_t, {"engine": oc.COPY_BULK},
                                        tiers=(("hbm", oc.TIER_HBM), ("pinned_host", oc.TIER_PINNED_HOST),
                                               ("pinned_host_ce", oc.TIER_PINNED_HOST)), timelines=False)
    if rank == 0 and not args.no_config3 and not args.profile:
        legs["config3"] = configs.config3_leg(args, oc, torch, dev, lay_t)
    if rank == 0 and args.stall_gemm:
        legs["stall_gemm"] = stall.stall_gemm_leg(args, oc, torch, dev, lay_t)
    if rank == 0 and args.sched:
        legs["sched"] = configs.sched_leg(args, oc, torch, dev, lay_t)
    fopts = {"engine": oc.COPY_BULK}
    for flag, name, fn in (("corun", "corun", lambda: extra.corun_leg(args, oc, torch, dev, lay_t)),
                           ("granularity", "granularity", lambda: extra.granularity_leg(args, oc, torch, dev, lay_t, fopts)),
                           ("offload", "offload", lambda: extra.offload_leg(args, oc, torch, dev, lay_t)),
                           ("sensitivity", "sensitivity", lambda: extra.sensitivity_leg(args, oc, torch, dev, lay_t)),
                           ("crossover", "crossover", lambda: extra.crossover_leg(args, oc, torch, dev, lay_t, fopts)),
                           ("sweep", "sweep", lambda: extra.sweep_leg(args, oc, torch, dev, lay_t)),
                           ("pool", "pool", lambda: extra.pool_leg(args, oc, torch, dev, lay_t)),
                           ("hash", "hash", lambda: extra.hash_leg(args, oc, torch, dev)),
                           ("batch", "batch", lambda: extra.batch_leg(args, oc, torch, dev, lay_t))):
        if rank == 0 and getattr(args, flag):
            legs[name] = fn()
    if ws > 1 and args.p2p:
        res = extra.p2p_leg(args, oc, torch, dev, lay_t, ws, rank, backend)
        if rank == 0:
            legs["p2p"] = res
    if args.serve:
        res = extra.serve_leg(args, oc, torch, dev, lay_t, ws, rank, backend)
        if rank == 0:
            legs["serve"] = res
    if not args.no_config5 and not args.profile:
        # a child process group per job (own port): a fault there cannot take this line with it
        from benchlib import config5
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
        if ws > 1:
            dist.barrier()
        res = config5.spawn(ws, rank, local)
        if ws > 1:
            dist.barrier()
        if rank == 0:
            legs["config5"] = res
    if rank == 0 and ws == 1 and not args.no_cpu_baseline and not args.profile:
        out["cpu_baseline"] = reference.cpu_baseline_leg()
        if "config3" in legs:   # the oracle's GB/s next to the GPU's for config 3 too
            legs["config3"]["oracle_cpu"] = reference.cpu_config3_leg()
    if legs:
        out["legs"] = legs
    if ws > 1:
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(out), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        from benchlib.reference import run_reference
        run_reference(args)
    else:
        main_ours(args)


if __name__ == "__main__":
    main()
