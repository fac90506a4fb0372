"""Shared helpers of the benchmark legs: the metric, peaks, the clock sampler, the in-harness copy
reference, rank environment, and the compute-window models (Table A5 windows, FLOP model)."""
import json
import os
import statistics
import subprocess
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

METRIC = "layerwise KV gather+scatter GB/s vs HBM peak; added per-layer stall ms at 4K/64K"


UNIT = "GB/s"


N_CHUNKS_4K = 256


ROTATE = 4


# The paper's scheduler workloads (Sec. 5.7; Table A6): requests named
# by (context, hit rate); per-layer bytes s_i = cached tokens * 4096 B and per-layer compute
# c_i = T_total / 32 from Table A5 (A100); caps 80 / 50 / 50 Gbps; delta = 5 Gbps.
TABLE_A5_T_TOTAL_MS = {(4096, 0.5): 185.31, (4096, 0.875): 63.47, (16384, 0.5): 955.89, (16384, 0.875): 281.76, (32768, 0.5): 2589.25,
                       (32768, 0.875): 763.19, (65536, 0.5): 8672.79, (65536, 0.875): 2423.90}


# ---- shared helpers ---------------------------------------------------------------------------------
def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, burst copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def kernel_src_sha16():
    import hashlib
    h = hashlib.sha256()
    for f in ("fetch_kernels.cuh", "fetch.cu", "oc_internal.h"):
        with open(os.path.join(ROOT, "paper_2605_22850_b200", "csrc", f), "rb") as fh:
            h.update(fh.read())
    return h.hexdigest()[:16]


def ncu_traffic():
    """(dram bytes per launch of the dominant kernel from the committed ncu --set full summary, whether
    that capture is of the current kernel sources); (None, False) without a capture."""
    path = os.path.join(ROOT, "profiles", "ncu_full_summary.json")
    try:
        with open(path) as f:
            s = json.load(f)
        return s.get("dram_bytes_per_launch"), s.get("kernel_src_sha16") == kernel_src_sha16()
    except Exception:
        return None, False


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 50 ms while running."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.Q,
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm = [float(r[0]) for r in self.rows if len(r) >= 7 and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) >= 7 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows if len(r) >= 7 for i in range(4)
                          if r[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(sm)}


def in_harness_copy(torch, dev, stream, nbytes):
    """Read+write GB/s of a plain device-to-device copy_ of nbytes (the MEASURED_PEAKS method, run
    in this process under this run's clocks)."""
    src = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    dst = torch.empty_like(src)
    ts = []
    with torch.cuda.stream(stream):
        src.fill_(1)
        for i in range(23):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            dst.copy_(src)
            b.record(stream)
            if i >= 3:
                ts.append((a, b))
    stream.synchronize()
    ms = statistics.median(a.elapsed_time(b) for a, b in ts)
    del src, dst
    torch.cuda.empty_cache()
    return 2 * nbytes / (ms / 1e3) / 1e9


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def cores_used():
    try:
        return len(os.sched_getaffinity(0)), os.cpu_count()
    except Exception:
        return 1, os.cpu_count()


def bench_config(args, lay_t, ws):
    """The N=1 workload (BASELINE configs[1]) -- shared by both arms so their lines compare."""
    L, G, Bs = lay_t[0], lay_t[4], 16
    return {"workload": "llama3-8b KV layout, single request, 4K-token prefix hit (N=256 x G=16), "
                        "paged NHD cache Bs=16 fragmented",
            "layout": {"L": L, "n_kv": lay_t[1], "d": lay_t[2], "p": lay_t[3], "G": G, "Bs": Bs},
            "fetch_mode": args.mode, "engine": args.engine, "tier": "hbm",
            "store_slots": "random slab positions (the rotating requests' chunks put in one seeded interleaving)",
            "l2": f"inputs larger than L2: {ROTATE} rotating request sets, "
                  f"{ROTATE * 2 * N_CHUNKS_4K * 2 * G * lay_t[1] * lay_t[2] * lay_t[3] * L / 2**30:.1f} GiB "
                  "touched per rotation",
            "parallelism": f"replicas x{ws} (independent requests per GPU, no collective)"}


def prefill_window_s(lay_name, ctx, hit, flops_per_s=0.5 * 1399.5e12):
    """Per-layer prefill compute exposed by the miss tokens (SURVEY 8(d) sanity model): with m
    miss tokens after h hit tokens a layer costs 2*m*P_layer + 4*n_heads*d*m*(h + m/2) FLOPs;
    executed at half of the measured sustained bf16 rate (MEASURED_PEAKS.json)."""
    h_d, n_heads, d, n_kv, inter = {"llama3-70b": (8192, 64, 128, 8, 28672),
                                   "llama3-8b": (4096, 32, 128, 8, 14336)}[lay_name]
    p_layer = 2 * h_d * h_d + 2 * h_d * n_kv * d + 3 * h_d * inter
    h = ctx * hit
    m = ctx - h
    return (2 * m * p_layer + 4 * n_heads * d * m * (h + m / 2)) / flops_per_s


def sched_workloads():
    """name -> (layout, cap Gbps, [(label, context, hit, c seconds per layer)], window source)."""
    import synth
    a5 = lambda ctx, hit: TABLE_A5_T_TOTAL_MS[(ctx, hit)] / 32 / 1e3
    cells = lambda lst: [(f"{c // 1024}K,{h:g}", c, h, a5(c, h)) for c, h in lst]
    ab = [(16384, 0.5), (16384, 0.875), (65536, 0.5), (65536, 0.875)]
    w = {"A": (synth.LLAMA3_8B, 80.0, cells(ab), "Table A5 (A100)"),
         "B": (synth.LLAMA3_8B, 50.0, cells(ab), "Table A5 (A100)"),
         "C": (synth.LLAMA3_8B, 50.0, cells(ab[:2] + [(32768, 0.5), (32768, 0.875)] + ab[2:]), "Table A5 (A100)")}
    # BASELINE.json configs[3]: Llama-3-70B layout, 16 concurrent 32K requests (hit 50% / 87.5%
    # alternating), cap at half the aggregate zero-stall rate (Workload B/C regime).
    c70 = [(f"32K,{h:g}#{i}", 32768, h, prefill_window_s("llama3-70b", 32768, h))
           for i, h in enumerate([0.5, 0.875] * 8)]
    sum_rstar = sum(int(ctx * h) * 4096 / c for _, ctx, h, c in c70)
    w["70B"] = (synth.LLAMA3_70B, round(sum_rstar / 2 * 8 / 1e9, 3), c70,
                "FLOP model at 50% of the measured sustained bf16 rate (B200)")
    return w
