"""Summarise ncu captures into the committed evidence files under profiles/.

  python profiles/summarize.py full  <report.ncu-rep> <out.json> [algorithmic_bytes_per_launch]
  python profiles/summarize.py launches <launches.csv> <out.json>

`full` keeps the DRAM bytes, throughput, occupancy and stall-reason sample counts of the captured
launch; `launches` aggregates the per-launch device times of an ncu launch list by kernel name
(cold-cache, serialised: compare shares, not absolutes).
"""
import csv
import io
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__bytes_read.sum.per_second",
        "dram__bytes_write.sum.per_second", "launch__grid_size", "launch__block_size",
        "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum", "l1tex__t_bytes.sum",
        "sm__cycles_elapsed.avg.per_second", "dram__cycles_elapsed.avg.per_second"]

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1,
         "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1, "byte/s": 1, "Kbyte/s": 1e3,
         "Mbyte/s": 1e6, "Gbyte/s": 1e9, "Tbyte/s": 1e12, "cycle/s": 1, "Kcycle/s": 1e3, "Mcycle/s": 1e6,
         "Gcycle/s": 1e9}


def raw(report):
    out = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def kernel_src_sha16():
    """Hash of the fetch kernel's sources: bench.py reports the committed traffic as stale when the
    kernel changed after the capture."""
    import hashlib
    import os
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    h = hashlib.sha256()
    for f in ("fetch_kernels.cuh", "fetch.cu", "oc_internal.h"):
        with open(os.path.join(root, "paper_2605_22850_b200", "csrc", f), "rb") as fh:
            h.update(fh.read())
    return h.hexdigest()[:16]


def full(report, dst, algo_bytes=None):
    hdr, units, launches = raw(report)
    res = []
    for vals in launches:
        rec = {"kernel": vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else None}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                v = vals[i].replace(",", "")
                try:
                    rec[k] = float(v) * SCALE.get(units[i], 1)
                except ValueError:
                    rec[k] = v
        stalls = {}
        for i, h in enumerate(hdr):
            if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
                try:
                    n = float(vals[i].replace(",", ""))
                except ValueError:
                    continue
                if n > 0:
                    stalls[h.replace("smsp__pcsamp_warps_issue_stalled_", "")] = n
        rec["stall_samples"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1]))
        traffic = rec.get("dram__bytes_read.sum", 0) + rec.get("dram__bytes_write.sum", 0)
        rec["dram_bytes_per_launch"] = traffic
        if algo_bytes:
            rec["algorithmic_bytes_per_launch"] = algo_bytes
            rec["traffic_over_algorithmic"] = traffic / algo_bytes
            rec["achieved_GBps_under_ncu"] = algo_bytes / rec["gpu__time_duration.sum"] / 1e9
        res.append(rec)
    summary = {"report": report, "launches": res,
               "dram_bytes_per_launch": res[0]["dram_bytes_per_launch"] if res else None,
               "kernel_src_sha16": kernel_src_sha16()}
    with open(dst, "w") as f:
        json.dump(summary, f, indent=1)
    return summary


def launches(path, dst):
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    rows = list(csv.DictReader(lines))
    agg = {}
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0]
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "nsecond")
        v *= SCALE.get(unit, 1e-9)
        a = agg.setdefault(name, {"launches": 0, "total_s": 0.0})
        a["launches"] += 1
        a["total_s"] += v
    tot = sum(a["total_s"] for a in agg.values()) or 1.0
    for a in agg.values():
        a["share"] = a["total_s"] / tot
        a["mean_us"] = a["total_s"] / a["launches"] * 1e6
    out = {"source": path, "kernels": dict(sorted(agg.items(), key=lambda kv: -kv[1]["total_s"]))}
    with open(dst, "w") as f:
        json.dump(out, f, indent=1)
    return out


if __name__ == "__main__":
    if sys.argv[1] == "full":
        print(json.dumps(full(sys.argv[2], sys.argv[3], float(sys.argv[4]) if len(sys.argv) > 4 else None), indent=1))
    else:
        print(json.dumps(launches(sys.argv[2], sys.argv[3]), indent=1))
