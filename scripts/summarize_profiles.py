"""Summaries of ncu captures for profiles/ (development script).

Usage:
  python scripts/summarize_profiles.py launches <launches.csv>          # per-kernel shares
  python scripts/summarize_profiles.py rep <report.ncu-rep> [...]        # key metrics
  python scripts/summarize_profiles.py traffic <metrics.csv> <out.json> <algo_bytes_per_launch>
      # per-launch DRAM bytes of the GEMM launches of one step (ncu --metrics
      # gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum -k regex:gemm_kernel)
"""
import json
import collections
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size",
        "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "l1tex__throughput.avg.pct_of_peak_sustained_active"]


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    agg = collections.defaultdict(lambda: [0, 0.0])
    for d in data:
        name = d["Kernel Name"].split("(")[0].replace("void ", "")
        us = float(d["Metric Value"].replace(",", "")) * scale[d["Metric Unit"]]
        agg[name][0] += 1
        agg[name][1] += us
    tot = sum(v[1] for v in agg.values())
    print(f"{len(data)} launches, {tot / 1e3:.3f} ms summed (cold-cache, serialised by ncu)")
    print(f"{'kernel':40s} {'launches':>8s} {'sum ms':>9s} {'avg us':>8s} {'share':>7s}")
    for k, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k:40s} {n:8d} {us / 1e3:9.3f} {us / n:8.2f} {us / tot:7.1%}")


def rep(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    hdr, units = r[0], r[1]
    for vals in r[2:]:
        name = vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        print(f"{path}: {name}")
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                print(f"  {k:64s} {vals[i]:>14s} {units[i]}")


def traffic(path, out, algo):
    rows = list(csv.reader(open(path)))
    hdr, per = None, collections.defaultdict(dict)
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            v = float(d["Metric Value"].replace(",", ""))
            unit = d["Metric Unit"]
            mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6,
                    "ns": 1e-9, "nsecond": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3}.get(unit, 1)
            per[d["ID"]][d["Metric Name"]] = v * mult
    n = len(per)
    rd = sum(x.get("dram__bytes_read.sum", 0) for x in per.values())
    wr = sum(x.get("dram__bytes_write.sum", 0) for x in per.values())
    t = sum(x.get("gpu__time_duration.sum", 0) for x in per.values())
    res = {"launches": n, "dram_bytes_per_gemm_launch": (rd + wr) / max(n, 1),
           "dram_read_bytes": rd, "dram_write_bytes": wr, "ncu_time_s": t,
           "algorithmic_bytes_per_gemm_launch": float(algo),
           "traffic_over_algorithmic": (rd + wr) / max(n, 1) / float(algo) if float(algo) else None,
           "source": path, "note": "ncu, --clock-control none, each launch replayed cold and serialised"}
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    if sys.argv[1] == "traffic":
        traffic(sys.argv[2], sys.argv[3], sys.argv[4])
    elif sys.argv[1] == "launches":
        launches(sys.argv[2])
    else:
        for p in sys.argv[2:]:
            rep(p)
