"""Summarise ncu evidence into profiles/.

    python tools/summarize_ncu.py --full REP.ncu-rep[:WORKLOAD] [...] --launches LAUNCHES.csv --tag r1

Writes profiles/ncu_summary_<tag>.md (per-launch duration, DRAM bytes, DRAM
GB/s and % of the measured HBM peak, SM/L1 throughput, registers, occupancy)
and profiles/ncu_traffic.json, plus a share-of-step table from the
gpu__time_duration launch list.  A report tagged with a bench workload is
expected to hold every launch of ONE step of that workload (bench.py
--steps 1 --warmup 0 under ncu); its per-kernel DRAM bytes averaged over the
step's launches are stored under ncu_traffic.json[workload][kernel] and read
by bench.py as roofline.traffic (comparable to alg_bytes_per_launch, which is
averaged over the same launches).
"""

import argparse
import collections
import csv
import io
import json
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__grid_size", "launch__block_size",
           "l1tex__throughput.avg.pct_of_peak_sustained_active"]


def short(name):
    m = re.search(r"(\w+_kernel)<([^>]*)>", name) or re.search(r"(\w+_kernel)", name)
    if not m:
        return name[:40]
    return f"{m.group(1)}<{m.group(2)}>" if m.lastindex and m.lastindex > 1 else m.group(1)


def to_bytes(v, unit):
    f = float(v)
    return f * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit, 1)


def to_ms(v, unit):
    f = float(v)
    return f * {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1, "ms": 1,
                "second": 1e3, "s": 1e3}[unit]


def full_rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(METRICS)],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        ms = to_ms(d["gpu__time_duration.sum"], u["gpu__time_duration.sum"])
        rd = to_bytes(d["dram__bytes_read.sum"], u["dram__bytes_read.sum"])
        wr = to_bytes(d["dram__bytes_write.sum"], u["dram__bytes_write.sum"])
        res.append({"kernel": short(d["Kernel Name"]), "ms": ms, "dram_read": rd, "dram_write": wr,
                    "dram_gbs": (rd + wr) / (ms * 1e-3) / 1e9 if ms else 0,
                    "mem_pct": float(d["gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed"]),
                    "sm_pct": float(d["sm__throughput.avg.pct_of_peak_sustained_elapsed"]),
                    "l1_pct": float(d["l1tex__throughput.avg.pct_of_peak_sustained_active"]),
                    "regs": int(float(d["launch__registers_per_thread"])),
                    "warps_active_pct": float(d["sm__warps_active.avg.pct_of_peak_sustained_active"]),
                    "grid": d["launch__grid_size"], "block": d["launch__block_size"], "report": os.path.basename(rep)})
    return res


def traffic_rows(rep):
    """(kernel, ms, dram bytes) per launch of a report that holds only
    gpu__time_duration.sum and the two dram__bytes metrics (the 2^32 / 2^31
    headline steps: a --set full capture replays every 16 GiB launch ~40x)."""
    m = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum"]
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(m)],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        res.append({"kernel": short(d["Kernel Name"]), "ms": to_ms(d[m[0]], u[m[0]]),
                    "dram_read": to_bytes(d[m[1]], u[m[1]]), "dram_write": to_bytes(d[m[2]], u[m[2]])})
    return res


def launch_rows(path):
    txt = open(path).read()
    i = txt.find('"ID"')
    rows = list(csv.reader(io.StringIO(txt[i:])))
    hdr = rows[0]
    agg = collections.OrderedDict()
    for r in rows[1:]:
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        k = short(d["Kernel Name"])
        ms = to_ms(d["Metric Value"].replace(",", ""), d["Metric Unit"])
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += ms
    return agg


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--full", nargs="*", default=[])
    ap.add_argument("--traffic", nargs="*", default=[], help="REP:WORKLOAD reports with time + DRAM bytes only")
    ap.add_argument("--launches", default=None)
    ap.add_argument("--tag", default="r1")
    ap.add_argument("--note", default="")
    a = ap.parse_args()
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    lines = [f"# ncu summary ({a.tag})", "", a.note, "",
             f"HBM peak for the % column: {peak} GB/s (MEASURED_PEAKS.json, measured).", ""]
    traffic = {}
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        traffic = json.load(open(tpath))
        traffic = {k: v for k, v in traffic.items() if isinstance(v, dict)}  # drop the old flat format
    if a.full:
        lines += ["## `ncu --set full --clock-control none` (cold, serialised launches)", "",
                  "| report | kernel | grid x block | regs | ms | DRAM read GB | DRAM write GB | DRAM GB/s | % of HBM peak "
                  "| mem-pipe % | SM % | L1 % | warps active % |",
                  "|---|---|---|---|---|---|---|---|---|---|---|---|---|"]
        for spec in a.full:
            rep, _, wl = spec.partition(":")
            acc = {}
            for r in full_rows(rep):
                lines.append(f"| {r['report']} | `{r['kernel']}` | {r['grid']}x{r['block']} | {r['regs']} | "
                             f"{r['ms']:.3f} | {r['dram_read']/1e9:.3f} | {r['dram_write']/1e9:.3f} | "
                             f"{r['dram_gbs']:.0f} | {100*r['dram_gbs']/peak:.1f} | {r['mem_pct']:.1f} | "
                             f"{r['sm_pct']:.1f} | {r['l1_pct']:.1f} | {r['warps_active_pct']:.1f} |")
                base = r["kernel"].split("<")[0]
                a_ = acc.setdefault(base, [0, 0.0, 0.0])
                a_[0] += 1
                a_[1] += r["dram_read"] + r["dram_write"]
                a_[2] += r["ms"]
            if wl:
                traffic[wl] = {k: {"bytes_per_launch": v[1] / v[0], "launches": v[0], "ms_per_launch": v[2] / v[0]}
                               for k, v in acc.items()}
        lines.append("")
    if a.traffic:
        lines += ["## DRAM bytes per launch of the headline steps (`--metrics gpu__time_duration.sum,"
                  "dram__bytes_read.sum,dram__bytes_write.sum`)", "",
                  "| workload | kernel | launches | ms / launch | DRAM read GB / launch | DRAM write GB / launch | DRAM GB/s "
                  "| % of HBM peak |", "|---|---|---|---|---|---|---|---|"]
        for spec in a.traffic:
            rep, _, wl = spec.partition(":")
            acc = collections.OrderedDict()
            for r in traffic_rows(rep):
                base = r["kernel"].split("<")[0]
                a_ = acc.setdefault(base, [0, 0.0, 0.0, 0.0])
                a_[0] += 1
                a_[1] += r["dram_read"]
                a_[2] += r["dram_write"]
                a_[3] += r["ms"]
            for k, v in acc.items():
                gbs = (v[1] + v[2]) / (v[3] * 1e-3) / 1e9 if v[3] else 0
                lines.append(f"| {wl} | `{k}` | {v[0]} | {v[3]/v[0]:.3f} | {v[1]/v[0]/1e9:.3f} | {v[2]/v[0]/1e9:.3f} | "
                             f"{gbs:.0f} | {100*gbs/peak:.1f} |")
            traffic[wl] = {k: {"bytes_per_launch": (v[1] + v[2]) / v[0], "launches": v[0], "ms_per_launch": v[3] / v[0]}
                           for k, v in acc.items()}
        lines.append("")
    if a.launches:
        agg = launch_rows(a.launches)
        tot = sum(v[1] for v in agg.values()) or 1
        lines += ["## Launch list (`--metrics gpu__time_duration.sum`, serialised): share of device time", "",
                  "| kernel | launches | total ms | share |", "|---|---|---|---|"]
        for k, (n, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            lines.append(f"| `{k}` | {n} | {ms:.3f} | {100*ms/tot:.1f}% |")
        lines.append("")
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", f"ncu_summary_{a.tag}.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    with open(tpath, "w") as f:
        json.dump(traffic, f, indent=1, sort_keys=True)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
