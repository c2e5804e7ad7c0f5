#!/usr/bin/env python3
"""Summarize ncu captures (run here, no GPU needed) into profiles/<round>_ncu_summary.md and the
per-launch DRAM traffic table bench.py reads (profiles/ncu_traffic.json).

    python profiles/summarize.py --round r1 gpurun_out/prof_*.ncu-rep [--launches gpurun_out/launches.csv]
"""
import argparse
import collections
import csv
import io
import json
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
METRICS = {
    "gpu__time_duration.sum": "time",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
    "launch__registers_per_thread": "regs",
    "launch__grid_size": "grid",
    "smsp__inst_executed.sum": "inst",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9,
         "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "ns": 1e-9, "us": 1e-6, "ms": 1e-3}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")]}
        for m, k in METRICS.items():
            if m in hdr:
                i = hdr.index(m)
                try:
                    v = float(r[i].replace(",", ""))
                except ValueError:
                    continue
                d[k] = v * SCALE.get(units[i], 1)
        res.append(d)
    return res


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                name = d["Kernel Name"].split("(")[0].replace("void ", "").replace("unnamed>::", "")
                agg[name][0] += 1
                agg[name][1] += float(d["Metric Value"]) * SCALE.get(d["Metric Unit"], 1e-9)
    return agg


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("reps", nargs="+")
    ap.add_argument("--round", default="r1")
    ap.add_argument("--launches", default=None)
    ap.add_argument("--traffic-key", action="append", default=[],
                    help="KEY=REPNAME[:INDEX]: write DRAM bytes of that launch into ncu_traffic.json")
    ap.add_argument("--traffic-avg", action="append", default=[],
                    help="KEY=REPNAME:SUBSTRING: mean DRAM bytes per launch over that report's "
                         "launches whose kernel name contains SUBSTRING")
    a = ap.parse_args()
    lines = [f"# ncu summary ({a.round})", "",
             "Captured with `ncu --set full --clock-control none --import-source on` on one B200 "
             "(profiles/run_step.py). Times are ncu's cold-cache, serialised replays (compare shares, "
             "not absolutes); DRAM bytes are per launch.", ""]
    tables = {}
    for rep in a.reps:
        name = os.path.basename(rep).replace(".ncu-rep", "")
        rows = raw(rep)
        tables[name] = rows
        lines += [f"## {name}", "", "| kernel | time us | DRAM read MB | DRAM write MB | DRAM % | tensor % | SM % | occupancy % | regs | grid |",
                  "|---|---|---|---|---|---|---|---|---|---|"]
        for d in rows:
            k = d["kernel"].split("(")[0].replace("void ", "").replace("unnamed>::", "")[:60]
            lines.append(f"| `{k}` | {d.get('time', 0) * 1e6:.1f} | {d.get('dram_read', 0) / 1e6:.1f} | "
                         f"{d.get('dram_write', 0) / 1e6:.1f} | {d.get('dram_pct', 0):.1f} | "
                         f"{d.get('tensor_pct', 0):.1f} | {d.get('sm_pct', 0):.1f} | "
                         f"{d.get('occupancy_pct', 0):.1f} | {d.get('regs', 0):.0f} | {d.get('grid', 0):.0f} |")
        lines.append("")
    if a.launches:
        agg = launches(a.launches)
        tot = sum(v for _, v in agg.values())
        lines += ["## Launch list (gpu__time_duration.sum, all launches of the command)", "",
                  "| kernel | launches | total us | share |", "|---|---|---|---|"]
        for k, (n, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
            lines.append(f"| `{k[:70]}` | {n} | {v * 1e6:.1f} | {v / tot:.3f} |")
        lines.append("")
    with open(os.path.join(HERE, f"{a.round}_ncu_summary.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    tpath = os.path.join(HERE, "ncu_traffic.json")
    traffic = json.load(open(tpath)) if os.path.exists(tpath) else {}
    for spec in a.traffic_key:
        key, rest = spec.split("=")
        rep, _, idx = rest.partition(":")
        d = tables[rep][int(idx or 0)]
        traffic[key] = d.get("dram_read", 0) + d.get("dram_write", 0)
    for spec in a.traffic_avg:
        key, rest = spec.split("=")
        rep, _, sub = rest.partition(":")
        rows = [d for d in tables[rep] if sub in d["kernel"]]
        traffic[key] = sum(d.get("dram_read", 0) + d.get("dram_write", 0) for d in rows) / max(len(rows), 1)
    with open(tpath, "w") as f:
        json.dump(traffic, f, indent=1, sort_keys=True)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
