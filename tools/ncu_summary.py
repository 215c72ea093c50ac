#!/usr/bin/env python
"""Summarise ncu captures brought back in gpurun_out/ into profiles/ (tracked).

    python tools/ncu_summary.py --round r1 --workload transformer_big_ende \
        --full k2_adam=gpurun_out/k2_r1.ncu-rep --full k1_add=gpurun_out/k1_r1.ncu-rep \
        --launches gpurun_out/launches_r1.csv

Writes profiles/<round>_<kernel>_ncu.txt (key metrics of one `ncu --set full` launch), profiles/<round>_launches.txt
(per-kernel launch count, summed device time and share from the `--metrics gpu__time_duration.sum` pass) and
merges dram traffic per launch into profiles/traffic.json (read by bench.py for roofline.traffic).
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
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__bytes.sum.per_second",
        "dram__bytes.sum.peak_sustained", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "launch__occupancy_limit_registers", "lts__t_bytes.sum",
        "smsp__average_warp_latency_issue_stalled_long_scoreboard", "smsp__inst_executed.sum",
        "sm__cycles_elapsed.avg.per_second", "dram__cycles_elapsed.avg.per_second"]
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True)
    rows = list(csv.reader(io.StringIO(out.stdout)))
    return rows[0], rows[1], rows[2:]


def to_bytes(val, unit):
    return float(val.replace(",", "")) * UNIT.get(unit.split("/")[0], 1)


def stall_top(rep, k=6):
    """Top warp-stall reasons summed over the source page (needs -lineinfo + --import-source)."""
    try:
        out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv", "--section", "WarpStateStats"],
                             capture_output=True, text=True, check=True).stdout
    except Exception:
        return ""
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--round", required=True)
    ap.add_argument("--workload", required=True)
    ap.add_argument("--full", action="append", default=[], help="kernel=path.ncu-rep")
    ap.add_argument("--launches", default=None)
    a = ap.parse_args()
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    traffic = json.load(open(tpath)) if os.path.exists(tpath) else {}
    for spec in a.full:
        kname, rep = spec.split("=", 1)
        hdr, units, rows = raw(rep)
        lines = [f"# ncu --set full --clock-control none, one launch of {kname} ({a.workload}); source {rep}"]
        for row in rows:
            name = row[hdr.index("Kernel Name")]
            lines.append(f"kernel: {name}")
            vals = {}
            for key in KEYS:
                if key in hdr:
                    i = hdr.index(key)
                    vals[key] = (row[i], units[i])
                    lines.append(f"{key:70s} {row[i]:>16s} {units[i]}")
            rd = to_bytes(*vals["dram__bytes_read.sum"])
            wr = to_bytes(*vals["dram__bytes_write.sum"])
            lines.append(f"{'dram bytes read+write per launch':70s} {rd + wr:16.0f} byte")
            traffic.setdefault(a.workload, {})[kname] = rd + wr
        path = os.path.join(ROOT, "profiles", f"{a.round}_{kname}_ncu.txt")
        with open(path, "w") as f:
            f.write("\n".join(lines) + "\n")
            ws = stall_top(rep)
            if ws:
                f.write("\n# WarpStateStats section\n" + ws)
        print("wrote", path)
    with open(tpath, "w") as f:
        json.dump(traffic, f, indent=1, sort_keys=True)
    if a.launches:
        tot = collections.defaultdict(float)
        cnt = collections.Counter()
        with open(a.launches) as f:
            text = f.read()
        text = text[text.index('"ID"'):] if '"ID"' in text else text
        for row in csv.DictReader(io.StringIO(text)):
            if row.get("Metric Name") != "gpu__time_duration.sum":
                continue
            name = re.sub(r"\(.*", "", row["Kernel Name"]).strip()
            v = float(row["Metric Value"].replace(",", ""))
            unit = row.get("Metric Unit", "")
            v = v / 1000.0 if unit in ("ns", "nsecond") else (v * 1000.0 if unit in ("ms", "msecond") else v)  # us
            tot[name] += v
            cnt[name] += 1
        s = sum(tot.values())
        lines = [f"# ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised launches); "
                 f"{a.workload}; source {a.launches}",
                 f"{'kernel':40s} {'launches':>9s} {'total_us':>12s} {'avg_us':>10s} {'share':>7s}"]
        for name in sorted(tot, key=lambda x: -tot[x]):
            lines.append(f"{name:40s} {cnt[name]:9d} {tot[name]:12.1f} {tot[name] / cnt[name]:10.2f} "
                         f"{tot[name] / s:7.3f}")
        path = os.path.join(ROOT, "profiles", f"{a.round}_launches.txt")
        with open(path, "w") as f:
            f.write("\n".join(lines) + "\n")
        print("wrote", path)


if __name__ == "__main__":
    main()
