"""Summarize ncu captures into the small text/JSON files committed here.

    python profiles/summarize.py full  <report.ncu-rep> <out.md>    # --set full capture
    python profiles/summarize.py launches <launches.csv> <out.md>   # gpu__time_duration list
    python profiles/summarize.py traffic <report.ncu-rep> <key> ...  # update ncu_traffic.json

The .ncu-rep files themselves stay in gpurun_out/ (scratch); only these
summaries are tracked.
"""

from __future__ import annotations

import csv
import io
import json
import os
import re
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))

DETAILS = ("Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput",
           "Executed Ipc Active", "Issue Slots Busy", "Registers Per Thread", "Theoretical Occupancy",
           "Achieved Occupancy", "L2 Hit Rate", "Grid Size", "Block Size",
           "Dynamic Shared Memory Per Block", "Static Shared Memory Per Block")


def _ncu(args):
    return subprocess.run(["ncu"] + args, capture_output=True, text=True, check=True).stdout


def full(rep, out):
    det = list(csv.reader(io.StringIO(_ncu(["-i", rep, "--page", "details", "--csv"]))))
    hdr = det[0]
    ki, mi, vi, ui = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    per = {}
    for row in det[1:]:
        if row[mi] in DETAILS:
            per.setdefault(row[ki], {}).setdefault(row[mi], f"{row[vi]} {row[ui]}".strip())
    raw = list(csv.reader(io.StringIO(_ncu(["-i", rep, "--page", "raw", "--csv"]))))
    rh = raw[0]
    idx = {h: i for i, h in enumerate(rh)}
    lines = [f"# ncu --set full summary: {os.path.basename(rep)}", ""]
    for row in raw[2:]:
        name = row[idx["Kernel Name"]]
        d = per.get(name, {})
        rd = float(row[idx["dram__bytes_read.sum"]])
        wr = float(row[idx["dram__bytes_write.sum"]])
        unit = raw[1][idx["dram__bytes_read.sum"]]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
        inst = float(row[idx["smsp__inst_executed.sum"]])
        stalls = []
        for h in rh:
            if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
                try:
                    stalls.append((float(row[idx[h]]), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        tot = sum(v for v, _ in stalls) or 1.0
        lines.append(f"## {name}")
        for k in DETAILS:
            if k in d:
                lines.append(f"- {k}: {d[k]}")
        lines.append(f"- dram__bytes_read.sum: {rd * scale:.0f} B; dram__bytes_write.sum: {wr * scale:.0f} B "
                     f"(traffic {(rd + wr) * scale:.0f} B)")
        lines.append(f"- smsp__inst_executed.sum: {inst:.0f} warp instructions")
        lines.append("- top stall reasons: " + ", ".join(f"{h} {100 * v / tot:.1f}%"
                                                       for v, h in sorted(stalls, reverse=True)[:6]))
        lines.append("")
    with open(out, "w") as f:
        f.write("\n".join(lines))
    print("\n".join(lines))


def launches(path, out):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    ki, mi, vi, ui = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    agg = {}
    for r in rows[start + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        v = float(r[vi].replace(",", ""))
        v = v / 1000.0 if r[ui] in ("nsecond", "ns") else (v * 1000.0 if r[ui] in ("msecond", "ms") else v)
        name = re.sub(r"\(.*", "", r[ki])[:90]
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v
    tot = sum(a[1] for a in agg.values()) or 1.0
    lines = [f"# launch list (ncu gpu__time_duration.sum, --clock-control none): {os.path.basename(path)}", "",
             "Cold-cache, serialized replay: compare SHARES, not absolute times.", "",
             "| kernel | launches | total us | share |", "|---|---|---|---|"]
    for name, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"| `{name}` | {n} | {t:.1f} | {100 * t / tot:.1f}% |")
    with open(out, "w") as f:
        f.write("\n".join(lines) + "\n")
    print("\n".join(lines))


def traffic(rep, keys):
    """keys: kernel-substring=json-key pairs, e.g. k_encode_grp=encode_b4_sr_g128."""
    raw = list(csv.reader(io.StringIO(_ncu(["-i", rep, "--page", "raw", "--csv"]))))
    rh = raw[0]
    idx = {h: i for i, h in enumerate(rh)}
    unit = raw[1][idx["dram__bytes_read.sum"]]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    p = os.path.join(HERE, "ncu_traffic.json")
    d = json.load(open(p)) if os.path.exists(p) else {}
    for kv in keys:
        sub, key = kv.split("=")
        for row in raw[2:]:
            if sub in row[idx["Kernel Name"]]:
                d[key] = round((float(row[idx["dram__bytes_read.sum"]]) +
                                float(row[idx["dram__bytes_write.sum"]])) * scale)
                break
    json.dump(d, open(p, "w"), indent=1, sort_keys=True)
    print(d)


if __name__ == "__main__":
    cmd = sys.argv[1]
    if cmd == "full":
        full(sys.argv[2], sys.argv[3])
    elif cmd == "launches":
        launches(sys.argv[2], sys.argv[3])
    elif cmd == "traffic":
        traffic(sys.argv[2], sys.argv[3:])
