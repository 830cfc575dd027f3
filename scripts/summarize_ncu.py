#!/usr/bin/env python
"""Summaries of ncu output for profiles/ (run here, no GPU needed).

    python scripts/summarize_ncu.py launches gpurun_out/launches.csv
        per-kernel share of device time from an `ncu --metrics gpu__time_duration.sum` list
    python scripts/summarize_ncu.py kernel gpurun_out/x.ncu-rep
        headline counters, stall reasons and the top source lines of one --set full capture
"""

from __future__ import annotations

import collections
import csv
import io
import subprocess
import sys


def launches(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    iK, iV, iU = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    scale = {"nsecond": 1.0, "usecond": 1e3, "msecond": 1e6, "second": 1e9}
    agg, cnt = collections.defaultdict(float), collections.Counter()
    for r in rows[start + 1:]:
        if len(r) <= iV:
            continue
        k = r[iK].split("(")[0]
        agg[k] += float(r[iV].replace(",", "")) * scale.get(r[iU], 1.0)
        cnt[k] += 1
    tot = sum(agg.values())
    print(f"{'kernel':70s} {'launches':>8s} {'ms':>10s} {'share':>7s}")
    for k, v in sorted(agg.items(), key=lambda t: -t[1]):
        print(f"{k[:70]:70s} {cnt[k]:8d} {v / 1e6:10.3f} {100 * v / tot:6.1f}%")
    print(f"{'total':70s} {sum(cnt.values()):8d} {tot / 1e6:10.3f}")


def _ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


def kernel(rep):
    det = list(csv.reader(io.StringIO(_ncu(rep, "--page", "details", "--csv"))))
    h = det[0]
    iS, iN, iU, iV = (h.index(x) for x in ("Section Name", "Metric Name", "Metric Unit",
                                           "Metric Value"))
    want = ("Duration", "DRAM Throughput", "Issue Slots Busy", "Issued Ipc Active",
            "L1/TEX Hit Rate", "L2 Hit Rate", "Registers Per Thread",
            "Dynamic Shared Memory Per Block", "Theoretical Active Warps per SM",
            "Achieved Active Warps Per SM", "Warp Cycles Per Issued Instruction",
            "Executed Instructions", "No Eligible")
    print("kernel:", det[1][h.index("Kernel Name")][:120])
    seen = set()
    for r in det[1:]:
        if len(r) > iV and r[iN] in want and r[iN] not in seen:
            seen.add(r[iN])
            print(f"  {r[iN]:40s} {r[iV]:>16s} {r[iU]}")
    raw = list(csv.reader(io.StringIO(_ncu(rep, "--page", "raw", "--csv"))))
    rh, rv = raw[0], raw[2]
    for name in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        if name in rh:
            print(f"  {name:40s} {rv[rh.index(name)]:>16s} {raw[1][rh.index(name)]}")
    st = [(rh[i], float(rv[i].replace(",", "") or 0)) for i in range(len(rh))
          if rh[i].startswith("smsp__pcsamp_warps_issue_stalled_")
          and not rh[i].endswith("not_issued")]
    tot = sum(v for _, v in st) or 1.0
    print("  stall samples:")
    for k, v in sorted(st, key=lambda t: -t[1])[:8]:
        print(f"    {k.replace('smsp__pcsamp_warps_issue_stalled_', ''):28s} {100 * v / tot:5.1f}%")
    src = list(csv.reader(io.StringIO(_ncu(rep, "--page", "source", "--csv",
                                           "--print-source", "cuda,sass"))))
    f, lines, tot_s = None, [], 0
    for r in src:
        if r and r[0] == "File Path":
            f = r[1].split("/")[-1]
            continue
        if len(r) < 8 or r[0] in ("Function Name", "Line No") or r[2] != "-":
            continue
        try:
            s, ins = int(r[4] or 0), int(r[7] or 0)
        except ValueError:
            continue
        lines.append((s, ins, f, r[0], r[1].strip()[:80]))
        tot_s += s
    tot_i = sum(x[1] for x in lines) or 1
    print("  top source lines (stall samples %, instructions %):")
    for s, ins, f, ln, txt in sorted(lines, reverse=True)[:15]:
        print(f"    {100 * s / max(tot_s, 1):5.1f}% {100 * ins / tot_i:5.1f}%i {f}:{ln} {txt}")


if __name__ == "__main__":
    {"launches": launches, "kernel": kernel}[sys.argv[1]](sys.argv[2])
