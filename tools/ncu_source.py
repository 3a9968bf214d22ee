"""Per-source-line breakdown of one kernel in an .ncu-rep (captured with
--import-source on and -lineinfo): instructions executed and warp-stall
samples per CUDA source line, the top lines, and totals per labelled line
range of a file.

    python tools/ncu_source.py REPORT [--file snp_device.cuh] [--top 40]
                               [--ranges phase1:1480-1530,phase2:1550-1660]
"""

from __future__ import annotations

import argparse
import csv
import io
import subprocess


def load(report: str, view: str = "cuda,sass") -> list[dict]:
    out = subprocess.run(["ncu", "-i", report, "--page", "source", "--csv", "--print-source", view],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    res, hdr, fname = [], None, None
    for r in rows:
        if not r:
            continue
        if len(r) == 1 and r[0].strip():
            fname = r[0].strip()  # some ncu versions print the file path on its own line
            continue
        if r[0] in ("File Path", "File Name") and len(r) == 2:
            fname = r[1].strip()  # ncu 2025: a ("File Path", path) row per file
            continue
        if r[0] == "Function Name":
            continue
        if hdr is None or r[0] in ("#", "Line", "Line No", "# Address", "Address"):
            hdr = r
            continue
        if view == "cuda,sass" and not r[0]:
            continue  # the mixed view's SASS rows under each source line
        d = {}
        for h_, v_ in zip(hdr, r):
            d.setdefault(h_, v_)  # the first "Source" column is the CUDA line
        d["_file"] = fname
        res.append(d)
    return res


def num(x) -> float:
    try:
        return float(str(x).replace(",", ""))
    except ValueError:
        return 0.0


def pick(d: dict, *names):
    for n in names:
        for k in d:
            if k.strip().lower() == n.lower():
                return d[k]
    for n in names:
        for k in d:
            if n.lower() in k.strip().lower():
                return d[k]
    return None


def main():
    p = argparse.ArgumentParser()
    p.add_argument("report")
    p.add_argument("--file", default=None, help="only lines of source files whose path contains this")
    p.add_argument("--top", type=int, default=40)
    p.add_argument("--ranges", default="", help="label:first-last,... line ranges to total")
    a = p.parse_args()
    rows = load(a.report)
    lines = []
    for d in rows:
        if a.file and d.get("_file") and a.file not in d["_file"]:
            continue
        ln = pick(d, "Line No", "#", "Line", "Line Number")
        inst = num(pick(d, "Instructions Executed", "inst_executed"))
        stall = num(pick(d, "Warp Stall Sampling (All Samples)", "Warp Stall Sampling"))
        src = pick(d, "Source") or ""
        try:
            ln = int(ln)
        except (TypeError, ValueError):
            continue
        lines.append((ln, inst, stall, src.strip()[:110]))
    tot_i = sum(x[1] for x in lines) or 1.0
    tot_s = sum(x[2] for x in lines) or 1.0
    print(f"total instructions executed (warp-level): {tot_i:.4g}; stall samples: {tot_s:.4g}")
    if a.ranges:
        for part in a.ranges.split(","):
            label, span = part.split(":")
            lo, hi = (int(x) for x in span.split("-"))
            ii = sum(x[1] for x in lines if lo <= x[0] <= hi)
            ss = sum(x[2] for x in lines if lo <= x[0] <= hi)
            print(f"  {label:>12s} lines {lo}-{hi}: inst {ii:.4g} ({100 * ii / tot_i:.1f} %), stalls {100 * ss / tot_s:.1f} %")
    print(f"top {a.top} lines by instructions executed:")
    for ln, inst, stall, src in sorted(lines, key=lambda x: -x[1])[:a.top]:
        print(f"  {ln:5d} {100 * inst / tot_i:5.1f}% inst {100 * stall / tot_s:5.1f}% stall  {src}")


if __name__ == "__main__":
    main()
