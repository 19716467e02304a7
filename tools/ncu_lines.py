"""Summarise an ncu report's source view by source line and by function.

  python tools/ncu_lines.py REPORT.ncu-rep [--top 40]

Runs `ncu -i REPORT --page source --csv --print-source cuda,sass`, sums the
warp-stall samples of each CUDA source line, and attributes lines to the
enclosing function (nearest preceding definition in the file).
"""
import argparse
import csv
import io
import os
import re
import subprocess
from collections import defaultdict

DEF = re.compile(r"^(?:template\s*<.*>\s*)?(?:HDN|HD|__device__|__global__|static|inline|int|void|double|bool)\b.*?\b(\w+)\s*\(")


def func_starts(path):
    starts = []
    try:
        with open(path) as f:
            for i, line in enumerate(f, 1):
                if line.startswith((" ", "\t", "//", "#", "}")):
                    continue
                m = DEF.match(line)
                if m:
                    starts.append((i, m.group(1)))
    except OSError:
        pass
    return starts


def main():
    p = argparse.ArgumentParser()
    p.add_argument("report")
    p.add_argument("--top", type=int, default=40)
    a = p.parse_args()
    out = subprocess.run(["ncu", "-i", a.report, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    cur = None
    hdr = None
    per_line = defaultdict(float)
    per_line_exec = defaultdict(float)
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            cur = r[1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or cur is None or not r[0]:
            continue
        try:
            ln = int(r[0])
        except ValueError:
            continue
        try:
            smp = float(r[4] or 0) if r[4] not in ("-", "") else 0.0
            ex = float(r[7] or 0) if r[7] not in ("-", "") else 0.0
        except (ValueError, IndexError):
            continue    # source text with unescaped quotes breaks the CSV row
        per_line[(cur, ln)] += smp
        per_line_exec[(cur, ln)] += ex
    tot = sum(per_line.values()) or 1.0
    starts = {}
    per_func = defaultdict(float)
    for (f, ln), v in per_line.items():
        if f not in starts:
            starts[f] = func_starts(f)
        name = "?"
        for s, nm in starts[f]:
            if s <= ln:
                name = nm
            else:
                break
        per_func[(os.path.basename(f), name)] += v
    print("== functions ==")
    for (f, nm), v in sorted(per_func.items(), key=lambda x: -x[1])[: a.top]:
        print(f"{v / tot:7.3f}  {f}:{nm}")
    print("== lines ==")
    for (f, ln), v in sorted(per_line.items(), key=lambda x: -x[1])[: a.top]:
        try:
            src = open(f).read().splitlines()[ln - 1].strip()[:90]
        except (OSError, IndexError):
            src = ""
        print(f"{v / tot:7.3f}  {os.path.basename(f)}:{ln}  {src}")


if __name__ == "__main__":
    main()
