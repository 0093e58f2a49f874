#!/usr/bin/env python3
"""Top SASS instructions by warp-stall samples from an ncu report's source page
(`ncu -i REP --page source --csv --print-source sass`). Usage:
  python tools/ncu_hot_sass.py REPORT.ncu-rep [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
ai, si, wi = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
data = []
for i, r in enumerate(rows[2:]):
    if len(r) <= wi:
        continue
    try:
        data.append((int(r[wi]), i, r[si].strip()))
    except ValueError:
        pass
tot = sum(d[0] for d in data)
print(f"{len(data)} instructions, {tot} samples")
for s, i, src in sorted(data, reverse=True)[:top]:
    print(f"{s:7d} {100.0 * s / tot:5.1f}%  #{i:5d}  {src}")
