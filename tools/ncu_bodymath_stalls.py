"""Stall reasons of the instructions a kernel runs with few active threads
(the per-body math: one lane per body) vs the full-warp particle phases.
Usage: python tools/ncu_bodymath_stalls.py report.ncu-rep [max_threads=8]"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
maxthr = float(sys.argv[2]) if len(sys.argv) > 2 else 8.0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
col = {n: i for i, n in enumerate(hdr)}
reasons = [n for n in hdr if n.startswith("stall_") and "Not Issued" not in n]
groups = {"few": defaultdict(int), "full": defaultdict(int)}
inst = {"few": 0, "full": 0}
n_inst = {"few": 0, "full": 0}
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    try:
        ex = int(r[col["Instructions Executed"]])
        thr = float(r[col["Avg. Threads Executed"]])
    except ValueError:
        continue
    g = "few" if (ex > 0 and thr <= maxthr) else "full"
    inst[g] += ex
    n_inst[g] += 1
    for n in reasons:
        groups[g][n] += int(r[col[n]])
for g in groups:
    tot = sum(groups[g].values()) or 1
    print(f"{g}: {n_inst[g]} SASS instructions, {inst[g]} executed, {tot} samples")
    for n in sorted(reasons, key=lambda n: -groups[g][n])[:8]:
        print(f"   {n:24s} {groups[g][n]:8d} {groups[g][n] / tot:6.3f}")
