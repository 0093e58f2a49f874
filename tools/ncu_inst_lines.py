"""Instructions executed per CUDA source line (ncu source page), with the
average active threads -- where a kernel's issue slots go.
Usage: python tools/ncu_inst_lines.py report.ncu-rep [top]"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
inst, thr, text = defaultdict(int), defaultdict(int), {}
cur, cur_file, hdr = None, "", None
for r in rows:
    if r and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 9:
        continue
    if r[0]:
        cur = (cur_file, int(r[0]))
        text[cur] = r[1].strip()[:80]
        continue
    try:
        inst[cur] += int(r[7])
        thr[cur] += int(r[8])
    except ValueError:
        pass
tot = sum(inst.values()) or 1
print(f"total warp instructions {tot}, mean active threads {sum(thr.values()) / tot:.1f}")
for k in sorted(inst, key=lambda k: -inst[k])[:top]:
    print(f"{inst[k] / tot:6.3f} {inst[k]:11d} thr {thr[k] / max(1, inst[k]):5.1f}  {k[0]}:{k[1]:4d}  {text.get(k, '')}")
