"""Aggregates ncu source-page stall samples per CUDA source line.
Usage: python tools/ncu_lines.py report.ncu-rep kernel_regex [top]"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "-k", f"regex:{kern}"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = None
cur_line, cur_src, cur_file = None, None, ""
samples = defaultdict(int)
inst = defaultdict(int)
text = {}
for r in rows:
    if r and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 7:
        continue
    if r[0]:
        cur_line = (cur_file, int(r[0]))
        text[cur_line] = r[1].strip()[:90]
        continue
    try:
        samples[cur_line] += int(r[4])
        inst[cur_line] += int(r[7])
    except (ValueError, IndexError):
        pass
tot = sum(samples.values()) or 1
print(f"total samples {tot}")
for k in sorted(samples, key=lambda k: -samples[k])[:top]:
    print(f"{samples[k] / tot:6.3f} {inst[k]:10d}  {k[0]}:{k[1]:4d}  {text.get(k, '')}")
