#!/usr/bin/env python3
"""Condenses `nvcc -Xptxas -v` output (stdin) to one line per kernel:
registers, stack frame, spill stores/loads. Used to check that a refactor
leaves the hot kernels' register allocation unchanged."""
import re
import subprocess
import sys

cur = None
props = None  # function whose "Function properties" block is being read
rows = {}
for line in sys.stdin:
    m = re.search(r"Compiling entry function '([^']+)'", line)
    if m:
        cur = m.group(1)
        rows[cur] = {}
        continue
    m = re.search(r"Function properties for (\S+)", line)
    if m:
        props = m.group(1)
        continue
    if cur is None:
        continue
    if "stack frame" in line and props != cur:
        continue
    m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m:
        rows[cur].update(stack=int(m.group(1)), st=int(m.group(2)), ld=int(m.group(3)))
    m = re.search(r"Used (\d+) registers", line)
    if m:
        rows[cur]["regs"] = int(m.group(1))
names = list(rows)
try:
    dem = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.split("\n")
except OSError:
    dem = names
for raw, d in zip(names, dem):
    r = rows[raw]
    short = re.sub(r"pbdr_dev::\(anonymous namespace\)::", "", d)
    short = re.sub(r"\(pbdr_dev::\w+\)", "", short)
    print(f"{short:48s} regs={r.get('regs','?'):>3} stack={r.get('stack','?'):>4} spill_st={r.get('st','?'):>4} spill_ld={r.get('ld','?'):>4}")
