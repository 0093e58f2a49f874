#!/usr/bin/env python
"""Writes the `roofline.traffic` source of bench.py: the iteration kernel's
measured DRAM bytes per launch (ncu dram__bytes_read.sum + dram__bytes_write.sum
from a launch-list CSV of one frame of the bench workload's timed window),
keyed by workload and window and stamped with the hash of the CUDA sources the
capture was taken on (bench.py quotes it only for that very build).

    python tools/ncu_traffic_json.py gpurun_out/X_launches_c5_frame90.csv \
        c5_giant_scene_131072_cubes:tail "k_iteration<4, 0, 0>" profiles/X_launches_c5_frame90.csv
"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

path, key, kernel, source = sys.argv[1:5]
rows = list(csv.reader(open(path)))
start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[start]
ki, mi, vi, ui = (hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"),
                  hdr.index("Metric Unit"))
scale_b = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
scale_t = {"nsecond": 1e-9, "ns": 1e-9, "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3, "ms": 1e-3, "second": 1.0}
dram, secs, launches = 0.0, 0.0, 0
for r in rows[start + 1:]:
    if kernel not in r[ki]:
        continue
    v = float(r[vi].replace(",", ""))
    if r[mi].startswith("dram__bytes"):
        dram += v * scale_b.get(r[ui], 1.0)
    elif r[mi] == "gpu__time_duration.sum":
        secs += v * scale_t.get(r[ui], 1.0)
        launches += 1
out = os.path.join(ROOT, "profiles", "ncu_iteration_summary.json")
try:
    d = json.load(open(out))
except (OSError, ValueError):
    d = {}
d[key] = {"kernel": kernel, "launches": launches, "dram_bytes_per_launch": dram / launches,
          "dram_gbs": dram / secs / 1e9, "avg_launch_ms_under_ncu": 1e3 * secs / launches,
          "build": bench.build_id(), "capture": source,
          "limiter": "latency (issue 51%, DRAM 55% of peak; barrier and long-scoreboard stalls)"}
json.dump(d, open(out, "w"), indent=1)
print(json.dumps(d[key], indent=1))
