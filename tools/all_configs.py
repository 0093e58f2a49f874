#!/usr/bin/env python
"""Every BASELINE config on one B200, each over its whole run, with the
clocks sampled during every timed region (bench.py's ClockSampler).

For each config: frames 0..W-1 warm-up, then frames W..F-1 timed in three
windows -- head (the first K frames after the warm-up, free flight for the
piles), middle, tail (the last K frames, contact-rich) -- whose sum is the
whole-run time. One JSON line per config:
    python tools/all_configs.py > profiles/rNN_all_configs.jsonl
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import ClockSampler, measured_peak, BYTES_PER_SUBSTEP  # noqa: E402
from paper_2603_14634_b200 import pbdr as P  # noqa: E402

FRAMES = {1: 1000, 2: 1000, 3: 500, 4: 200, 5: 100}

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="1,2,3,4,5")
ap.add_argument("--window", type=int, default=20)
ap.add_argument("--warmup", type=int, default=5)
a = ap.parse_args()
peak, _ = measured_peak()
for cid in [int(c) for c in a.configs.split(",")]:
    g = P.GeneratedScene(cid)
    s = P.GpuSolver(g.desc, g.cfg)
    F, W, K = FRAMES[cid], a.warmup, a.window
    s.step_frames(W)
    mid = max(0, (F - W - 2 * K))
    with ClockSampler(0) as clocks:
        head = s.time_frames(K)
        middle = s.time_frames(mid) if mid > 0 else 0.0
        tail = s.time_frames(K)
    n = s.n
    rate = lambda frames, ms: n * g.cfg.substeps * frames / (ms / 1e3) if ms > 0 else None  # noqa: E731
    whole = rate(2 * K + mid, head + middle + tail)
    print(json.dumps({
        "config": cid, "workload": P.CONFIG_NAMES[cid], "particles": n, "bodies": s.nb, "tile_kp": s.info.tile_kp,
        "unit": "particle-substeps/s",
        "head": {"frames": f"{W}..{W + K - 1}", "value": rate(K, head), "ms_per_frame": head / K},
        "tail": {"frames": f"{F - K}..{F - 1}", "value": rate(K, tail), "ms_per_frame": tail / K},
        "whole_run": {"frames": f"{W}..{F - 1}", "value": whole,
                      "substep_frac_1120B": whole * BYTES_PER_SUBSTEP / (peak * 1e9) if whole else None},
        "clocks": clocks.summary(),
    }), flush=True)
    s.close()
