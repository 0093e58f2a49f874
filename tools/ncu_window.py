#!/usr/bin/env python
"""Workload for ncu captures of a chosen window: pre-roll `--preroll` frames
with the profiler off, then cudaProfilerStart, `--substeps` substeps (or
`--frames` frames of graph replay), cudaProfilerStop. Run under
`ncu --profile-from-start off ...` so only the window's kernels are captured.
`--phase` instead prints the clock64 phase stamps of one iteration launch in
that state (tools/phase_timing.py's table)."""
import argparse
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_14634_b200 import pbdr as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=5)
ap.add_argument("--scale", type=int, default=0)
ap.add_argument("--preroll", type=int, default=80)
ap.add_argument("--substeps", type=int, default=1)
ap.add_argument("--frames", type=int, default=0)
ap.add_argument("--phase", action="store_true")
a = ap.parse_args()

g = P.GeneratedScene(a.config, seed=0, scale=a.scale)
s = P.GpuSolver(g.desc, g.cfg)
s.step_frames(a.preroll)
if a.phase:
    s.debug_prologue()
    s.debug_iteration()
    t = s.debug_phase_timing().astype(np.float64)
    names = ["stage(TMA)", "phaseA", "bodymathA", "phaseB", "bodymathB", "phaseC"]
    d = np.diff(t[:, :7], axis=1)
    print(f"config {a.config} frame {a.preroll}: {s.n} particles, {s.info.num_ctas} CTAs, kp {s.info.tile_kp}")
    for i, nm in enumerate(names):
        print(f"  {nm:12s} mean {d[:, i].mean():9.0f} cyc   p50 {np.median(d[:, i]):9.0f}   "
              f"p90 {np.percentile(d[:, i], 90):9.0f}")
    life = t[:, 6] - t[:, 0]
    print(f"  CTA lifetime mean {life.mean():.0f} cyc; kernel span {(t[:, 6].max() - t[:, 0].min()):.0f} cyc")
    sub = t[:, 8:14]
    ok = sub[:, 5] > 0
    if ok.any():
        sa = sub[ok]
        print(f"  body math A: sums read {np.mean(sa[:, 0] - t[ok, 2]):.0f}, pre-polar {np.mean(sa[:, 4] - sa[:, 0]):.0f}, "
              f"polar {np.mean(sa[:, 5] - sa[:, 4]):.0f}, post-polar {np.mean(sa[:, 1] - sa[:, 5]):.0f}, "
              f"to barrier exit {np.mean(t[ok, 3] - sa[:, 1]):.0f} cyc")
        print(f"  body math B: sums read {np.mean(sa[:, 2] - t[ok, 4]):.0f}, math {np.mean(sa[:, 3] - sa[:, 2]):.0f}, "
              f"to barrier exit {np.mean(t[ok, 5] - sa[:, 3]):.0f} cyc")
    hist = (t[:, 7].astype(np.int64) >> 16)
    if hist.max() > 0:  # PBDR_GN_PROBE build: Gauss-Newton steps per body (5 = cold polar)
        counts = [int(((hist >> (4 * k)) & 15).sum()) for k in range(6)]
        print("  GN steps histogram (0..4, cold):", counts)
    sys.exit(0)
rt = C.CDLL("libcudart.so.12")
rt.cudaDeviceSynchronize()
rt.cudaProfilerStart()
if a.frames:
    s.step_frames(a.frames)
else:
    s.step(a.substeps)
rt.cudaDeviceSynchronize()
rt.cudaProfilerStop()
print(f"config {a.config}: window after {a.preroll} frames done")
