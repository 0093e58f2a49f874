"""Per-CTA phase durations of one k_iteration launch (clock64 stamps)."""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_14634_b200 import pbdr as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4)
ap.add_argument("--scale", type=int, default=0)
ap.add_argument("--frames", type=int, default=3)
a = ap.parse_args()
g = P.GeneratedScene(a.config, seed=0, scale=a.scale)
s = P.GpuSolver(g.desc, g.cfg)
s.step_frames(a.frames)
s.debug_prologue()
s.debug_iteration()
t = s.debug_phase_timing().astype(np.float64)
sub = t[:, 8:14]
names = ["stage(TMA)", "phaseA", "bodymathA", "phaseB", "bodymathB", "phaseC"]
d = np.diff(t[:, :7], axis=1)
print(f"config {a.config}: {s.n} particles, {s.info.num_ctas} CTAs")
for i, nm in enumerate(names):
    print(f"  {nm:12s} mean {d[:, i].mean():9.0f} cyc   p50 {np.median(d[:, i]):9.0f}   p90 {np.percentile(d[:, i], 90):9.0f}")
life = t[:, 6] - t[:, 0]
print(f"  CTA lifetime mean {life.mean():.0f} cyc; kernel span {(t[:, 6].max() - t[:, 0].min()):.0f} cyc")
sm = t[:, 7].astype(int)
# average concurrency per SM: sum of lifetimes / span per SM
conc = []
for k in np.unique(sm):
    m = sm == k
    span = t[m, 6].max() - t[m, 0].min()
    conc.append(life[m].sum() / span)
print(f"  mean resident CTAs per SM {np.mean(conc):.2f}")
