"""Small fixed workload for ncu captures: one config, a few frames."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_14634_b200 import pbdr as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4)
ap.add_argument("--scale", type=int, default=512)
ap.add_argument("--frames", type=int, default=2)
ap.add_argument("--graph", type=int, default=1)
a = ap.parse_args()
g = P.GeneratedScene(a.config, seed=0, scale=a.scale)
s = P.GpuSolver(g.desc, g.cfg)
if a.graph:
    s.step_frames(a.frames)
else:
    s.step(a.frames * g.cfg.substeps)
p, _ = s.read_f32()
print(f"config {a.config} scale {a.scale}: {s.n} particles, {a.frames} frames, z mean {p[:, 2].mean():.6f}")
