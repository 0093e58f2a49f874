"""Near (broadphase-filtered) particle fraction per config after a few frames."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_14634_b200 import pbdr as P
for cid in (3, 4, 5):
    g = P.GeneratedScene(cid)
    s = P.GpuSolver(g.desc, g.cfg)
    s.step_frames(3)
    s.debug_prologue()
    print(f"C{cid}: near fraction {len(s.debug_sorted()[0]) / s.n:.3f}")
