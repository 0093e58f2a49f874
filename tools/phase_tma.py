import os, sys, numpy as np
sys.path.insert(0, "/root/repo" if os.path.exists("/root/repo") else ".")
from paper_2603_14634_b200 import pbdr as P
g = P.GeneratedScene(4); s = P.GpuSolver(g.desc, g.cfg); s.step_frames(3); s.debug_prologue(); s.debug_iteration()
t = s.debug_phase_timing().astype(np.float64)
iss = t[:, 7] - t[:, 0]; stg = t[:, 1] - t[:, 0]
print("entry->TMA issue mean %.0f p50 %.0f p90 %.0f" % (iss.mean(), np.median(iss), np.percentile(iss, 90)))
print("entry->staged   mean %.0f ; issue->staged mean %.0f" % (stg.mean(), (stg - iss).mean()))
