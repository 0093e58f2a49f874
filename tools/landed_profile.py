#!/usr/bin/env python
"""Where a contact-rich frame goes: for each (config, frame) state, the
per-kernel-class device times of one frame, the near-particle count, the
candidate statistics and the iteration kernel's clock64 phase table.

    python tools/landed_profile.py 3:300 3:480 5:80 5:99
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_14634_b200 import pbdr as P  # noqa: E402

for spec in sys.argv[1:] or ["3:300", "3:480", "5:80"]:
    cid, frame = (int(x) for x in spec.split(":"))
    g = P.GeneratedScene(cid)
    s = P.GpuSolver(g.desc, g.cfg)
    s.step_frames(frame)
    prof = s.profile_frames(1)
    s.debug_prologue()
    k, _ = s.debug_sorted()
    c, _ = s.debug_candidates()
    s.debug_iteration()
    t = s.debug_phase_timing().astype(np.float64)
    d = np.diff(t[:, :7], axis=1)
    names = ["stage", "phaseA", "bodymathA", "phaseB", "bodymathB", "phaseC"]
    print(json.dumps({
        "config": cid, "frame": frame, "particles": s.n, "tile_kp": s.info.tile_kp, "ctas": s.info.num_ctas,
        "frame_ms": {kk: round(v[0], 3) for kk, v in prof.items() if v[0] > 0},
        "near": int(len(k)), "near_frac": len(k) / s.n,
        "cand_mean": float(c.mean()), "cand_mean_near": float(c.sum() / max(1, len(k))),
        "with_cand_frac": float((c > 0).mean()), "cand_max": int(c.max()),
        "phase_cycles_mean": {nm: round(float(d[:, i].mean())) for i, nm in enumerate(names)},
        "phase_cycles_p90": {nm: round(float(np.percentile(d[:, i], 90))) for i, nm in enumerate(names)},
        "cta_life_mean": round(float((t[:, 6] - t[:, 0]).mean())),
    }), flush=True)
    s.close()
