#!/usr/bin/env python
"""A/B timing of library builds in contact-rich (landed) states.

    python tools/ab_landed.py --prep            # saves the states under /tmp (one process)
    PBDR_LIB_PATH=... python tools/ab_landed.py  # times one build on every saved state

States: C5 at frame 80 (the bench's tail window start), C3 at frame 300 and
C4 at frame 150, each with its anchors and warm-start rotations, so every
build steps the identical state. Prints ms/frame, particle-substeps/s and a
hash of the final state (builds that only reorganise work must agree)."""
import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_14634_b200 import pbdr as P  # noqa: E402

STATES = [(5, 80), (3, 300), (4, 150)]


def path(cid, f):
    return f"/tmp/pbdr_ab_c{cid}_f{f}.npz"


ap = argparse.ArgumentParser()
ap.add_argument("--prep", action="store_true")
ap.add_argument("--frames", type=int, default=5)
ap.add_argument("--only", type=int, default=0)
ap.add_argument("--states", default="", help="config:frame list, e.g. 5:80,3:480 (default: the three above)")
a = ap.parse_args()
if a.states:
    STATES = [tuple(int(x) for x in t.split(":")) for t in a.states.split(",")]

for cid, f in STATES:
    if a.only and cid != a.only:
        continue
    g = P.GeneratedScene(cid)
    s = P.GpuSolver(g.desc, g.cfg)
    if a.prep:
        s.step_frames(f)
        p4, v4 = s.read_f32()
        np.savez(path(cid, f), p4=p4, v4=v4, anchor=s.debug_anchor(), rquat=s.debug_rquat())
        print(f"saved C{cid} frame {f}", flush=True)
        s.close()
        continue
    d = np.load(path(cid, f))
    s.write_f32(d["p4"], d["v4"])
    s.debug_write_anchor(d["anchor"])
    s.debug_write_rquat(d["rquat"])
    s.step_frames(2)
    t0 = time.time()
    ms = s.time_frames(a.frames)
    prof = s.profile_frames(1)
    p4, v4 = s.read_f32()
    h = hashlib.sha1(p4.tobytes() + v4.tobytes()).hexdigest()[:12]
    rate = s.n * 10 * a.frames / (ms / 1e3)
    print(json.dumps({"config": cid, "frame": f, "ms_per_frame": ms / a.frames, "rate": rate,
                      "iter_ms": prof["iteration"][0], "nbr_ms": prof["neighbours"][0], "hash": h,
                      "lib": os.path.basename(P.LIB_PATH)}), flush=True)
    s.close()
