#!/usr/bin/env python
"""One small invocation of an execution path of the library, for
compute-sanitizer (memcheck / racecheck / synccheck). Every path the engine
selects has a case; contact-rich states come from a
state file written by `--prep` in a separate, un-instrumented process, so the
sanitized process runs only a frame or two.

    python tools/sanitize_case.py --prep CASE      # writes gpurun_out/san_CASE.npz
    compute-sanitizer --tool racecheck python tools/sanitize_case.py CASE
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2603_14634_b200 import pbdr as P  # noqa: E402

# name -> (config, scale, env, prep frames, frames under the sanitizer)
CASES = {
    "c1": (1, 0, {}, 0, 1),                                   # single body: all iterations in one launch
    "c2_coop": (2, 0, {}, 60, 1),                             # one-wave cooperative multi-iteration launch
    "c2_split": (2, 0, {"PBDR_COOP_ITERS": "0"}, 60, 1),      # isolated/contact split, fused integrate
    "c2_persistent": (2, 0, {"PBDR_COOP_ITERS": "0", "PBDR_ITER_GRID_CAP": "4"}, 60, 1),  # multi-tile loop
    "c4_cluster": (4, 8, {}, 60, 1),                          # one cluster per batched scene
    "c4_percall": (4, 8, {"PBDR_CLUSTER_ITERS": "0"}, 60, 1),  # per-iteration launches, scene partners
    "c5_coarse": (5, 6, {"PBDR_COOP_ITERS": "0"}, 40, 1),     # coarse body grid, oriented boxes
    "big": ("big", 0, {}, 30, 1),                             # bodies above one CTA: cluster kernel
    "torque": ("torque", 0, {}, 0, 1),                        # wrench prepass + windowed programs
}


def scene_for(case):
    cid, scale, env, _, _ = CASES[case]
    if cid == "big":
        g = np.stack(np.meshgrid(*[np.arange(13)] * 3, indexing="ij"), -1).reshape(-1, 3) * 0.02
        small = np.stack(np.meshgrid(*[np.arange(3)] * 3, indexing="ij"), -1).reshape(-1, 3) * 0.02
        bodies = [g + [0, 0, 0.2], g + [0.3, 0, 0.25]] + [small + [0.05 * k, 0.1, 0.6] for k in range(6)]
        return P.ArrayScene(**P.rigid_body_arrays(bodies, 0.01, [2.0, 2.0] + [0.1] * 6),
                            ground=P.Plane((0, 0, 0), (0, 0, 1), 0.5)), P.solver_cfg(frame_rate=240.0)
    if cid == "torque":
        g = P.GeneratedScene(2)
        progs = [P.ForceProgram((1.0, 0, 0), (0.0, 0.02, 0.01 * (b % 3)), 0.0, 0.002 if b % 2 else float("inf"),
                                b % 5 == 0, 0) for b in range(g.num_bodies)]
        return P.scene_with_programs(g, progs), g.cfg
    g = P.GeneratedScene(cid, scale=scale)
    return g, g.cfg


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("case", choices=sorted(CASES))
    ap.add_argument("--prep", action="store_true")
    args = ap.parse_args()
    _, _, env, prep_frames, frames = CASES[args.case]
    os.environ.update(env)
    sc, cfg = scene_for(args.case)
    s = P.GpuSolver(sc.desc, cfg)
    path = os.path.join(ROOT, "gpurun_out", f"san_{args.case}.npz")
    if args.prep:
        s.step_frames(prep_frames)
        p4, v4 = s.read_f32()
        np.savez(path, p4=p4, v4=v4, anchor=s.debug_anchor(), rquat=s.debug_rquat())
        return
    if prep_frames and os.path.exists(path):
        d = np.load(path)
        s.write_f32(d["p4"], d["v4"])
        s.debug_write_anchor(d["anchor"])
        s.debug_write_rquat(d["rquat"])
    s.step_frames(frames)
    s.step(1)  # direct (non-graph) substep
    s.read_bodies()
    pos, vel = s.read_particles()
    s.write_particles(pos, vel)
    s.step(1)
    print(f"{args.case}: ok ({s.n} particles)")


if __name__ == "__main__":
    main()
