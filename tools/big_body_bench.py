"""Throughput of scenes made of large bodies (resolution-study sizes) on one
B200: per body size, a batch of independent one-body scenes (no contact pairs:
all iterations of a substep in one launch) and a pile variant (bodies side by
side in shared scenes: contacts, one launch per iteration). Prints one JSON
line per case with particle-substeps/s and the iteration kernels' share.
Bodies of <= 2048 particles run on the tiled kernel, larger ones on the
cluster kernel (k_iteration_big)."""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_14634_b200 import pbdr as P  # noqa: E402


def box(n_axis, s=0.02):
    g = np.stack(np.meshgrid(*[np.arange(n_axis)] * 3, indexing="ij"), -1).reshape(-1, 3)
    return (g - (n_axis - 1) / 2.0) * s


def scene(n_axis, target, pile):
    nper = n_axis ** 3
    nb = max(1, target // nper)
    b0 = box(n_axis)
    ext = 0.02 * n_axis
    bodies, scenes = [], []
    side = int(np.ceil(np.sqrt(nb)))
    for b in range(nb):
        i, j = divmod(b, side)
        if pile:  # bodies in rows of 4 touching neighbours within one scene
            scenes.append(b // 4)
            c = np.array([(b % 4) * (ext + 0.005), 0.0, ext / 2 + 0.001]) + np.array([0.0, 100.0 * (b // 4), 0.0])
        else:
            scenes.append(b)
            c = np.array([i * (ext + 0.1), j * (ext + 0.1), ext / 2 + 0.05])
        bodies.append(b0 + c)
    arr = P.rigid_body_arrays(bodies, 0.01, [1.0] * nb)
    return P.ArrayScene(**arr, body_scene=np.array(scenes, dtype=np.int32),
                        ground=P.Plane((0, 0, 0), (0, 0, 1), 0.5))


ap = argparse.ArgumentParser()
ap.add_argument("--sizes", default="12,13,16,21,26,32")
ap.add_argument("--target", type=int, default=8_000_000, help="particles per case")
ap.add_argument("--frames", type=int, default=3)
ap.add_argument("--case", choices=["single", "pile", "both"], default="both")
a = ap.parse_args()
cfg = P.solver_cfg(frame_rate=240.0)
for pile in {"single": (False,), "pile": (True,), "both": (False, True)}[a.case]:
    for n_axis in [int(x) for x in a.sizes.split(",")]:
        sc = scene(n_axis, a.target, pile)
        s = P.GpuSolver(sc.desc, cfg)
        s.step_frames(1)
        ms = s.time_frames(a.frames)
        prof = s.profile_frames(1)
        n = sc.num_particles
        tot = sum(v[0] for v in prof.values())
        row = {"case": "pile" if pile else "single", "n_axis": n_axis, "body_particles": n_axis ** 3,
               "bodies": sc.num_bodies, "particles": n,
               "particle_substeps_per_s": n * cfg.substeps * a.frames / (ms * 1e-3),
               "iteration_share": prof["iteration"][0] / tot if tot else None,
               "iteration_ms_per_frame": prof["iteration"][0],
               "iteration_launches_per_frame": prof["iteration"][1],
               "iteration_GBps_at_96B": n * cfg.substeps * cfg.solver_iterations * 96 / (prof["iteration"][0] * 1e-3) / 1e9}
        print(json.dumps(row), flush=True)
        del s
