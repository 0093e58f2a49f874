"""Trajectory emission: the per-frame, per-body sample of SPEC.md:357 (t, com,
orientation quaternion, P, L) written in the Trajectory CSV schema of
SPEC.md:485. The samples come from the device ring of
pbdr_gpu_trajectory_enable / _drain (one stats launch per frame, no host sync
per frame); this module only formats them.

The schema's ref_* / pos_err / rot_err_deg columns belong to the benchmark
module's analytic oracles (out of scope here): they are filled
when the caller passes a `reference(t, body) -> (ref_xyz, ref_angle_deg)`
callable, else left empty.
"""
from __future__ import annotations

import math

import numpy as np

HEADER = ("frame,t,body,com_x,com_y,com_z,qw,qx,qy,qz,Px,Py,Pz,Lx,Ly,Lz,"
          "ref_x,ref_y,ref_z,ref_angle_deg,pos_err,rot_err_deg")


def quat_angle_deg(q) -> float:
    """Rotation angle of a unit quaternion (w, x, y, z), degrees in [0, 180]."""
    w = min(1.0, abs(float(q[0])))
    return math.degrees(2.0 * math.acos(w))


class TrajectoryWriter:
    def __init__(self, path: str, bodies=None, reference=None):
        self.f = open(path, "w")
        self.f.write(HEADER + "\n")
        self.bodies = bodies
        self.reference = reference
        self.frame = 0
        self.last_t = -math.inf

    def write(self, t: np.ndarray, stats: np.ndarray):
        """t[frames], stats[frames, num_bodies, 13] as drained from the solver."""
        bodies = range(stats.shape[1]) if self.bodies is None else self.bodies
        for k in range(len(t)):
            tk = float(t[k])
            if not tk > self.last_t:
                raise ValueError("trajectory time must increase strictly (SPEC TrajectoryFrame invariant)")
            self.last_t = tk
            self.frame += 1
            for b in bodies:
                s = stats[k, b]
                ref = ["", "", "", "", "", ""]
                if self.reference is not None:
                    rxyz, rang = self.reference(tk, b)
                    perr = float(np.linalg.norm(np.asarray(s[0:3]) - np.asarray(rxyz)))
                    rerr = abs(quat_angle_deg(s[3:7]) - rang)
                    ref = [f"{rxyz[0]:.9g}", f"{rxyz[1]:.9g}", f"{rxyz[2]:.9g}", f"{rang:.9g}",
                           f"{perr:.9g}", f"{rerr:.9g}"]
                vals = [str(self.frame), f"{tk:.9g}", str(b)] + [f"{v:.9g}" for v in s] + ref
                self.f.write(",".join(vals) + "\n")

    def close(self):
        self.f.close()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def record(solver, frames: int, path: str, chunk: int = 64, bodies=None, reference=None):
    """Steps `frames` frames with emission on and writes the CSV; returns the
    number of rows written."""
    solver.enable_trajectory(min(chunk, frames))
    rows = 0
    with TrajectoryWriter(path, bodies, reference) as w:
        left = frames
        while left > 0:
            k = min(chunk, left)
            solver.step_frames(k)
            t, st = solver.drain_trajectory()
            w.write(t, st)
            rows += st.shape[0] * (st.shape[1] if bodies is None else len(bodies))
            left -= k
    solver.enable_trajectory(0)
    return rows
