"""Generates tests/golden/ref_golden.json from the reference's OWN compiled code.

Runs only where /root/reference exists (this container): `make ref` compiles
/root/reference/proj/src/{math,body,geometry}.cpp in place (oracle/Makefile)
into oracle/_ref/libpbdr_ref.so, and this script evaluates the reference's
functions on fixed, seeded inputs:
  * Rng (rng.hpp:10-29): splitmix64 u64 / next_unit streams,
  * pack_box (geometry.cpp:32-55),
  * polar_decompose (math.cpp:170-210), sym_eigen (math.cpp:26-71),
    invert_spd / pseudo_invert_spd (math.cpp:73-108), inverse (math.cpp:8-24),
  * make_body + compute_com / compute_inertia / compute_momentum
    (body.cpp:16-83), extract_pose (body.cpp:103-124), distribute_wrench
    (body.cpp:126-150).
The committed JSON travels to the GPU box; nothing at test time reads
/root/reference. Usage:  python tests/golden/make_golden.py
"""
from __future__ import annotations

import ctypes as C
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import pyoracle  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "ref_golden.json")


def p(a):
    return a.ctypes.data_as(C.c_void_p)


def rot(axis, ang):
    axis = np.asarray(axis, float) / np.linalg.norm(axis)
    K = np.array([[0, -axis[2], axis[1]], [axis[2], 0, -axis[0]], [-axis[1], axis[0], 0]])
    return np.eye(3) + np.sin(ang) * K + (1 - np.cos(ang)) * K @ K


def main():
    L = pyoracle.rlib()
    if L is None:
        sys.exit("oracle/_ref/libpbdr_ref.so missing: run `make ref` (needs /root/reference)")
    rs = np.random.default_rng(20261020)
    g = {"source": "reference proj/src/{math,body,geometry}.cpp via oracle/_ref", "cases": {}}

    # Rng streams.
    rng = []
    for seed in (0, 1, 42, 0xDEADBEEF):
        u = np.zeros(16, np.uint64)
        L.ref_rng_u64(seed, 16, p(u))
        d = np.zeros(16)
        L.ref_rng_unit(seed, 16, p(d))
        rng.append({"seed": seed, "u64": [int(x) for x in u], "unit": d.tolist()})
    g["cases"]["rng"] = rng

    # pack_box.
    boxes = []
    for h, n in (((0.1, 0.1, 0.1), 4), ((0.08, 0.08, 0.08), 8), ((0.06, 0.06, 0.06), 6),
                 ((0.1, 0.1, 0.1), 1), ((0.1, 0.05, 0.2), 3)):
        c = np.zeros(3 * n ** 3)
        r = C.c_double()
        cnt = L.ref_pack_box(h[0], h[1], h[2], n, p(c), C.byref(r))
        boxes.append({"half": h, "n": n, "count": cnt, "radius": r.value, "centers": c.tolist()})
    g["cases"]["pack_box"] = boxes

    # Polar decompositions: SPEC examples + seeded near-rigid and general matrices.
    mats = [np.eye(3), 2 * np.eye(3), rot([0, 0, 1], np.pi / 6) @ np.diag([2, 1, 1])]
    for _ in range(24):
        R0 = rot(rs.normal(size=3), rs.uniform(0, np.pi))
        S = np.eye(3) + 1e-3 * rs.normal(size=(3, 3))
        mats.append(R0 @ ((S + S.T) / 2) * rs.uniform(1e-4, 10))
    for _ in range(8):
        A = rs.normal(size=(3, 3))
        if np.linalg.det(A) < 0:
            A[0] *= -1
        mats.append(A)
    polar = []
    for A in mats:
        A = np.ascontiguousarray(A)
        R = np.zeros(9)
        S = np.zeros(9)
        q = np.zeros(4)
        st = L.ref_polar(p(A.reshape(9)), p(R), p(S), p(q), 1e-12)
        polar.append({"A": A.reshape(9).tolist(), "status": st, "R": R.tolist(), "q": q.tolist()})
    g["cases"]["polar"] = polar

    # SPD inverse / pseudo-inverse / eigen.
    spd = [np.diag([2.0, 4.0, 8.0]), np.eye(3), np.diag([0.0, 2.0, 2.0])]
    for _ in range(10):
        B = rs.normal(size=(3, 3))
        spd.append(B @ B.T + 0.1 * np.eye(3))
    spd.append(np.diag([1e-13, 1.0, 1.0]))
    inv = []
    for M in spd:
        M = np.ascontiguousarray(M, dtype=np.float64)
        out = np.zeros(9)
        axis = np.zeros(3)
        st = L.ref_invert_spd(p(M.reshape(9)), p(out), p(axis))
        pinv = np.zeros(9)
        rank = C.c_int()
        nax = np.zeros(3)
        L.ref_pseudo_invert_spd(p(M.reshape(9)), p(pinv), C.byref(rank), p(nax))
        ev = np.zeros(3)
        vecs = np.zeros(9)
        L.ref_sym_eigen(p(M.reshape(9)), p(ev), p(vecs))
        inv.append({"M": M.reshape(9).tolist(), "inv_status": st, "inv": out.tolist(),
                    "axis": axis.tolist(), "pinv": pinv.tolist(), "rank": rank.value,
                    "null_axis": nax.tolist(), "ev": ev.tolist(), "vecs": vecs.tolist()})
    g["cases"]["spd"] = inv

    # Body properties.
    bodies = []
    sets = [
        (np.array([[1.0, 0, 0], [-1.0, 0, 0]]), np.array([[0, 0.5, 0], [0, -0.5, 0]]), np.array([1.0, 1.0])),
        (np.array([[0.0, 0, 0], [4.0, 0, 0]]), np.zeros((2, 3)), np.array([1.0, 1 / 3])),
    ]
    c64 = np.zeros(3 * 64)
    r = C.c_double()
    L.ref_pack_box(0.1, 0.1, 0.1, 4, p(c64), C.byref(r))
    sets.append((c64.reshape(64, 3), np.zeros((64, 3)), np.full(64, 16.0)))
    for _ in range(4):
        n = int(rs.integers(3, 40))
        sets.append((rs.normal(size=(n, 3)) * 0.1 + rs.normal(size=3) * 5,
                     rs.normal(size=(n, 3)), rs.uniform(1, 100, size=n)))
    for pos, vel, w in sets:
        pos = np.ascontiguousarray(pos, np.float64)
        vel = np.ascontiguousarray(vel, np.float64)
        w = np.ascontiguousarray(w, np.float64)
        com = np.zeros(3)
        I = np.zeros(9)
        P = np.zeros(3)
        Lm = np.zeros(3)
        col = C.c_int()
        axis = np.zeros(3)
        st = L.ref_body_props(len(w), p(pos), p(vel), p(w), p(com), p(I), p(P), p(Lm), C.byref(col), p(axis))
        bodies.append({"pos": pos.reshape(-1).tolist(), "vel": vel.reshape(-1).tolist(), "inv_mass": w.tolist(),
                       "status": st, "com": com.tolist(), "inertia": I.tolist(), "P": P.tolist(), "L": Lm.tolist(),
                       "collinear": col.value, "rest_axis": axis.tolist()})
    g["cases"]["bodies"] = bodies

    # extract_pose: rest = a lattice, current = rigidly moved (+ small noise).
    poses = []
    c27 = np.zeros(3 * 27)
    L.ref_pack_box(0.06, 0.06, 0.06, 3, p(c27), C.byref(r))
    rest = c27.reshape(27, 3) + np.array([0.3, -0.2, 0.5])
    for k in range(6):
        R0 = rot(rs.normal(size=3), rs.uniform(0, np.pi))
        t = rs.normal(size=3)
        cur = (rest @ R0.T) + t + (0 if k < 3 else 1e-4 * rs.normal(size=rest.shape))
        w = np.full(27, 27.0 / 2.0)
        com = np.zeros(3)
        q = np.zeros(4)
        st = L.ref_extract_pose(27, p(np.ascontiguousarray(rest)), p(np.ascontiguousarray(cur)), p(w), p(com), p(q))
        poses.append({"rest": rest.reshape(-1).tolist(), "cur": cur.reshape(-1).tolist(), "inv_mass": w.tolist(),
                      "status": st, "com": com.tolist(), "quat": q.tolist()})
    g["cases"]["extract_pose"] = poses

    # distribute_wrench (SPEC.md:279 sum rule).
    wr = []
    pos = np.ascontiguousarray(c64.reshape(64, 3) + np.array([0, 0, 0.1]))
    w = np.full(64, 16.0)
    for F, tau in (((17.0, 0, 0), (0, 0, 0)), ((0, 0, 0), (0, 0, 0.01)), ((1.0, -2.0, 0.5), (0.01, 0.02, -0.03))):
        out = np.zeros(3 * 64)
        axis = np.zeros(3)
        st = L.ref_distribute_wrench(64, p(pos), p(w), p(np.array(F, float)), p(np.array(tau, float)), p(out), p(axis))
        wr.append({"pos": pos.reshape(-1).tolist(), "inv_mass": w.tolist(), "F": F, "tau": tau, "status": st,
                   "forces": out.tolist()})
    g["cases"]["wrench"] = wr

    with open(OUT, "w") as f:
        json.dump(g, f, indent=None, separators=(",", ":"))
    print(f"wrote {OUT} ({os.path.getsize(OUT)} bytes)")


if __name__ == "__main__":
    main()
