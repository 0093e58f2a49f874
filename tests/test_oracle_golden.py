"""Pins the oracle's restated numerics (and the product's host-side scene
helpers) against golden vectors produced by the reference's OWN compiled code
(tests/golden/ref_golden.json, made by tests/golden/make_golden.py from
/root/reference/proj/src/{math,body,geometry}.cpp)."""
import numpy as np
import pytest

from paper_2603_14634_b200 import pbdr as P


def test_rng_stream_bit_exact(pbdr, golden):
    # rng.hpp:10-29 splitmix64 and its fixed 53-bit double mapping.
    for case in golden["rng"]:
        u = P.rng_u64(case["seed"], 16)
        assert [int(x) for x in u] == case["u64"]
        d = P.rng_unit(case["seed"], 16)
        assert d.tolist() == case["unit"]
    # Rng(0).next_u64() = 7960286522194355700.
    assert int(P.rng_u64(0, 1)[0]) == 7960286522194355700


def test_pack_box_bit_exact(pbdr, golden):
    # geometry.cpp:32-55 (z-fastest lattice, radius = half the smallest spacing).
    for case in golden["pack_box"]:
        c, r = P.pack_box(case["half"], case["n"])
        assert len(c) == case["count"]
        assert r == case["radius"]
        assert c.reshape(-1).tolist() == case["centers"]


def test_polar_matches_reference(pyoracle, golden):
    # math.cpp:170-210 scaled-Newton polar (tol 1e-9). Ours differs in the
    # scaling schedule, the stopping rule and a scale-relative degeneracy test
    # (DESIGN.md), so both are within the 1e-9 tolerance of the polar factor.
    checked = 0
    for case in golden["polar"]:
        A = np.array(case["A"])
        ok, R, q = pyoracle.polar(A)
        if case["status"] != 0:
            continue
        assert ok, A
        Rref = np.array(case["R"]).reshape(3, 3)
        np.testing.assert_allclose(R, Rref, atol=2e-9)
        qref = np.array(case["q"])
        assert min(np.abs(q - qref).max(), np.abs(q + qref).max()) < 2e-9
        checked += 1
    assert checked >= 30


def test_polar_spec_examples(pyoracle):
    # A = I -> R = I; A = 2I -> R = I; A = Rz(30) diag(2,1,1) -> Rz(30).
    ok, R, _ = pyoracle.polar(np.eye(3))
    assert ok and np.allclose(R, np.eye(3), atol=1e-15)
    ok, R, _ = pyoracle.polar(2 * np.eye(3))
    assert ok and np.allclose(R, np.eye(3), atol=1e-15)
    t = np.pi / 6
    Rz = np.array([[np.cos(t), -np.sin(t), 0], [np.sin(t), np.cos(t), 0], [0, 0, 1]])
    ok, R, _ = pyoracle.polar(Rz @ np.diag([2, 1, 1]))
    assert ok and np.allclose(R, Rz, atol=1e-12)
    # Degenerate: det <= 1e-12 * (|A|_F/sqrt3)^3 (scale-relative).
    ok, _, _ = pyoracle.polar(np.diag([1.0, 1.0, 0.0]))
    assert not ok
    ok, _, _ = pyoracle.polar(np.diag([1.0, 1.0, -1.0]))
    assert not ok
    # Small but valid moments (config 3's 3^3 boxes) pass.
    ok, R, _ = pyoracle.polar(3e-5 * np.eye(3))
    assert ok and np.allclose(R, np.eye(3))


def test_sym_eigen_matches_reference(pyoracle, golden):
    # math.cpp:26-71 cyclic Jacobi.
    for case in golden["spd"]:
        M = np.array(case["M"]).reshape(3, 3)
        ev, V = pyoracle.sym_eigen(M)
        np.testing.assert_allclose(ev, case["ev"], rtol=1e-12, atol=1e-14 * max(1, abs(M).max()))
        Vr = np.array(case["vecs"]).reshape(3, 3)
        for k in range(3):
            if min(abs(ev[k] - ev[(k + 1) % 3]), abs(ev[k] - ev[(k + 2) % 3])) > 1e-9:
                d = min(np.abs(V[:, k] - Vr[:, k]).max(), np.abs(V[:, k] + Vr[:, k]).max())
                assert d < 1e-9


def test_inertia_solve_matches_reference_pinv(pyoracle, golden):
    # math.cpp:90-108 pseudo-inverse; omega = pinv(I) dL.
    rs = np.random.default_rng(3)
    for case in golden["spd"]:
        M = np.array(case["M"]).reshape(3, 3)
        pinv = np.array(case["pinv"]).reshape(3, 3)
        for _ in range(3):
            dL = rs.normal(size=3)
            if case["rank"] < 3:
                nax = np.array(case["null_axis"])
                dL = dL - dL.dot(nax) * nax  # projected onto the range
            st, w, _ = pyoracle.inertia_solve(M, dL)
            assert st == 0
            np.testing.assert_allclose(w, pinv @ dL, rtol=1e-8, atol=1e-10 * np.abs(pinv @ dL).max() + 1e-300)


def test_inertia_solve_rank_deficient(pyoracle):
    # SPEC.md:61 / :325: diag(0,2,2) is singular about x.
    st, w, axis = pyoracle.inertia_solve(np.diag([0.0, 2.0, 2.0]), [0.0, 0.0, 0.2])
    assert st == 0 and np.allclose(w, [0, 0, 0.1])
    st, w, axis = pyoracle.inertia_solve(np.diag([0.0, 2.0, 2.0]), [1.0, 0.0, 0.2])
    assert st == 2 and abs(abs(axis[0]) - 1) < 1e-12
    # Below 1e-12 along the null axis: projected out silently.
    st, w, _ = pyoracle.inertia_solve(np.diag([0.0, 2.0, 2.0]), [1e-13, 0.0, 0.2])
    assert st == 0 and np.allclose(w, [0, 0, 0.1])


def _one_body_oracle(pyoracle, pos, vel, inv_mass, rest=None):
    pos = np.asarray(pos, float)
    n = len(pos)
    m = 1.0 / np.asarray(inv_mass, float)
    rest = pos if rest is None else np.asarray(rest, float)
    com = (rest * m[:, None]).sum(0) / m.sum()
    sc = P.ArrayScene(position=rest, velocity=vel, inv_mass=inv_mass, radius=np.full(n, 0.01),
                      body_offsets=[0, n], rest_offsets=rest - com, total_mass=[m.sum()],
                      rest_com=[com], has_ground=False)
    o = pyoracle.Oracle(sc.desc, P.solver_cfg(gravity=0.0), threads=1)
    if rest is not pos:
        p4, v4 = o.read_f32()
        p4[:, :3] = pos.astype(np.float32)
        o.write_f32(p4, None)
    return sc, o


def test_body_stats_match_reference(pbdr, pyoracle, golden):
    # compute_com / compute_momentum (body.cpp:50-83) in the oracle's fp32 tree
    # sums vs the reference's fp64 sums.
    for case in golden["bodies"]:
        if case["collinear"]:
            continue
        pos = np.array(case["pos"]).reshape(-1, 3)
        vel = np.array(case["vel"]).reshape(-1, 3)
        sc, o = _one_body_oracle(pyoracle, pos, vel, case["inv_mass"])
        st = o.body_stats()[0]
        scale = max(1.0, np.abs(pos).max())
        np.testing.assert_allclose(st[0:3], case["com"], atol=2e-6 * scale)
        np.testing.assert_allclose(st[7:10], case["P"], atol=1e-5 * max(1, np.abs(case["P"]).max()))
        lref = np.array(case["L"])
        lscale = (np.abs(pos - np.array(case["com"])).max() * np.abs(vel).max() / np.min(case["inv_mass"]) * len(pos))
        np.testing.assert_allclose(st[10:13], lref, atol=1e-5 * max(lscale, 1e-6))


def test_extract_pose_matches_reference(pbdr, pyoracle, golden):
    # extract_pose (body.cpp:103-124): polar of sum m (x - com) q0^T.
    for case in golden["extract_pose"]:
        rest = np.array(case["rest"]).reshape(-1, 3)
        cur = np.array(case["cur"]).reshape(-1, 3)
        sc, o = _one_body_oracle(pyoracle, cur, np.zeros_like(cur), case["inv_mass"], rest=rest)
        st = o.body_stats()[0]
        np.testing.assert_allclose(st[0:3], case["com"], atol=2e-6 * max(1, np.abs(cur).max()))
        q, qref = st[3:7], np.array(case["quat"])
        assert min(np.abs(q - qref).max(), np.abs(q + qref).max()) < 2e-5


def test_warm_started_polar_matches_cold(pyoracle, golden):
    # The warm start (previous rotation, Gauss-Newton on the symmetry
    # condition) converges to the same polar factor as the cold Newton path --
    # to fp32 resolution: the warm steps run in fp32 (PBDR_POLAR_WARM_F32,
    # pbdr_pinned.h; their rotation is rounded to fp32 for the particles anyway).
    rs = np.random.default_rng(11)
    for case in golden["polar"]:
        if case["status"] != 0:
            continue
        A = np.array(case["A"]).reshape(3, 3)
        ok, Rc, qc = pyoracle.polar(A)
        for tilt in (5e-6, 1e-4, 1e-2, 0.2):  # 5e-6: a single Gauss-Newton step
            axis = rs.normal(size=3)
            axis /= np.linalg.norm(axis)
            dq = np.concatenate([[np.cos(tilt / 2)], np.sin(tilt / 2) * axis])
            w0, v0 = qc[0], qc[1:]
            w1, v1 = dq[0], dq[1:]
            rq = np.concatenate([[w0 * w1 - v0 @ v1], w0 * v1 + w1 * v0 + np.cross(v0, v1)])
            okw, Rw, _ = pyoracle.polar_warm(A, rq)
            assert okw
            np.testing.assert_allclose(Rw, Rc, atol=1e-6)
            np.testing.assert_allclose(Rw @ Rw.T, np.eye(3), atol=1e-6)
    ok, R, _ = pyoracle.polar_warm(np.eye(3), np.zeros(4))
    assert ok and np.allclose(R, np.eye(3))
