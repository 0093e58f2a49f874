"""The independent fp64 oracle (oracle/pbdr_oracle64.cpp) on its own, on CPU:
SPEC.md solver-level examples and invariants that a plain fp64 restatement
must meet exactly or to fp64 precision, and agreement with the fp32
bit-exact oracle at the north_star one-step tolerance. The GPU is compared
with it in tests/test_gpu_fp64_oracle.py."""
import numpy as np
import pytest

from paper_2603_14634_b200 import pbdr as P


def cube(n=4, r=0.025, z=1.0, vel=(0.0, 0.0, 0.0), spin=(0.0, 0.0, 0.0), has_ground=False, mu=0.0):
    c = np.stack(np.meshgrid(*[np.arange(n)] * 3, indexing="ij"), -1).reshape(-1, 3) * 2 * r
    c = c - c.mean(0) + [0, 0, z]
    v = np.asarray(vel) + np.cross(np.asarray(spin), c - c.mean(0))
    arr = P.rigid_body_arrays([c], r, [1.0], velocities=[v])
    return P.ArrayScene(**arr, has_ground=has_ground, ground=P.Plane((0, 0, 0), (0, 0, 1), mu))


def test_free_flight_displacement(pyoracle):
    # free body, no gravity, v0 = (1,0,0), 100 steps of dt = 1 ms -> 0.1 m.
    sc = cube(vel=(1.0, 0.0, 0.0))
    o = pyoracle.Oracle64(sc.desc, P.solver_cfg(gravity=0.0), threads=1)
    assert o.step(100) == 0
    p, v = o.read_particles()
    np.testing.assert_allclose(p.mean(0) - sc.position.mean(0), [0.1, 0, 0], atol=1e-12)
    np.testing.assert_allclose(v, np.tile([1.0, 0, 0], (len(v), 1)), atol=1e-12)


def test_momentum_conserved_fp64(pyoracle):
    # SPEC.md:337 (momentum conservation) at fp64: P and L of a spinning,
    # translating free body over 2000 substeps.
    sc = cube(vel=(0.3, -0.2, 0.1), spin=(1.0, 2.0, -0.5))
    o = pyoracle.Oracle64(sc.desc, P.solver_cfg(gravity=0.0), threads=1)
    s0 = o.body_stats()[0]
    assert o.step(2000) == 0
    s1 = o.body_stats()[0]
    assert np.abs(s1[7:10] - s0[7:10]).max() <= 1e-9 * max(1.0, np.abs(s0[7:10]).max())
    assert np.abs(s1[10:13] - s0[10:13]).max() <= 1e-9 * max(1.0, np.abs(s0[10:13]).max())


def test_legacy_equals_incremental_in_fp64(pyoracle):
    # legacy and incremental velocity updates give identical
    # trajectories in double precision within 1e-7 over 100 steps (Test 1:
    # a box sliding on a plane with friction).
    sc = cube(z=0.05 - 0.0, vel=(0.5, 0.0, 0.0), has_ground=True, mu=0.4)
    sc.position[:, 2] -= sc.position[:, 2].min() - 0.025  # resting on the ground
    sc = P.ArrayScene(position=sc.position, velocity=sc.velocity, inv_mass=sc.inv_mass, radius=sc.radius,
                      body_offsets=sc.body_offsets, rest_offsets=sc.rest_offsets, total_mass=sc.total_mass,
                      rest_com=sc.rest_com, has_ground=True, ground=P.Plane((0, 0, 0), (0, 0, 1), 0.4))
    runs = []
    for mode in (1, 0):
        o = pyoracle.Oracle64(sc.desc, P.solver_cfg(velocity_update=mode), threads=1)
        traj = []
        for _ in range(100):
            assert o.step(1) == 0
            traj.append(o.read_particles()[0].copy())
        runs.append(np.array(traj))
    assert np.abs(runs[0] - runs[1]).max() <= 1e-7


@pytest.mark.parametrize("cid,scale", [(1, 0), (2, 0), (3, 24), (4, 3), (5, 6)])
def test_fp64_and_fp32_oracles_agree_one_step(pyoracle, cid, scale):
    # Two restatements that share only the semantic pins: after one frame
    # (10 substeps) positions agree within the north_star 1e-5 m.
    g = P.GeneratedScene(cid, scale=scale)
    o32 = pyoracle.Oracle(g.desc, g.cfg)
    o64 = pyoracle.Oracle64(g.desc, g.cfg)
    assert o32.step(g.cfg.substeps) == 0 and o64.step(g.cfg.substeps) == 0
    assert np.abs(o32.read_particles()[0] - o64.read_particles()[0]).max() <= 1e-5
    s32, s64 = o32.body_stats(), o64.body_stats()
    np.testing.assert_allclose(s32[:, 0:3], s64[:, 0:3], atol=1e-5)


def test_degenerate_body_reported(pyoracle):
    # A planar body: the polar of its moment is degenerate (DegenerateConfigError).
    x = np.stack(np.meshgrid(np.arange(4), np.arange(4), [0], indexing="ij"), -1).reshape(-1, 3) * 0.02
    sc = P.ArrayScene(**P.rigid_body_arrays([x + [0, 0, 1]], 0.01, [1.0]), has_ground=False)
    o = pyoracle.Oracle64(sc.desc, P.solver_cfg(), threads=1)
    assert o.step(1) == P.ERR_DEGENERATE
